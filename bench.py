#!/usr/bin/env python3
"""Device-timed benchmark of the batched dynamics hot path (BASELINE.json).

Headline (`value`): Franka Panda (robots::chain7) forward dynamics by the
articulated-body algorithm, fp64, N = 4,194,304 random states per GPU (weak
scaling across ranks), inputs resident in HBM (705 MB/GPU of q, q̇, τ: larger
than the 126 MB L2, so no flush is needed between steps).  One step = one
vd_aba launch over the rank's shard.  Throughput = states / s over all ranks,
step time = max over ranks (CUDA events on the launching stream).

e2e: the same metric through the public host API (vd_batch_forward_dynamics_host
= batch_forward_dynamics, batch.hpp:154-165) from pinned host buffers: H2D of
q, q̇, τ, the kernel, D2H of q̈ inside the timed region.

Also measured in the same run (reported under "configs"): the other
BASELINE.json configurations (FK + Jacobian, fused M/bias/ABA fp32+fp64, G1
RNEA + ABA, OSC for Panda and G1).

cpu_baseline / --impl reference: the reference CPU path — the oracle's
restatement of forward_dynamics (CRBA + bias + LLT, dynamics.hpp:421-444) run
through batch_eval's static std::thread chunking (batch.hpp:82-125) on all host
cores, on a bounded sample of the same random states.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "dynamics evals/sec (Panda & G1 ABA/RNEA) vs batch, 1/2/4/8 B200, % roofline"
N_HEAD = 4194304
SEED = 2604


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-configs", action="store_true", help="skip the secondary configuration sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    return ap.parse_args()


def init_dist(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        backend = "nccl" if (args.impl == "ours" and torch.cuda.is_available()) else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled through NVML (nvidia-ml-py) every
    ~2 ms in a background thread for the duration of the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu):
        self.gpu = gpu
        self.sm, self.mask, self.max = [], 0, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.nv = None
        return self

    def _run(self):
        while not self._stop.is_set():
            try:
                self.sm.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.mask |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max,
                "reasons": reasons, "samples": len(self.sm), "source": "NVML during the timed region"}


# ------------------------------------------------------------------ helpers
def event_time(fn, steps, warmup, stream):
    """Average ms per call of fn() measured with CUDA events on `stream`."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    return e0.elapsed_time(e1) / steps


def graph_time(fn_s, steps, warmup, per_graph=20):
    """Average ms per call of fn_s(stream_ptr), replayed from a CUDA graph of
    per_graph back-to-back calls on a side stream: for small batches, where
    one host call per step would time the host launch path instead of the GPU.
    Falls back to None when capture is not possible."""
    import torch

    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    try:
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn_s(sp)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_graph):
                fn_s(sp)
        torch.cuda.synchronize()
    except Exception:  # noqa: BLE001
        return None
    reps = max(2, steps // per_graph)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * per_graph)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return {}


def flops_per_eval(robot, algo, dense=False):
    """Frozen algorithmic flops per evaluation from the op-counting oracle
    (oracle/orc_count.hpp): the recursive algorithm instantiated with a
    counting scalar.  Default: structure-aware count (ops with a structural
    zero / unit operand are free — the work the robot's structure requires);
    dense=True: every 6x6 / 3x3 op of the generic recursion."""
    import oracle_ffi

    L = oracle_ffi.lib()
    L.orc_count_flops.restype = ctypes.c_double
    L.orc_count_flops.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    m = oracle_ffi.Model.builtin(robot)
    code = {"rnea": 0, "crba": 1, "aba": 2, "fk": 3}[algo]
    return L.orc_count_flops(m.h, code if dense else code + 100, None)


_CPU_SAMPLE = {}


def cpu_reference_rate(robot, threads, target_s=12.0, op="fd", batch=262144):
    """Reference CPU path (LLT forward dynamics / mask RNEA) on host cores:
    repeated passes over one seeded batch until ~target_s of CPU work."""
    import oracle_ffi

    key = (robot, batch)
    if key not in _CPU_SAMPLE:
        om = oracle_ffi.Model.builtin(robot)
        _CPU_SAMPLE[key] = (om, om.random_states(batch, SEED, True, True))
    om, (q, qd, qdd, tau) = _CPU_SAMPLE[key]
    n_done, t0 = 0, time.perf_counter()
    while True:
        if op == "fd":
            om.forward_dynamics(q, qd, tau, threads=threads)
        else:
            om.rnea(q, qd, qdd, threads=threads)
        n_done += batch
        dt = time.perf_counter() - t0
        if dt >= target_s:
            return n_done / dt, n_done, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def headline_config(world):
    """The headline workload's `config`, identical in both arms (the driver
    compares them); the algorithm each arm runs is reported beside it."""
    return {"workload": f"chain7 (Franka Panda stand-in, robots::chain7) forward dynamics qdd = FD(q, qd, tau), "
                        f"fp64, {N_HEAD} random states per GPU", "robot": "chain7", "dof": 7,
            "states_per_gpu": N_HEAD, "global_batch": N_HEAD * world, "parallelism": f"dp{world} (batch shards)",
            "l2": "inputs 705 MB/GPU > 126 MB L2 (no flush needed)", "seed": SEED}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = init_dist(args)
    if rank != 0:
        return 0
    threads = host_cores()
    vals = []
    for _ in range(args.warmup):
        cpu_reference_rate("chain7", threads, target_s=0.5)
    total_n, total_t = 0, 0.0
    for _ in range(args.steps):
        r, n, dt = cpu_reference_rate("chain7", threads, target_s=2.0)
        vals.append(r)
        total_n += n
        total_t += dt
    value = total_n / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(world),
        "algorithm": "reference CPU path: CRBA + RNEA bias + LLT (dynamics.hpp:421-444) via batch_eval threads "
                     "(batch.hpp:82-125), oracle port built -O3 -march=x86-64-v3",
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"bounded sample of the workload: {int(total_n / args.steps)} evaluations per "
                                   f"step (repeated passes over 262144 random chain7 states, mt19937_64 seed "
                                   f"{SEED}), {threads} threads, {cpu_model()}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch

    rank, world, local = init_dist(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2604_04310_b200 as vd
    from paper_2604_04310_b200 import dist as vdist

    lib = vd._lib.load()
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)

    # ---------------- headline: chain7 ABA fp64, N_HEAD states per GPU
    model = vd.robots.chain7()
    dm = vd.DeviceModel(model, local)
    n = model.dof()
    N = N_HEAD
    g = torch.Generator(device=dev).manual_seed(SEED + rank)
    rnd = lambda dt=torch.float64: ((torch.rand((n, N), generator=g, device=dev, dtype=dt) * 2 - 1) * np.pi)  # noqa
    q, qd, tau = rnd(), rnd(), rnd()
    qdd = torch.empty((n, N), dtype=torch.float64, device=dev)
    status = torch.empty(N, dtype=torch.int32, device=dev)

    def step():
        rc = lib.vd_aba(dm.handle, 0, N, q.data_ptr(), qd.data_ptr(), tau.data_ptr(), N, None, None, qdd.data_ptr(), N,
                        status.data_ptr(), sptr)
        if rc:
            raise RuntimeError(lib.vd_last_error().decode())

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = vdist.max_over_ranks(ms_local, device=dev)
    value = N * world / (ms * 1e-3)
    assert int(status.max()) == 0

    # per-launch duration of the dominant kernel (it is the only kernel in the step)
    flops = flops_per_eval("chain7", "aba")
    flops_dense = flops_per_eval("chain7", "aba", dense=True)
    bytes_per_eval = 8 * n * 4  # q, qd, tau in; qdd out
    achieved_tf = flops * N / (ms_local * 1e-3) / 1e12
    lib.vdi_fma_peak_tflops.restype = ctypes.c_double
    lib.vdi_fma_peak_tflops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    fp64_peak = lib.vdi_fma_peak_tflops(local, 0, 200)
    fp32_peak = lib.vdi_fma_peak_tflops(local, 1, 200)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    roofline = {
        "bound": "fp64", "achieved": round(achieved_tf, 4), "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
        "frac": round(achieved_tf / fp64_peak, 4) if fp64_peak > 0 else None, "traffic": None,
        "flops_per_eval": flops, "flops_per_eval_dense": flops_dense,
        "flops_source": "frozen structure-aware op count of the oracle's aba_loop (oracle/orc_count.hpp)",
        "peak_source": "measured in this run: FP64 FMA-stream microbenchmark (vdi_fma_peak_tflops)",
        "hbm_gbs_achieved": round(bytes_per_eval * N / (ms_local * 1e-3) / 1e9, 1), "hbm_gbs_peak": hbm,
        "hbm_frac": round(bytes_per_eval * N / (ms_local * 1e-3) / 1e9 / hbm, 4),
    }
    # DRAM traffic per launch of this kernel at this N from the committed
    # `ncu --set full` capture (tools/capture_profiles.sh; ncu cannot run
    # inside the timed bench)
    prof = next((os.path.join(ROOT, "profiles", f"{r}_chain7_aba_f64.json") for r in ("r02d", "r02b", "r02", "r01")
                 if os.path.exists(os.path.join(ROOT, "profiles", f"{r}_chain7_aba_f64.json"))), "")
    if prof:
        with open(prof) as f:
            pj = json.load(f)
        if int(pj.get("states_per_launch", 0)) == N:
            roofline["traffic"] = pj["dram_bytes_per_launch"]
            roofline["traffic_over_algorithmic"] = pj["traffic_over_algorithmic"]
            roofline["traffic_source"] = (f"profiles/{os.path.basename(prof)} (ncu --set full, "
                                          "dram__bytes_read+write)")

    # ---------------- e2e through the public host API (pinned buffers)
    e2e = None
    try:
        hq = torch.empty((n, N), dtype=torch.float64, pin_memory=True)
        hqd = torch.empty_like(hq).pin_memory()
        htau = torch.empty_like(hq).pin_memory()
        hout = torch.empty_like(hq).pin_memory()
        hst = torch.empty(N, dtype=torch.int32).pin_memory()
        hq.copy_(q.cpu())
        hqd.copy_(qd.cpu())
        htau.copy_(tau.cpu())
        devs = (ctypes.c_int * 1)(local)

        def e2e_step():
            rc = lib.vd_batch_forward_dynamics_host(model.handle, N, hq.data_ptr(), hqd.data_ptr(), htau.data_ptr(),
                                                    None, hout.data_ptr(), hst.data_ptr(), devs, 1)
            if rc:
                raise RuntimeError(lib.vd_last_error().decode())

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        k = max(3, args.steps // 4)
        for _ in range(k):
            e2e_step()
        t1 = time.perf_counter()
        barrier()
        e2e_ms = vdist.max_over_ranks((t1 - t0) * 1e3 / k, device=dev)
        got = hout.to(dev)
        same = bool(torch.equal(got, qdd))
        diff = float(((got - qdd).abs().amax(0) / qdd.abs().amax(0).clamp(min=1)).max())
        e2e = {"value": N * world / (e2e_ms * 1e-3), "unit": "evals/s", "h2d_bytes_per_step": 3 * n * N * 8,
               "d2h_bytes_per_step": n * N * 8 + N * 4, "ms_per_step": e2e_ms,
               "api": "vd_batch_forward_dynamics_host (batch_forward_dynamics, batch.hpp:154-165)",
               "bitwise_equal_to_device_run": same, "max_rel_diff_vs_device_run": diff}
        del hq, hqd, htau, hout
    except Exception as ex:  # noqa: BLE001
        e2e = {"value": None, "unit": "evals/s", "error": str(ex)}

    # ---------------- secondary configurations (same run)
    configs = {}
    if not args.no_configs:
        configs = run_configs(vd, lib, dev, stream, sptr, args, rank, world)

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = host_cores()
        r, ns, dt = cpu_reference_rate("chain7", threads, target_s=12.0)
        cpu = {"value": r, "unit": "evals/s", "cores": threads, "kind": "port",
               "sample": f"{ns} evaluations (repeated passes over 262144 random chain7 states, seed {SEED}) of "
                         f"the reference forward_dynamics (CRBA + bias + LLT) in {dt:.1f} s on {threads} threads, "
                         f"{cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": headline_config(world),
            "algorithm": "ABA (articulated-body algorithm), generated straight-line sm_100a kernel, one thread "
                         "per state",
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "fp32_peak_tflops": round(fp32_peak, 3),
            "configs": configs,
        }
        print(json.dumps(line))
    return 0


def run_configs(vd, lib, dev, stream, sptr, args, rank, world):
    """The other BASELINE.json configurations, device-timed in the same run."""
    import torch

    out = {}
    steps, warm = max(5, args.steps // 2), 3
    gen = torch.Generator(device=dev).manual_seed(SEED + 7)

    def states(n, N, dt):
        return [((torch.rand((n, N), generator=gen, device=dev, dtype=torch.float64) * 2 - 1) * np.pi).to(dt)
                for _ in range(3)]

    def rec(key, N, ms, flops=None, extra=None):
        d = {"states": N, "ms": round(ms, 5), "evals_per_s": N / (ms * 1e-3)}
        if flops:
            d["algorithmic_tflops"] = round(flops * N / (ms * 1e-3) / 1e12, 4)
        if extra:
            d.update(extra)
        out[key] = d

    chain = vd.robots.chain7()
    tree = vd.robots.tree29()
    dc, dt_ = vd.DeviceModel(chain, dev.index), vd.DeviceModel(tree, dev.index)

    # config 1: Panda RNEA on one random state.  The reference number is CPU
    # latency (CLOCK_MONOTONIC, median of 10,000 calls) of the
    # oracle port's rnea on one host thread; beside it the device time of one
    # vd_rnea call at N = 1 (host launch included) and its CUDA-graph replay.
    if True:  # every rank (event_time's barriers)
        import oracle_ffi

        L = oracle_ffi.lib()
        L.orc_rnea_latency_ns.restype = ctypes.c_double
        L.orc_rnea_latency_ns.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64]
        cpu_ns = L.orc_rnea_latency_ns(oracle_ffi.Model.builtin("chain7").h, 10000, SEED + 1)
        q1, qd1, qdd1 = states(7, 1, torch.float64)
        tau1 = torch.empty((7, 1), dtype=torch.float64, device=dev)
        fn1 = lambda sp: lib.vd_rnea(dc.handle, 0, 1, q1.data_ptr(), qd1.data_ptr(), qdd1.data_ptr(), 1, None,  # noqa
                                     None, tau1.data_ptr(), 1, sp)
        g1 = graph_time(fn1, 400, 20)
        out["1_panda_rnea_single_state_f64"] = {
            "states": 1, "cpu_reference_median_ns": round(cpu_ns, 1), "cpu_threads": 1,
            "gpu_ms_one_call": round(event_time(lambda: fn1(sptr), 200, 20, stream), 5),
            "gpu_ms_graph": round(g1, 5) if g1 else None,
            "note": "latency, not throughput: a single state is the reference's CPU use case (config 1)"}

    # config 2: Panda FK + EE Jacobian, batch 4096
    for dt, code in ((torch.float64, 0), (torch.float32, 1)):
        N = 4096
        q, _, _ = states(7, N, dt)
        pose = torch.empty((12, N), dtype=dt, device=dev)
        J = torch.empty((42, N), dtype=dt, device=dev)
        fid = chain.frame_index("ee")
        pq, pp, pj = q.data_ptr(), pose.data_ptr(), J.data_ptr()
        fn_s = lambda sp: lib.vd_jacobian(dc.handle, code, N, pq, N, fid, pp, pj, N, sp)  # noqa
        key = f"2_panda_fk_jacobian_b4096_{'f64' if code == 0 else 'f32'}"
        rec(key, N, event_time(lambda: fn_s(sptr), 200, 20, stream), flops_per_eval("chain7", "fk"))
        gms = graph_time(fn_s, 400, 20)
        if gms:  # the per-call loop above is host-launch bound at this size
            out[key].update({"ms_graph": round(gms, 5), "evals_per_s_graph": N / (gms * 1e-3),
                             "note": "ms: one host call per step; ms_graph: CUDA-graph replay of the same calls"})
    # config 3: Panda M + bias + ABA (fused), batch 65536, fp32 and fp64
    for dt, code in ((torch.float64, 0), (torch.float32, 1)):
        N = 65536
        q, qd, tau = states(7, N, dt)
        M = torch.empty((49, N), dtype=dt, device=dev)
        b = torch.empty((7, N), dtype=dt, device=dev)
        a = torch.empty((7, N), dtype=dt, device=dev)
        ptrs = [t.data_ptr() for t in (q, qd, tau, M, b, a)]  # resolved once, as a C caller holds them
        fn_s = lambda sp: lib.vd_dynamics(dc.handle, code, N, ptrs[0], ptrs[1], ptrs[2], N, None,  # noqa
                                          ptrs[3], ptrs[4], ptrs[5], N, None, sp)
        fl = flops_per_eval("chain7", "crba") + flops_per_eval("chain7", "rnea") + flops_per_eval("chain7", "aba")
        key = f"3_panda_M_bias_aba_b65536_{'f64' if code == 0 else 'f32'}"
        rec(key, N, event_time(lambda: fn_s(sptr), 50, warm, stream), fl)
        gms = graph_time(fn_s, 200, 20)
        if gms:  # ~20 us per call: the one-call-per-step loop can be host-bound here
            out[key].update({"ms_graph": round(gms, 5), "evals_per_s_graph": N / (gms * 1e-3),
                             "algorithmic_tflops_graph": round(fl * N / (gms * 1e-3) / 1e12, 4),
                             "note": "ms: one host call per step; ms_graph: CUDA-graph replay of the same calls"})
    # config 4: G1 RNEA + ABA, batch 262144 (fp64 and fp32)
    for dt, code in ((torch.float64, 0), (torch.float32, 1)):
        N = 262144
        q, qd, x = states(29, N, dt)
        t = torch.empty((29, N), dtype=dt, device=dev)
        a = torch.empty((29, N), dtype=dt, device=dev)
        f_r = lambda: lib.vd_rnea(dt_.handle, code, N, q.data_ptr(), qd.data_ptr(), x.data_ptr(), N, None, None,  # noqa
                                  t.data_ptr(), N, sptr)
        f_a = lambda: lib.vd_aba(dt_.handle, code, N, q.data_ptr(), qd.data_ptr(), x.data_ptr(), N, None, None,  # noqa
                                 a.data_ptr(), N, None, sptr)
        sfx = "f64" if code == 0 else "f32"
        rec(f"4_g1_rnea_b262144_{sfx}", N, event_time(f_r, steps, warm, stream), flops_per_eval("tree29", "rnea"))
        rec(f"4_g1_aba_b262144_{sfx}", N, event_time(f_a, steps, warm, stream), flops_per_eval("tree29", "aba"))
    # config 4': G1 CRBA, batch 262144 fp64: dense M (841 planes, the reference's
    # output) vs the branch-sparse packed lower triangle (242 planes); both HBM bound
    N = 262144
    q, _, _ = states(29, N, torch.float64)
    nnz = len(tree.crba_pattern()[0])
    Md = torch.empty((29 * 29, N), dtype=torch.float64, device=dev)
    Mp = torch.empty((nnz, N), dtype=torch.float64, device=dev)
    f_d = lambda: lib.vd_crba(dt_.handle, 0, N, q.data_ptr(), N, Md.data_ptr(), N, sptr)  # noqa
    f_p = lambda: lib.vd_crba_packed(dt_.handle, 0, N, q.data_ptr(), N, Mp.data_ptr(), N, sptr)  # noqa
    for key, fn, planes in (("4p_g1_crba_dense_b262144_f64", f_d, 29 * 29), ("4p_g1_crba_packed_b262144_f64", f_p, nnz)):
        ms = event_time(fn, steps, warm, stream)
        byts = (29 + planes) * 8 * N
        rec(key, N, ms, flops_per_eval("tree29", "crba"),
            {"out_planes": planes, "hbm_gbs": round(byts / (ms * 1e-3) / 1e9, 1),
             "hbm_frac": round(byts / (ms * 1e-3) / 1e9 / measured_peaks().get("hbm_gbs", 6650.0), 4)})
    del Md, Mp, q
    # the headline workload in fp32 (the north star's fp32 mode, 1e-4 parity):
    # Panda ABA, 4M states per GPU, generated kernel with double-buffered async state input
    N = N_HEAD
    q, qd, x = states(7, N, torch.float32)
    a32 = torch.empty((7, N), dtype=torch.float32, device=dev)
    f32 = lambda: lib.vd_aba(dc.handle, 1, N, q.data_ptr(), qd.data_ptr(), x.data_ptr(), N, None, None,  # noqa
                             a32.data_ptr(), N, None, sptr)
    ms = event_time(f32, steps, warm, stream)
    rec("headline_panda_aba_b4194304_f32", N, ms, flops_per_eval("chain7", "aba"),
        {"fp32_peak_frac_note": "algorithmic TFLOP/s against the in-run FP32 FMA peak: see fp32_peak_tflops"})
    del q, qd, x, a32
    # config 5: OSC terms, batch 4M (per GPU), Panda and G1
    for robot, dmod, frame in (("chain7", dc, "ee"), ("tree29", dt_, "l_palm")):
        m = chain if robot == "chain7" else tree
        n = m.dof()
        N = 4194304  # config 5: batch 4M per GPU for both robots
        q, qd, _ = states(n, N, torch.float64)
        P = vd._lib.OscParams()
        P.frame = m.frame_index(frame)
        z = torch.zeros((1, n), dtype=torch.float64, device=dev)
        pose = vd.frame_transform(dmod, z, frame).cpu().numpy()[0]
        for k in range(12):
            P.target[k] = float(pose[k])
        for k in range(6):
            P.kp[k], P.kd[k], P.accel_ff[k] = 100.0, 20.0, 0.0
        post = (ctypes.c_double * n)(*([0.0] * n))
        P.posture = ctypes.cast(post, vd._lib.Pd)
        P.posture_kp, P.posture_kd = 10.0, 2.0
        P.gravity[0], P.gravity[1], P.gravity[2] = 0.0, 0.0, 9.81
        P.epsilon = 1e-6
        tau = torch.empty((n, N), dtype=torch.float64, device=dev)
        lam = torch.empty((36, N), dtype=torch.float64, device=dev)
        fn = lambda: lib.vd_osc(dmod.handle, 0, N, q.data_ptr(), qd.data_ptr(), N, ctypes.byref(P),  # noqa
                                tau.data_ptr(), lam.data_ptr(), N, None, sptr)
        rec(f"5_{'panda' if robot == 'chain7' else 'g1'}_osc_b{N}_f64", N, event_time(fn, 5, 2, stream),
            None, {"note": "tau + Lambda outputs"})
        del q, qd, tau, lam
        torch.cuda.empty_cache()
    out["batch_sweep"] = batch_sweep(vd, lib, dev, stream, sptr, dc, dt_)
    return out


def batch_sweep(vd, lib, dev, stream, sptr, dc, dt_):
    """evals/s vs batch size (BASELINE.json: "... vs batch"), fp64, device-timed:
    Panda and G1, ABA and RNEA, from 1 K states (launch/latency bound) to the
    full configurations (compute bound).  Sizes ≤ 64 K are also timed as CUDA
    graph replays (no host launch path per call); the faster figure is kept."""
    import torch

    res = {}
    gen = torch.Generator(device=dev).manual_seed(SEED + 11)
    for robot, dmod, n, Nmax in (("panda", dc, 7, 4194304), ("g1", dt_, 29, 1048576)):
        x = [((torch.rand((n, Nmax), generator=gen, device=dev, dtype=torch.float64) * 2 - 1) * np.pi)
             for _ in range(3)]
        y = torch.empty((n, Nmax), dtype=torch.float64, device=dev)
        for op in ("aba", "rnea"):
            row = {}
            N = 1024
            while N <= Nmax:
                if op == "aba":
                    fn = lambda N=N: lib.vd_aba(dmod.handle, 0, N, x[0].data_ptr(), x[1].data_ptr(),  # noqa
                                                x[2].data_ptr(), Nmax, None, None, y.data_ptr(), Nmax, None, sptr)
                else:
                    fn = lambda N=N: lib.vd_rnea(dmod.handle, 0, N, x[0].data_ptr(), x[1].data_ptr(),  # noqa
                                                 x[2].data_ptr(), Nmax, None, None, y.data_ptr(), Nmax, sptr)
                ms = event_time(fn, 20 if N < 65536 else 10, 3, stream)
                if N <= 65536:  # launch-bound sizes: time graph replays of the same call
                    if op == "aba":
                        fs = lambda sp, N=N: lib.vd_aba(dmod.handle, 0, N, x[0].data_ptr(), x[1].data_ptr(),  # noqa
                                                        x[2].data_ptr(), Nmax, None, None, y.data_ptr(), Nmax, None,
                                                        sp)
                    else:
                        fs = lambda sp, N=N: lib.vd_rnea(dmod.handle, 0, N, x[0].data_ptr(), x[1].data_ptr(),  # noqa
                                                         x[2].data_ptr(), Nmax, None, None, y.data_ptr(), Nmax, sp)
                    gms = graph_time(fs, 100, 3)
                    ms = min(ms, gms) if gms else ms
                row[str(N)] = round(N / (ms * 1e-3), 1)
                N *= 4
            res[f"{robot}_{op}_f64_evals_per_s"] = row
        del x, y
        torch.cuda.empty_cache()
    return res


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
