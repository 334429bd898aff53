#!/usr/bin/env python3
"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into
profiles/<round>_*.{json,txt} — the evidence committed with each round.

Usage: python tools/summarize_profiles.py r01 [REPS_DIR [OUT_DIR]]
(defaults gpurun_out/ and profiles/; on the GPU box the reports stay in /tmp
and only the summaries travel back through gpurun_out/).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__stack_size",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", "smsp__cycles_elapsed.avg",
    "sm__cycles_elapsed.avg", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        d[h] = (v, u)
    return d


def stalls(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    agg, cnt, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        sass = r[idx["Source"]].split()
        if not sass:
            continue
        op = (sass[1] if sass[0].startswith("@") else sass[0]).split(".")[0]
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        agg[op] += s
        cnt[op] += int(float(r[idx["Instructions Executed"]] or 0))
        tot += s
    ninst = sum(cnt.values()) or 1
    return [{"op": op, "stall_pct": round(100 * s / max(tot, 1), 1), "inst_pct": round(100 * cnt[op] / ninst, 1)}
            for op, s in agg.most_common(12)]


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def summarize_rep(name, rep, states, algo_flops, bytes_per_state):
    d = raw(rep)
    m = {k: (to_num(d[k][0]), d[k][1]) for k in METRICS if k in d}
    t = m["gpu__time_duration.sum"]
    t_s = t[0] * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(t[1], 1e-9)

    def mb(key):
        v, u = m[key]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    dram = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    cyc = m.get("smsp__cycles_elapsed.avg", (0, ""))[0]
    pc = lambda k: m.get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed", (0, ""))[0]  # noqa
    executed = (2 * pc("dfma") + pc("dmul") + pc("dadd")) * cyc
    return {
        "kernel": name, "states_per_launch": states, "duration_s_ncu_cold": t_s,
        "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": bytes_per_state * states,
        "traffic_over_algorithmic": round(dram / (bytes_per_state * states), 3),
        "executed_fp64_flops_per_state": round(executed / states, 1),
        "algorithmic_fp64_flops_per_state": algo_flops,
        "metrics": {k: {"value": v, "unit": u} for k, (v, u) in m.items()},
        "top_stalls_by_sass_op": stalls(rep),
    }


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) != len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        if "vdk::" in name:
            short = name.split("(")[0].replace("void vdk::", "")
        per[short[:90]].append(float(r[idx["Metric Value"]].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    return [{"kernel": k, "launches": len(v), "total_ns": sum(v), "share": round(sum(v) / tot, 4)}
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))]


def main():
    global OUT, PROF
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    if len(sys.argv) > 2:
        OUT = sys.argv[2]
    if len(sys.argv) > 3:
        PROF = sys.argv[3]
    os.makedirs(PROF, exist_ok=True)
    sys.path.insert(0, os.path.join(ROOT))
    import bench

    out = {}
    # (key, kernel, states per launch, algorithmic flops / state, algorithmic bytes / state)
    specs = [("chain7_aba_f64", "k_gen_db<GenChain7::Aba, double> (generated, double-buffered cp.async state input, fast fp64 "
                                "sincos)", 4194304,
              bench.flops_per_eval("chain7", "aba"), 224),
             ("tree29_aba_f64", "k_gen_call<GenTree29::Aba, double> (generated, constants from the __constant__ table, routine out of line per state)", 262144, bench.flops_per_eval("tree29", "aba"), 928),
             ("tree29_rnea_f64", "k_gen<GenTree29::Rnea, double> (generated)", 262144,
              bench.flops_per_eval("tree29", "rnea"), 928),
             ("tree29_crba_f64", "k_gen<GenTree29::Crba, double> (generated)", 262144,
              bench.flops_per_eval("tree29", "crba"), 232 + 6728),
             ("tree29_crba_packed_f64", "k_gen<GenTree29::CrbaPacked, double> (generated, 242 packed planes)", 262144,
              bench.flops_per_eval("tree29", "crba"), 232 + 242 * 8),
             ("tree29_osc_f64", "k_gen_osc<GenTree29::Osc23, double> (generated, frame l_palm, out-of-line sin/cos)", 262144, None,
              464 + 232 + 288)]
    for key, name, states, fl, bps in specs:
        rep = os.path.join(OUT, f"{r}_{key}.ncu-rep")
        if os.path.exists(rep):
            out[key] = summarize_rep(name, rep, states, fl, bps)
            with open(os.path.join(PROF, f"{r}_{key}.json"), "w") as f:
                json.dump(out[key], f, indent=1)
    lc = os.path.join(OUT, f"{r}_launches.csv")
    if os.path.exists(lc):
        ls = launches(lc)
        with open(os.path.join(PROF, f"{r}_bench_launches.json"), "w") as f:
            json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py "
                                  "--steps 3 --warmup 3 --no-configs --no-cpu",
                       "note": "cold-cache, serialised launch times: compare shares, not absolutes",
                       "kernels": ls}, f, indent=1)
    for k, v in out.items():
        print(k, "dram/algo", v["traffic_over_algorithmic"], "executed flops/state", v["executed_fp64_flops_per_state"],
              "fp64 pipe %", v["metrics"].get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"))


if __name__ == "__main__":
    main()
