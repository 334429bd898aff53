# A/B timing of the generated G1 JVP kernels through the Python API (run under gpurun with PYTHONPATH=repo root).
import torch, sys, paper_2604_04310_b200 as vd
dev=torch.device("cuda:0")
for robot in ["tree29"]:
    m=vd.robots.by_name(robot); dm=vd.DeviceModel(m,0); n=m.dof(); N=262144
    for dt in [torch.float64, torch.float32]:
        g=torch.Generator(device="cuda").manual_seed(1)
        X=[((torch.rand((N,n),generator=g,device="cuda",dtype=torch.float64)*2-1)*3.14159).to(dt) for _ in range(6)]
        fns={"fk_jvp":lambda: vd.forward_kinematics_jvp(dm,X[0],X[1]),
             "rnea_jvp":lambda: vd.rnea_jvp(dm,X[0],X[1],X[2],X[3],X[4],X[5]),
             "crba_jvp":lambda: vd.crba_jvp(dm,X[0],X[1]),
             "aba_jvp":lambda: vd.forward_dynamics_jvp(dm,X[0],X[1],X[2],X[3],X[4],X[5])}
        for k,f in fns.items():
            for _ in range(3): f()
            torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): f()
            b.record(); torch.cuda.synchronize()
            print(robot, dt, k, round(a.elapsed_time(b)/10,4), "ms")
