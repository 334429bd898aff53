#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU).  Every ncu command is
# preceded by the same command without ncu (B200_PROFILING.md rule).
R=${1:-r01}
set -x
python tools/prof_kernel.py aba chain7 f64 4194304 3 > gpurun_out/${R}_p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_aba -s 1 -c 1 -o gpurun_out/${R}_chain7_aba_f64 \
    python tools/prof_kernel.py aba chain7 f64 4194304 3 > gpurun_out/${R}_n1.log 2>&1
python tools/prof_kernel.py aba tree29 f64 262144 3 > gpurun_out/${R}_p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_aba -s 1 -c 1 -o gpurun_out/${R}_tree29_aba_f64 \
    python tools/prof_kernel.py aba tree29 f64 262144 3 > gpurun_out/${R}_n2.log 2>&1
python tools/prof_kernel.py rnea tree29 f64 262144 3 > gpurun_out/${R}_p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rnea -s 1 -c 1 -o gpurun_out/${R}_tree29_rnea_f64 \
    python tools/prof_kernel.py rnea tree29 f64 262144 3 > gpurun_out/${R}_n3.log 2>&1
python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > gpurun_out/${R}_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > gpurun_out/${R}_ncu_launch.log 2>&1
echo captured
