#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU).  Every ncu command is
# preceded by the same command without ncu (B200_PROFILING.md rule).  The
# .ncu-rep files stay in /tmp on the box; summaries (JSON), the headline
# kernel's SASS-level stall listing and the bench launch list come back in
# gpurun_out/prof_<round>/ (copy them to profiles/).
R=${1:-r02}
REPS=/tmp/reps_$R
OUTD=gpurun_out/prof_$R
mkdir -p $REPS $OUTD
set -x
cap() {  # key op robot dtype N kernel-regex
  python tools/prof_kernel.py $2 $3 $4 $5 3 > $OUTD/$1.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$6" -s 1 -c 1 -f -o $REPS/${R}_$1 \
      python tools/prof_kernel.py $2 $3 $4 $5 3 > $OUTD/$1.ncu.log 2>&1
}
cap chain7_aba_f64 aba chain7 f64 4194304 'k_gen|k_tiled|k_aba'
cap tree29_aba_f64 aba tree29 f64 262144 'k_gen'
cap tree29_rnea_f64 rnea tree29 f64 262144 'k_gen'
cap tree29_crba_f64 crba tree29 f64 262144 'k_gen'
cap tree29_crba_packed_f64 crbap tree29 f64 262144 'k_gen'
cap tree29_osc_f64 osc tree29 f64 262144 'k_gen_osc'
ncu -i $REPS/${R}_chain7_aba_f64.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUTD/${R}_chain7_aba_f64_sass.csv.gz
python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > $OUTD/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $REPS/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-configs --no-cpu > $OUTD/ncu_launch.log 2>&1
python tools/summarize_profiles.py $R $REPS $OUTD > $OUTD/summary.txt 2>&1
cp $REPS/${R}_launches.csv $OUTD/ 2>/dev/null
echo captured
