#!/bin/bash
# ncu capture of one kernel launched by tools/prof_kernel.py (plain run first).
set -e
op=$1; robot=$2; dt=$3; N=$4; regex=$5; out=$6
python tools/prof_kernel.py $op $robot $dt $N 3 > gpurun_out/${out}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$regex -s 1 -c 1 -o gpurun_out/$out python tools/prof_kernel.py $op $robot $dt $N 3 > gpurun_out/${out}_ncu.log 2>&1
