#!/bin/bash
# ncu evidence for round summaries (run on the GPU box from the repo root):
#   1. launch list (gpu__time_duration, cold cache, serialised) of bench.py
#   2. one --set full capture per hot kernel family of a C2 factorization
set -x
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-microbench > gpurun_out/bench_under_ncu.json 2>&1
for k in k_cpqr_narrow k_cpqr_smem k_qr_tile k_assemble k_cpqr; do
    REPS=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name "regex:^${k}\$|^${k}<" \
        --launch-count 1 -o gpurun_out/c2_${k} python tools/time_c2.py > gpurun_out/ncu_${k}.log 2>&1
done
ls -la gpurun_out
