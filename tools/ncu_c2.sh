#!/bin/bash
# ncu evidence for round summaries (run on the GPU box from the repo root):
#   1. launch list (gpu__time_duration, cold cache, serialised) of the timed step of bench.py
#      (the three warm-up steps run unprofiled: --launch-skip)
#   2. one --set full capture per hot kernel family of a C2 factorization + solve
set -x
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 38000 --launch-count 13000 \
    --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-microbench > gpurun_out/bench_under_ncu.json 2>&1
for spec in "k_qr_tile:0" "k_cpqr_narrow:100" "k_assemble:0" "k_stats:0" "k_wsweep:50" "k_wsweep_big:10" "k_cpqr:0"; do
    k=${spec%%:*}; skip=${spec##*:}
    REPS=1 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name "regex:^${k}\$|^${k}<" \
        --launch-skip $skip --launch-count 1 -o gpurun_out/c2_${k} python tools/time_c2.py > gpurun_out/ncu_${k}.log 2>&1
done
ls -la gpurun_out
