#!/bin/bash
# round-2 closing measurement: default bench line (config 5), the reference arm, bench lines of configs
# 1-4, the config-5 and config-4 ncu launch lists, full captures of the top kernels
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1; echo "reference rc=$?"
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_cfg$c.json 2> gpurun_out/r02_bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv \
  python bench.py --config 5 --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_l5.log 2>&1; echo "launches5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg4.csv \
  python bench.py --config 4 --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_l4.log 2>&1; echo "launches4 rc=$?"
NO_LAUNCHES=1 bash tools/prof.sh 5 r02c5 k_ffa_w:49 k_ffb_w:57 k_ffb_w:56 k_ffa_pkt:7 k_nee_w:56
NO_LAUNCHES=1 bash tools/prof.sh 4 r02c4 k_ffa_w:17 k_ffb_w:17 k_nee_w:17
