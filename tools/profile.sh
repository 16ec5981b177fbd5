#!/bin/bash
# round-end style measurement: gpu tests, full bench, launch list, full captures of the top kernels
# (the 4 launches of the second step = the 4 LOD masks of config 2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/plain.log 2>&1; rc=$?; echo "plain rc=$rc"
if [ $rc = 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu1.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k k_ff_pkt -s 4 -c 4 -f -o gpurun_out/prof_ff \
    python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu2.log 2>&1; echo "ncu ff rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k k_nee_w -s 4 -c 4 -f -o gpurun_out/prof_nee \
    python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu3.log 2>&1; echo "ncu nee rc=$?"
fi
# export on the box (keeps gpurun_out under the 64 MiB copy-back limit)
for f in prof_ff prof_nee; do
  if [ -f gpurun_out/$f.ncu-rep ]; then
    ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
    ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/${f}_sass.csv 2>/dev/null
    rm -f gpurun_out/$f.ncu-rep
  fi
done
