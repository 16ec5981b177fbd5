#!/bin/bash
# full ncu captures of the round's new kernels: k_tomo_pkt (bench --tomography, cfg2: the mask-{0..3}
# launch of step 2) and k_grad_pkt (tools/bench_grad.py: a mask-{0..3} launch); each command first
# runs plain and must exit 0
mkdir -p gpurun_out
B="python bench.py --config 2 --tomography --profile-pass --steps 1 --warmup 1"
timeout 300 $B > gpurun_out/plain_tomo.log 2>&1; rc=$?; echo "plain tomo rc=$rc"
if [ $rc = 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tomo.csv \
    $B > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k k_tomo_pkt -s 4 -c 4 -f -o gpurun_out/prof_tomo \
    $B > gpurun_out/ncu_t.log 2>&1; echo "ncu tomo rc=$?"
fi
G="python tools/bench_grad.py"
timeout 300 $G > gpurun_out/plain_grad.log 2>&1; rc=$?; echo "plain grad rc=$rc"
if [ $rc = 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k k_grad_pkt -s 31 -c 1 -f -o gpurun_out/prof_grad \
    $G > gpurun_out/ncu_g.log 2>&1; echo "ncu grad rc=$?"
fi
for f in prof_tomo prof_grad; do
  if [ -f gpurun_out/$f.ncu-rep ]; then
    ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
    rm -f gpurun_out/$f.ncu-rep
  fi
done
