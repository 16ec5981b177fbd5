#!/bin/bash
# profile: tools/prof.sh <config> <tag> <kernel regex> [<kernel regex> ...]
# plain run (must exit 0), ncu launch list, then one --set full capture per kernel regex (2nd step)
cfg=$1; tag=$2; shift 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/plain_$tag.log 2>&1; rc=$?
echo "plain rc=$rc"; [ $rc = 0 ] || { tail -20 gpurun_out/plain_$tag.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_l_$tag.log 2>&1; echo "launches rc=$?"
for k in "$@"; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k $k -s 2 -c 1 -f -o gpurun_out/p_${tag}_$k \
    python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_${tag}_$k.log 2>&1; echo "ncu $k rc=$?"
  if [ -f gpurun_out/p_${tag}_$k.ncu-rep ]; then
    ncu -i gpurun_out/p_${tag}_$k.ncu-rep --page raw --csv > gpurun_out/p_${tag}_${k}_raw.csv 2>/dev/null
    ncu -i gpurun_out/p_${tag}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/p_${tag}_${k}_sass.csv 2>/dev/null
    ncu -i gpurun_out/p_${tag}_$k.ncu-rep --page details --csv > gpurun_out/p_${tag}_${k}_details.csv 2>/dev/null
    rm -f gpurun_out/p_${tag}_$k.ncu-rep
  fi
done
