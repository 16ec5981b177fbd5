#!/bin/bash
# profile: tools/prof.sh <config> <tag> <kernel regex> [<kernel regex> ...]
# plain run (must exit 0), ncu launch list, then one --set full capture per kernel regex; "name:skip" picks
# the launch (default skip 2)
cfg=$1; tag=$2; shift 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/plain_$tag.log 2>&1; rc=$?
echo "plain rc=$rc"; [ $rc = 0 ] || { tail -20 gpurun_out/plain_$tag.log; exit 1; }
[ -n "$NO_LAUNCHES" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_l_$tag.log 2>&1; echo "launches rc=$?"
for ks in "$@"; do
  k=${ks%%:*}; skip=2; [ "$k" != "$ks" ] && skip=${ks#*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k $k -s $skip -c 1 -f -o gpurun_out/p_${tag}_${k}_$skip \
    python bench.py --config $cfg --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_${tag}_${k}_$skip.log 2>&1; echo "ncu $k:$skip rc=$?"
  b=gpurun_out/p_${tag}_${k}_$skip
  if [ -f $b.ncu-rep ]; then
    ncu -i $b.ncu-rep --page raw --csv > ${b}_raw.csv 2>/dev/null
    ncu -i $b.ncu-rep --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
    ncu -i $b.ncu-rep --page details --csv > ${b}_details.csv 2>/dev/null
    rm -f $b.ncu-rep
  fi
done
