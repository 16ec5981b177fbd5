#!/bin/bash
# A/B sweep: default lib and variants x configs x env settings; one summary line each
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in ${CFGS:-2}; do
for v in default $(ls paper_2602_05081_b200/variants/*.so 2>/dev/null); do
 for envs in ${ENVS:-none}; do
  if [ "$v" = default ]; then unset GF_LIB; name=default; else export GF_LIB=$PWD/$v; name=$(basename $v .so); fi
  if [ "$envs" != none ]; then export $envs; fi
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-3} --warmup 2 --no-e2e --no-cpu-baseline 2>gpurun_out/sweep_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$cfg', '$name', '$envs', round(d['value'],2), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['stage_ms_per_step'].items()})" || tail -3 gpurun_out/sweep_err.txt
  if [ "$envs" != none ]; then unset ${envs%%=*}; fi
 done
done
done
