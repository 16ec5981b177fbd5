#!/bin/bash
# A/B sweep with work counters: configs x env settings; per run the value, stage times and the work per
# stage (nodes / tests / hits / erfs per path)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in ${CFGS:-2}; do
 for envs in ${ENVS:-none}; do
  if [ "$envs" != none ]; then export $envs; fi
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-3} --warmup 2 --no-e2e --no-cpu-baseline 2>gpurun_out/sweep_err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('cfg$cfg', '$envs', round(d['value'],2), {k: round(v,1) for k,v in d['stage_ms_per_step'].items()})
for st, w in d['work_per_step'].items():
    n = max(1, w.get('paths', 0))
    print('    ', st, {k: (round(v / n, 1) if st != 'ffB' else int(v)) for k, v in w.items()})
" || tail -3 gpurun_out/sweep_err.txt
  if [ "$envs" != none ]; then unset ${envs%%=*}; fi
 done
done
