#!/bin/bash
# quick GPU check: the parity suites (no -x), then short bench lines
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/pytest_gpu.txt | tail -25
fi
for c in ${BENCH_CFGS:-2}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "bench cfg$c rc=$?"; python - <<PY
import json
try:
    d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1])
    print('cfg$c', round(d['value'],2), 'Mrays/s', {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'hbm frac', round(d['roofline']['frac'],3))
    print('   work', {k: {kk: int(vv) for kk, vv in v.items()} for k, v in d['work_per_step'].items()})
except Exception as e:
    print('cfg$c parse failed', e); print(open('gpurun_out/bench_cfg$c.err').read()[-2000:])
PY
done
