#!/bin/bash
# full ncu capture of one kernel launch: tools/ncu_one.sh <regex> <skip> <name>
timeout 300 python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k $1 -s $2 -c 1 -f -o gpurun_out/$3 \
  python bench.py --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_$3.log 2>&1; echo "ncu rc=$?"
