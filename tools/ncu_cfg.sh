#!/bin/bash
# tools/ncu_cfg.sh <config> <kernel> <skip> <count> <name>: full ncu capture of launches of one kernel
timeout 600 python bench.py --config $1 --profile-pass --steps 1 --warmup 1 > gpurun_out/plain_$5.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k $2 -s $3 -c $4 -f -o gpurun_out/$5 \
  python bench.py --config $1 --profile-pass --steps 1 --warmup 1 > gpurun_out/ncu_$5.log 2>&1; echo "ncu rc=$?"
