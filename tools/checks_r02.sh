#!/bin/bash
# GPU suite on the default library and on the bounds-checked variant (GF_DEBUG_CHECKS, the stand-in for
# compute-sanitizer, which this pool does not run), the uniform-in-segment bias measurement and its
# config-5 bench line
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_gpu.txt
GF_LIB=$PWD/paper_2602_05081_b200/variants/libgf_checked.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_checked.txt 2>&1; echo "checked rc=$?"; tail -2 gpurun_out/r02_checked.txt
timeout 900 python tools/uniform_bias.py > gpurun_out/r02_uniform_bias.json 2> gpurun_out/uniform_bias.err; echo "bias rc=$?"
timeout 900 python bench.py --estimator uniform --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_cfg5_uniform.json 2> gpurun_out/uni.err; echo "uniform bench rc=$?"
