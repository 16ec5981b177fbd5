exec > gpurun_out/tomo_ab.txt 2>&1
python -m pytest tests -m gpu -x -q -k "tomo or smoke or abi" 2>&1 | tail -3
for c in 1 2 3 5; do
python bench.py --config $c --tomography --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print($c,'pkt',l['value'],l['roofline']['frac'],l['ms_per_step'])"
GF_DEBUG_NO_CAMERA_BVH=1 python bench.py --config $c --tomography --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print($c,'warp',l['value'],l['roofline']['frac'],l['ms_per_step'])"
done
