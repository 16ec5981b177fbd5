for v in default paper_2602_05081_b200/variants/gradp5.so paper_2602_05081_b200/variants/gradp6.so paper_2602_05081_b200/variants/gradp8.so; do
  if [ $v = default ]; then unset GF_LIB; else export GF_LIB=$PWD/$v; fi
  python tools/bench_grad.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', [round(x['grad_params_packets_ms'],2) for x in d['per_mask'].values()])"
done
