for v in default v1nr v2nr; do
  if [ "$v" != "default" ]; then export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so; else unset SK_LIB_PATH; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('VARIANT $v', d['value'], d['roofline']['frac'], d['config']['final_rel_residual'])"
  timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -2
done
