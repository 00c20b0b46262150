for v in dv1like v1nr; do
  export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
  echo "== variant $v"
  python profiles/r2/c3_diff.py /tmp/h_$v.npy 1024 3000 2>&1 | tail -1
  python profiles/r2/c3_diff.py /tmp/h2_$v.npy 1024 3000 2>&1 | tail -1
done
export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_v1nr.so
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('V1NR C5', d['value'], d['roofline']['frac'], d['config']['final_rel_residual'])"
timeout 600 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1
