T=tests/test_gpu_configs.py
for v in dsync dtop; do
  export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
  echo "== variant $v"
  for i in 1 2; do timeout 600 python -m pytest "$T::test_config_bitwise_vs_reproducible_golden[3]" -m gpu -q -x 2>&1 | grep -E "passed|failed" | tail -1; done
done
