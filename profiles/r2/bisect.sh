T=tests/test_gpu_configs.py
for v in default nofast inl v1; do
  if [ "$v" != "default" ]; then export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so; else unset SK_LIB_PATH; fi
  echo "== variant $v"
  timeout 600 python -m pytest "$T::test_config_bitwise_vs_reproducible_golden[3]" -m gpu -q -x 2>&1 | grep -E "passed|failed|max rel" | tail -2
  timeout 600 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1
done
