T=tests/test_gpu_configs.py; timeout 900 python -m pytest "$T::test_config_bitwise_vs_reproducible_golden[4]" "$T::test_bicgstab_config_vs_reference_order_golden[4]" -m gpu -q 2>&1 | tail -2
for v in dpad dalla; do
export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
echo "== $v"
python profiles/r2/c3_diff.py /tmp/h_$v.npy 1024 3000 2>&1 | tail -1
python profiles/r2/c3_diff.py /tmp/h2_$v.npy 1024 3000 2>&1 | tail -1
done
