timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('RED5 C5', d['value'], d['roofline']['frac'], d['config']['final_rel_residual'])"
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1; done
python profiles/r2/c3_diff.py /tmp/h_a.npy 1024 3000 2>&1 | tail -1
python profiles/r2/c3_diff.py /tmp/h_b.npy 1024 3000 2>&1 | tail -1
T=tests/test_gpu_configs.py; timeout 900 python -m pytest "$T::test_config_bitwise_vs_reproducible_golden[3]" "$T::test_config_bitwise_vs_reproducible_golden[5]" "$T::test_config_bitwise_vs_reproducible_golden[1]" -m gpu -q 2>&1 | tail -2
