export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_nc1.so
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('NC1 C5', d['value'], d['roofline']['frac'], d['config']['final_rel_residual'])"
timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1
unset SK_LIB_PATH
python tools/xparity_config.py 3 > gpurun_out/xparity_c3.json 2> gpurun_out/xparity_c3.err; cat gpurun_out/xparity_c3.json; tail -2 gpurun_out/xparity_c3.err
