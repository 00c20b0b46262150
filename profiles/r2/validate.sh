python profiles/r2/c3_diff.py /tmp/h_a.npy 1024 3000 2>&1 | tail -1
python profiles/r2/c3_diff.py /tmp/h_b.npy 1024 3000 2>&1 | tail -1
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_sweep.py -m gpu -q -x 2>&1 | tail -1; done
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5_r2b.json 2> gpurun_out/bench_c5_r2b.err; tail -c 2500 gpurun_out/bench_c5_r2b.json
