timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_configs.py -m gpu -q 2>&1 | tail -3
for c in 1 3 5; do python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C$c', d['ms_per_step'], d['value'], d['gpu_launches'], d['config']['status'])"; done
