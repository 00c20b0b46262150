# per-config device throughput with and without the fused sweep (SK_NO_SWEEP=1)
for c in "$@"; do
  echo "config=$c sweep" >> gpurun_out/cfg.log
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 1 >> gpurun_out/cfg.log 2>&1
  echo "config=$c nosweep" >> gpurun_out/cfg.log
  SK_NO_SWEEP=1 timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 1 >> gpurun_out/cfg.log 2>&1
done
