# final round-2 captures with the default build: launch lists for C5 / C3 / C2 / C4 (skip far into
# the runs), one full capture of the C5 fused sweep
bash profiles/run_ncu.sh r2_c5 5 "k_lanczos_cols" 100 1
for cfg in 3 2 4; do
  CMD="python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
  SKIP=8000; [ $cfg = 2 ] && SKIP=9000; [ $cfg = 4 ] && SKIP=3200
  $CMD > gpurun_out/plain_r2_c$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $SKIP -c 200 --csv \
      --log-file gpurun_out/launches_r2_c$cfg.csv $CMD > gpurun_out/ncu_launch_r2_c$cfg.log 2>&1
  echo cfg$cfg rc=$?
done
