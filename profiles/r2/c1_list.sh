CMD="python bench.py --config 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_r2_c1.log 2>&1 && tail -1 gpurun_out/plain_r2_c1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C1', d['ms_per_step'], d['config']['iterations_per_step'], d['gpu_launches'], json.dumps(d['roofline']['classes']))"
ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 300 --csv --log-file gpurun_out/launches_r2_c1.csv $CMD > gpurun_out/ncu_launch_r2_c1.log 2>&1
echo rc=$?
