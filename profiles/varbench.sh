# variant sweep: python bench.py on several in-tree library builds (SK_LIB_PATH)
for v in "$@"; do
  if [ "$v" != "default" ]; then export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so; else unset SK_LIB_PATH; fi
  echo "variant=$v" >> gpurun_out/var.log
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 2 >> gpurun_out/var.log 2>&1
done
