python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -4
python bench.py > gpurun_out/bench_c5_final.json 2> gpurun_out/bench_c5_final.err; tail -c 1500 gpurun_out/bench_c5_final.json; tail -2 gpurun_out/bench_c5_final.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; cat gpurun_out/bench_ref_final.json | cut -c1-900; tail -2 gpurun_out/bench_ref_final.err
for c in 1 2 3 4; do python bench.py --config $c --steps 2 --warmup 1 --no-factors > gpurun_out/bench_c${c}_final.json 2> gpurun_out/bench_c${c}_final.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c${c}_final.json')); print('C$c', d['ms_per_step'], d['config']['iterations_per_step'], d['config']['status'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['bound'], round(d['roofline']['whole_step_frac'],3), d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))"; done
