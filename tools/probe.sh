nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
