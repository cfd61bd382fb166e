nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r01l.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01l.log 2>&1
echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01l.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py --no-sweep --no-steps > gpurun_out/bench_r01l_quick.jsonl 2> gpurun_out/bench_r01l_quick.err; echo bench_rc=$?
tail -3 gpurun_out/pytest_gpu_r01l.log
