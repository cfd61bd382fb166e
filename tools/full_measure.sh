set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r01p.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01p.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01p.jsonl 2> gpurun_out/bench_r01p.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r01p.jsonl 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep --no-steps > gpurun_out/plain_r01p.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r01p.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep --no-steps > gpurun_out/ncu_launch_r01p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass --launch-skip 3 -c 3 -o gpurun_out/prof_r01p_full python tools/run_point.py 7 256 > gpurun_out/ncu_full_r01p.log 2>&1
tail -c 600 gpurun_out/bench_r01p.jsonl
