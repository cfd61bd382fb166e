# One measurement point on the GPU box: tests, bench (contract line), reference arm,
# ncu launch list and one ncu --set full capture of the passes at 512^2, M = 256.
# usage: bash tools/full_measure.sh TAG      (outputs in gpurun_out/*_TAG.*)
T=${1:?tag}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$T.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$T.jsonl 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep --no-steps > gpurun_out/plain_$T.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sweep --no-steps > gpurun_out/ncu_launch_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass --launch-skip 3 -c 3 -o gpurun_out/prof_${T}_full python tools/run_point.py 7 256 > gpurun_out/ncu_full_$T.log 2>&1
tail -c 600 gpurun_out/bench_$T.jsonl
tail -3 gpurun_out/pytest_gpu_$T.log
