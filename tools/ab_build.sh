# A/B of two builds on one box (HEAD = $1, new = the in-tree library): bits of 13 evaluations,
# the C2 step timings alternated, then the GPU tests and the step configs of bench.py for both.
H=$(realpath $1)
set -x
PSWE_LIB_PATH=$H python tools/bits_check.py /tmp/bits_head.npz > gpurun_out/bits_head.log 2>&1
python tools/bits_check.py /tmp/bits_new.npz /tmp/bits_head.npz > gpurun_out/bits_new.log 2>&1
rm -f gpurun_out/sp_head.log gpurun_out/sp_new.log
for i in 1 2 3; do
  python tools/step_probe.py >> gpurun_out/sp_new.log 2>&1
  PSWE_LIB_PATH=$H python tools/step_probe.py >> gpurun_out/sp_head.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_early.log 2>&1
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_reference_checks.py -m gpu -q 2>&1 | tail -1 >> gpurun_out/pytest_gpu_early_repeat.log; done
python tools/bits_check.py /tmp/bits_new2.npz /tmp/bits_new.npz > gpurun_out/bits_repeat.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_early.jsonl 2> gpurun_out/bench_early.err
PSWE_LIB_PATH=$H timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_headlib.jsonl 2> gpurun_out/bench_headlib.err
cat gpurun_out/bits_new.log gpurun_out/bits_repeat.log gpurun_out/pytest_gpu_early_repeat.log; cat gpurun_out/sp_new.log gpurun_out/sp_head.log | cut -c1-90; tail -3 gpurun_out/pytest_gpu_early.log
