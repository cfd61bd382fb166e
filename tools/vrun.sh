( timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 ) > gpurun_out/v_pytest.log
for i in 1 2; do for L in abl/a2base.so abl/v1.so abl/v2.so; do echo -n "$L "; PSWE_LIB_PATH=$L STEPS=10 CHUNKS=2048 bash tools/chunk_sweep.sh; done; done > gpurun_out/v_ab.log 2>&1
cat gpurun_out/v_pytest.log gpurun_out/v_ab.log
