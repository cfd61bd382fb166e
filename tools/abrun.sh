# usage: bash tools/abrun.sh tag libs...   (A/B timing of builds + gpu tests of the in-tree build)
tag=$1; shift
( [ -n "$NOTEST" ] || timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 ) > gpurun_out/ab_${tag}_pytest.log
for i in 1 2 3; do for L in "$@"; do
  echo -n "$(basename $L) "; PSWE_LIB_PATH=$L STEPS=10 CHUNKS=2048 bash tools/chunk_sweep.sh
done; done > gpurun_out/ab_${tag}.log 2>&1
cat gpurun_out/ab_${tag}_pytest.log gpurun_out/ab_${tag}.log
