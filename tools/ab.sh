# A/B timing of two builds on one box: PSWE_LIB_PATH=$A / $B alternately.
# usage: bash tools/ab.sh libA.so libB.so [rounds]
A=$1; B=$2; R=${3:-3}
for i in $(seq $R); do
  for L in $A $B; do
    echo -n "$(basename $L) "; PSWE_LIB_PATH=$L STEPS=${STEPS:-10} CHUNKS=${CHUNKS:-2048} bash tools/chunk_sweep.sh
  done
done
