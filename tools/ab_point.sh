# usage: bash tools/ab_point.sh "points" libs...   (bitwise check vs the first lib + mid_probe timings, two rounds)
pts=$1; shift
first=$1
PSWE_LIB_PATH=$first python tools/bits_check.py /tmp/bits_ref.npz > /dev/null 2>&1
for L in "$@"; do echo "== $(basename $L)"; PSWE_LIB_PATH=$L python tools/bits_check.py /tmp/bits_x.npz /tmp/bits_ref.npz 2>&1 | grep -vc bitwise; done
for i in 1 2; do for L in "$@"; do echo "== $(basename $L)"; PSWE_LIB_PATH=$L python tools/mid_probe.py $pts 2>&1 | tail -n +1; done; done
