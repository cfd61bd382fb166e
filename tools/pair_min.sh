for m in 0 200 450 900; do echo "MIN=$m"; PSWE_PAIR_MIN_CTAS=$m python tools/small_probe.py; done
for m in 0 450 900; do echo -n "MIN=$m "; PSWE_PAIR_MIN_CTAS=$m bash tools/sweep_ab.sh paper_2103_07706_b200/lib/libpswe_b200.so; done
