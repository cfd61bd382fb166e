( timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 )
python tools/small_probe.py
bash tools/sweep_ab.sh abl/base.so abl/bsel.so abl/bsel_gc.so
