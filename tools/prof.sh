# usage: bash tools/prof.sh tag kernel-regex [count]
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 --launch-skip 3 -c ${3:-1} -o gpurun_out/prof_$1 python tools/run_point.py 7 256 > gpurun_out/prof_$1.log 2>&1
ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv > gpurun_out/prof_$1_src.csv 2>/dev/null
ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
tail -2 gpurun_out/prof_$1.log
