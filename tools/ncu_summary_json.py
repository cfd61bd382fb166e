"""Write profiles/ncu_summary_<tag>.json from an `ncu --page raw --csv` dump:
per-kernel DRAM bytes and fp64 thread-instruction / flop counts per launch
and per phase (bench.py reads these for `traffic` and the fp64 roofline)."""
import csv, json, sys

raw, out, phases = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {"note": f"ncu --set full --clock-control none (cold cache), tools/run_point.py 7 256 (512^2, M=256, "
               f"{phases}-phase chunks); dram__bytes_read.sum + dram__bytes_write.sum; fp64 thread instructions "
               "from smsp__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum.per_cycle_elapsed x "
               "smsp__cycles_elapsed.avg (flop counts dfma as 2)", "units": "bytes"}
for d in data:
    name = d[ix["Kernel Name"]].split("(")[0].split("<")[0].split()[-1].replace("pswe::", "")
    k = name.replace("_pair", "").replace("_kernel", "")
    val = lambda m: float(d[ix[m]]) * scale.get(units[ix[m]], 1)
    dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    cyc = float(d[ix["smsp__cycles_elapsed.avg"]])
    op = {o: float(d[ix[f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed"]]) for o in ("dadd", "dmul", "dfma")}
    res[k] = {"512": {"bytes_per_launch": dram, "phases_per_launch": phases, "bytes_per_phase": dram / phases,
                      "duration_us": float(d[ix["gpu__time_duration.sum"]]),
                      "dp_thread_instr_per_phase": sum(op.values()) * cyc / phases,
                      "dp_flop_per_phase": (op["dadd"] + op["dmul"] + 2 * op["dfma"]) * cyc / phases,
                      # pipe utilisation of this (serialised, cold-cache) launch
                      "fp64_pipe_frac": float(d[ix["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]]) / 100,
                      "smem_wavefront_frac": float(d[ix["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]]) / 100}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k.startswith("pass")}, indent=1))
