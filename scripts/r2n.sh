set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct
LAYOUT_PROBE_QUICK=1 ncu --metrics $M --clock-control none -k regex:"assemble_numeric_kernel|barrier_stencil_kernel" --csv --log-file gpurun_out/r2n_layout_ncu.csv python scripts/layout_probe.py stack > gpurun_out/r2n_probe.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r2n_layout_ncu.csv")) if len(r) > 10]
h = rows[0]; ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault((r[idi], r[ki][:60]), {})[r[mi]] = r[vi]
for (i, k), m in per.items():
    print(i, k)
    for name, v in m.items():
        print("    %-60s %s" % (name, v))
PY
