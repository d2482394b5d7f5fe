# LSU wavefront breakdown of the streamed SpMV (shared vs global, loads vs stores, bank conflicts) on the bench matrix
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds_cmd_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_gds_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
ncu --metrics $M --clock-control none -k regex:"bsr_spmv_stream_kernel" -c 2 --csv --log-file gpurun_out/spmv_wavefronts.csv python scripts/pcg_phase_probe.py > gpurun_out/spmv_wavefronts.log 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/spmv_wavefronts.csv")) if len(r) > 10]
h = rows[0]; mi, vi, idi = h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
last = max(r[idi] for r in rows[1:])
for r in rows[1:]:
    if r[idi] == last:
        print("%-70s %s" % (r[mi], r[vi]))
PY
