"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv, subprocess, sys

KEEP = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size',
        'launch__block_size', 'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__inst_executed.avg.per_cycle_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'sm__cycles_elapsed.avg.per_second',
        'smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed',
        'smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed',
        'smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed',
        'derived__smsp__sass_thread_inst_executed_op_ffma_pred_on_x2',
        'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']


def main(rep, title, out):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    with open(out, 'w') as f:
        f.write(title + '\n')
        if 'Kernel Name' in hdr:
            f.write('kernel: ' + vals[hdr.index('Kernel Name')] + '\n')
        f.write('\n')
        for k in KEEP:
            if k in hdr:
                f.write(f"{k:75s} {vals[hdr.index(k)]} {units[hdr.index(k)]}\n")
        f.write("\nwarp stall reasons (per issued instruction):\n")
        for k in hdr:
            if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
                v = float(vals[hdr.index(k)])
                if v > 0.005:
                    name = k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')
                    f.write(f"  {name:28s} {v:.3f}\n")
    print(open(out).read())


if __name__ == '__main__':
    main(*sys.argv[1:4])
