"""Summarise the tcgen05 kernel captures of an ncu --set full report (one
file per captured launch index given): tensor-pipe activity, shared-memory
and DRAM traffic, occupancy, stall reasons."""
import csv, subprocess, sys

KEEP = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'launch__shared_mem_per_block_dynamic', 'sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed.avg.per_cycle_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__cycles_elapsed.avg.per_second']


def main(rep, title, out, idx):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    names = {h.split('.', 1)[1] if h.startswith(('TPC.', 'SM_C.')) else h: i for i, h in enumerate(hdr)}
    with open(out, 'w') as f:
        f.write(title + '\n')
        f.write(f"kernel: {vals[hdr.index('Kernel Name')]}\n\n")
        for k in KEEP:
            i = names.get(k, names.get('TriageCompute.' + k))
            if i is not None:
                f.write(f"{k:75s} {vals[i]} {units[i]}\n")
        f.write("\nwarp stall reasons (per issued instruction):\n")
        for k in hdr:
            if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
                v = float(vals[hdr.index(k)] or 0)
                if v > 0.005:
                    f.write(f"  {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:.3f}\n")


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]))
