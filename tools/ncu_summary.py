import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; units = r[1]; v = r[2] if len(r) > 2 else r[1]
want = sys.argv[2:] or ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
 'sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active',
 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
 'sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__inst_executed.sum',
 'sm__inst_executed.avg.per_cycle_active','sm__cycles_elapsed.avg.per_second','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','lts__t_bytes.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed']
for w in want:
    for i, k in enumerate(h):
        if k == w:
            print(f"{w:70s} {v[i]} {units[i]}")
