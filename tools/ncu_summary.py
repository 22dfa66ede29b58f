"""Summarise an ncu report: key throughput metrics + stall reasons + hottest SASS."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for w in want:
    if w in hdr:
        i = hdr.index(w); print(f"{w:70s} {vals[i]:>16s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in cols}
s = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{c[6:]} {v/s*100:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source")
T = sum(float(r[i_s] or 0) for r in data)
top = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for k in sorted(top):
    r = data[k]
    print(f"{k:5d} {float(r[i_s])/T*100:5.1f}%  {r[i_src][:80]}")
