"""Summarise an ncu report: key metrics, stall reasons, top stalled SASS lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.max.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "lts__t_sector_op_read_hit_rate.pct"]
for w in want:
    if w in hdr: print(f"  {w:70s} {vals[hdr.index(w)]} {rows[1][hdr.index(w)]}")
stalls = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
tot = sum(float(v or 0) for _, v in stalls)
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')} {float(v)/tot*100:.1f}" for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:10]))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr, data = rows[1], rows[2:]
ix = hdr.index("Instructions Executed"); iss = hdr.index("Warp Stall Sampling (All Samples)"); src = hdr.index("Source")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ts = sum(int(r[iss]) for r in data)
top = sorted(range(len(data)), key=lambda i: -int(data[i][iss]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for i in sorted(top):
    r = data[i]
    st = sorted(((int(r[c]), hdr[c]) for c in sc), reverse=True)[:2]
    print(f"{i:5d} {r[src][:58]:58s} {r[ix]:>9s} {int(r[iss])/ts*100:5.2f}% {st}")
