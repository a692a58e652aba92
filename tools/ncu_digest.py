"""Digest of one kernel in an ncu report: key raw metrics, stall reasons, and the SASS hot spots
(region breakdown by instruction index).  Usage: python tools/ncu_digest.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__cycles_active.avg",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]:>20s} {units[i]}")
st = [(float(vals[i] or 0), h) for i, h in enumerate(hdr)
      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
st.sort(reverse=True)
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v:.0f}" for v, h in st[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
isrc, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[iex] or 0) for r in data))
for i in sorted(sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:top]):
    r = data[i]
    s3 = sorted([(int(r[c] or 0), hdr[c][6:]) for c in stc], reverse=True)[:2]
    print(f"{i:5d} {r[isrc].strip()[:58]:58s} {int(r[iss] or 0):7d} {int(r[iex] or 0):11d} {s3}")
