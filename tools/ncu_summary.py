"""Summarise an ncu --set full report into profiles/<name>.md (+ traffic.json entry).

    python tools/ncu_summary.py gpurun_out/prof_fused_r1.ncu-rep profiles/ncu_fused_r1.md [--traffic-kernel REGEX --workload config3]
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    args = sys.argv[3:]
    traffic_re = args[args.index("--traffic-kernel") + 1] if "--traffic-kernel" in args else None
    workload = args[args.index("--workload") + 1] if "--workload" in args else "config3"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary: `{rep.split('/')[-1]}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (gpurun);",
             "cold-cache, serialised replays -- compare shares and DRAM bytes, not absolute wall time.", ""]
    hdrs = ["#", "kernel"] + [lbl for _, lbl in METRICS]
    lines.append("| " + " | ".join(hdrs) + " |")
    lines.append("|" + "---|" * len(hdrs))
    traffic = []
    for k, d in enumerate(data):
        name = d[ix["Kernel Name"]]
        short = re.sub(r"\(.*", "", name).replace("void ", "").replace("(anonymous namespace)::", "")
        vals = []
        for m, _ in METRICS:
            v = d[ix[m]] if m in ix else "n/a"
            u = units[ix[m]] if m in ix else ""
            vals.append(f"{v} {u}".strip())
        lines.append("| " + " | ".join([str(k), short] + vals) + " |")
        if traffic_re and re.search(traffic_re, name):
            def gb(metric):
                v = float(d[ix[metric]])
                u = units[ix[metric]]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
            if wr > 0.05 * rd:  # update launches only (the prologue writes no H)
                traffic.append(rd + wr)
    stall = []
    for k, d in enumerate(data):
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), d[i])
              for h, i in ix.items() if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio") and d[i] not in ("", "n/a")]
        st.sort(key=lambda x: -float(x[1]))
        stall.append(f"- launch {k}: " + ", ".join(f"{a} {float(b):.2f}" for a, b in st[:6]))
    lines += ["", "Top warp stall reasons (per issue-active cycle):", ""] + stall
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        try:
            tj = json.load(open("profiles/traffic.json"))
        except Exception:
            tj = {}
        tj[workload] = {"dram_bytes_per_launch": sum(traffic) / len(traffic), "kernel_regex": traffic_re,
                        "source": out, "launches_averaged": len(traffic)}
        json.dump(tj, open("profiles/traffic.json", "w"), indent=1)


if __name__ == "__main__":
    main()
