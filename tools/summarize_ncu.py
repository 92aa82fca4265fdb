"""Summarise an ncu report (run here, no GPU): key counters, stall reasons,
SASS hot spots.  Usage: python tools/summarize_ncu.py report.ncu-rep > out.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
print(f"# ncu summary of {rep.split('/')[-1]}")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(f"\n## kernel: {d.get('Kernel Name')}")
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__warps_eligible.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
              "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
              "sass__inst_executed_local_loads", "sass__inst_executed_local_stores"]:
        if k in d:
            print(f"{k:60s} {d[k]:>20s} {u.get(k, '')}")
    st = []
    for h, v in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(v), h))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("\nwarp stall samples:")
    for x, h in sorted(st, reverse=True)[:10]:
        print(f"  {100 * x / tot:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    h = srows[1]
    ie = h.index("Instructions Executed")
    data = [(r[1], int(r[ie] or 0)) for r in srows[2:] if len(r) > ie]
    tot = sum(x for _, x in data) or 1
    print(f"\nSASS: {len(data)} instructions in the kernel, {tot} executed (warp-level)")
    print("TMA / barrier evidence (executed counts):")
    for mn in ("UBLKCP", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "VOTE", "POPC", "LDS", "STS", "SHFL"):
        c = sum(x for s, x in data if mn in s)
        print(f"  {mn:16s} {c}")
