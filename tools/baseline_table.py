"""BASELINE.md section 4 results table from a bench JSON line.
Usage: python tools/baseline_table.py profiles/r2_bench_line.json"""
import json
import sys

d = json.load(open(sys.argv[1]))
peak = d["roofline"]["peak"]


def f3(xs):
    return " / ".join(f"{x:.3f}" for x in xs) if xs else ""


def row(cfg, strat, shape, children_s, alg_gbs, lane, full="", base=""):
    pct = f"{100 * alg_gbs / peak:.1f} %" if alg_gbs else "—"
    gbs = f"{alg_gbs:.0f}" if alg_gbs else "—"
    print(f"| {cfg} | {strat} | {shape} | 1 | {children_s / 1e9:.1f} G | {gbs} | {pct} | {lane} | {full} | {base} |")


print(f"| Config | Strategy | L / shape | GPUs | children/s | alg. GB/s | % of {peak} | lane fraction per node | "
      "full-ensemble rate per node | oracle 1-thread / all-core (cores) |")
print("|---|---|---|---|---|---|---|---|---|---|")
occ = d["occupancy"]
cb = d["cpu_baseline"]
base = (f"{cb['brute_1thread']['value'] / 1e6:.0f}M fold, {cb['interp_1thread']['value'] / 1e6:.0f}M interp / "
        f"{cb['value'] / 1e6:.0f}M ({cb['cores']})")
row("configs[1] sweep (headline)", d["config"]["strategy"], "fixed L=4096, 2^29", d["value"], d["roofline"]["achieved"],
    f3([o["lane_fraction"] for o in occ]), f3([o["full_rate"] for o in occ]), base)
for s in d["sweep"]:
    name = "configs[1] sweep" + (" unfused" if s.get("unfused") else "") + (" f32" if s.get("dtype") == "f32" else "")
    strat = s["strategy"] + (f" ({s['kernel']} kernel)" if s.get("kernel") and s["strategy"] == "signal" else "")
    shape = f"{s.get('dist', 'fixed')} L={s['L']}"
    row(name, strat, shape, s["items_per_s"], s["hbm_frac"] * peak, f3(s["lane_fraction"]), f3(s.get("full_rate", [])))
names = {"graph": "configs[2] R-MAT 24", "text": "configs[3] text 4 GiB", "zipf": "configs[4] Zipf 2^30 (1 GPU)"}
for c in d.get("configs", []):
    if c["workload"] == "taxi":
        row("taxi (f1/f3)", c["strategy"], "2^28 bytes, 220K lines", c["items_per_s"], 0, f3(c["lane_fraction"]),
            f3(c.get("full_rate", [])))
    else:
        row(names[c["workload"]], c["strategy"], "", c["items_per_s"], c["hbm_frac"] * peak, f3(c["lane_fraction"]))
