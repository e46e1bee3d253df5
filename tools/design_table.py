"""Markdown rows of DESIGN.md §0's measured table from profiles/r02_bench_*.json."""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"C2": "C2", "C3": "C3", "C4": "C4", "C5": "C5 (64 k-points cycled)",
         "C2NS": "C2NS (l_nonsph 6, not BASELINE)", "C2IND": "C2IND (indefinite T, not BASELINE)"}
NG = {"C5": "4967–5013"}
for c, label in NAMES.items():
    d = json.load(open(os.path.join(REPO, "profiles", f"r02_bench_{c}.json")))
    e, r, a = d["e2e"], d["roofline"], d["ab_gen"]
    x = a.get("expand_AB")
    gen = (f"{a['ms']:.3f} ms ({x['frac']:.2f}; {x['frac_of_write_ceiling']:.2f})" if x
           else f"{a['ms']:.3f} ms (per-atom path)")
    print(f"| {label} | {NG.get(c, d['config']['n_basis'])} | {d['config']['rows']} | "
          f"{d['ms_per_step']:.2f} | {d['value']:.1f} | {r['frac']:.3f} | "
          f"{e['ms_per_step']:.2f} / {e['single_call_ms']:.2f} / {e['dropin_ms']:.2f} | {gen} |")
