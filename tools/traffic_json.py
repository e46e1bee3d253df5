"""Per-launch DRAM bytes of one bench step's contraction launches -> profiles/traffic_<cfg>.json.

    python tools/traffic_json.py gpurun_out/traffic_C2.csv C2 [merged] > profiles/traffic_C2.json
The last contract launches of the capture are one step on the template path: S, the per-type
W = L^H [A; B] application, H (joint form: H = W1^H W1 + W2^H W2); with `merged` (device-
resident builds, bench.py's `value`): the W application, then S and H as one launch.
"""
import collections
import csv
import json
import sys

sys.path.insert(0, ".")
path, cfg = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
hdr = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
h = rows[hdr]
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    assert d["Metric Unit"] in ("byte", "ns", "nsecond", "usecond", "msecond"), d["Metric Unit"]
    launch.setdefault(d["ID"], {"kernel": d["Kernel Name"][:60]})[d["Metric Name"]] = (
        float(d["Metric Value"]), d["Metric Unit"])
merged = len(sys.argv) > 3 and sys.argv[3] == "merged"
step = list(launch.values())[-2:] if merged else list(launch.values())[-3:]
names = ["apply_W", "contract_SH"] if merged else ["contract_S", "apply_W", "contract_H"]
from paper_1602_06589_b200 import configs  # noqa: E402

inst = configs.make_instance(cfg)
n = inst.spec.n_basis
r = int(sum(inst.spec.layout().block_heights))
op = 16 * r * n
alg = {"contract_S": (2 * op, 16 * n * n), "contract_H": (2 * op, 16 * n * n),
       "contract_SH": (4 * op, 32 * n * n)}
per = {}
for name, l in zip(names, step):
    rd, wr = l["dram__bytes_read.sum"][0], l["dram__bytes_write.sum"][0]
    e = {"kernel": l["kernel"], "read": int(rd), "write": int(wr),
         "time": l["gpu__time_duration.sum"]}
    if name in alg:
        e["algorithmic_read"], e["algorithmic_write"] = alg[name]
        e["read_over_algorithmic"] = round(rd / alg[name][0], 2)
    per[name] = e
total = sum(per[k]["read"] + per[k]["write"] for k in per if k.startswith("contract_"))
print(json.dumps({
    "source": f"{path}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "-k regex:contract --clock-control none, python bench.py --steps 1 --warmup 3 (last step)",
    "kernel": "contract_kernel (S + H triangular contractions" + (", one merged launch)" if merged else ")"),
    "dram_bytes_per_step": int(total),
    "per_launch": per,
    "note": "algorithmic_read = operand bytes read once (S: A*, UB*; H: W1, W2); "
            "algorithmic_write = both triangles of the mirrored N_G x N_G result",
}, indent=1))
