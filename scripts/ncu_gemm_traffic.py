"""Per-launch DRAM traffic of the K4 GEMM from an ncu --set full report (units-aware)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
m = int(sys.argv[3]) if len(sys.argv) > 3 else 32  # token rows of the captured launches (gemm_one.py m)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "%": 1}


def val(r, k):
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1)


names = ["qkv", "o", "gate_up", "down", "lm_head"]
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (24576, 4096), "down": (4096, 12288),
          "lm_head": (151936, 4096)}
per = {}
for i, n in enumerate(names):
    sub = rows[2 + 3 * i: 5 + 3 * i]
    dram = sum(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in sub) / 3
    t = sum(val(r, "gpu__time_duration.sum") for r in sub) / 3
    alg = shapes[n][0] * shapes[n][1] * 2 + m * shapes[n][1] * 2
    per[n] = {"time_us": t * 1e6, "dram_bytes": dram, "algorithmic_bytes": alg, "traffic_over_alg": dram / alg,
              "dram_GBps": dram / t / 1e9,
              "dram_pct_peak": sum(val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") for r in sub) / 3}
step_dram = sum(per[n]["dram_bytes"] * 36 for n in names[:4]) + per["lm_head"]["dram_bytes"]
step_alg = sum(per[n]["algorithmic_bytes"] * 36 for n in names[:4]) + per["lm_head"]["algorithmic_bytes"]
res = {"source": f"ncu --set full {rep} (scripts/gemm_one.py {m}; cold L2, serialized launches)", "m": m,
       "per_shape": per, "dram_bytes_per_launch": step_dram / 145, "algorithmic_bytes_per_launch": step_alg / 145,
       "traffic_over_algorithmic": step_dram / step_alg,
       "note": "per-launch average over one verify step: 36 x (qkv, o, gate_up, down) + lm_head"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
