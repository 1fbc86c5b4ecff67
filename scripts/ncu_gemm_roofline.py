"""Summarise an `ncu --set full -k regex:k_gemm` capture of scripts/roofline_shapes.py (one
launch per shape, in SHAPES order) into profiles/<name>_gemm_roofline_ncu.json: DRAM bytes
per launch (bench.py's roofline.traffic), duration, tensor-pipe activity, algorithmic bytes.

usage: python scripts/ncu_gemm_roofline.py gpurun_out/gemm.ncu-rep profiles/r02_gemm_roofline_ncu_<cfg>_B<b>.json \
           [--config gpt2-1.3b] [--B 2]
A split-K shape is two launches (the kAccF32 slices, then k_splitk_finalize): the
finalize row is folded into the preceding GEMM row (time and DRAM bytes summed)."""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, "scripts")
from roofline_shapes import shapes_for  # noqa: E402

rep, out = sys.argv[1], sys.argv[2]
opt = dict(zip(sys.argv[3::2], sys.argv[4::2]))
SHAPES = [s[:5] for s in shapes_for(opt.get("--config", "gpt2-1.3b"), int(opt.get("--B", 0)))]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def col(name):
    return hdr.index(name)


def val(r, name):
    i = col(name)
    v = float(r[i].replace(",", ""))
    u = units[i]
    return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
                "nsecond": 1e-3}.get(u, 1.0)


groups = []  # one entry per shape: its GEMM row (+ its finalize row)
for r in data:
    if "k_splitk_finalize" in r[col("Kernel Name")] and groups:
        groups[-1].append(r)
    else:
        groups.append([r])
launches = []
for (M, N, K, a, b), grp in zip(SHAPES, groups):
    r = grp[0]
    dram = sum(val(x, "dram__bytes_read.sum") + val(x, "dram__bytes_write.sum") for x in grp)
    us = sum(val(x, "gpu__time_duration.sum") for x in grp)
    out_b = M * N * (4 if (a and b) else 2)
    alg = (M * K + N * K) * 2 + out_b * (2 if (a and b) else 1)  # operands once + output (fp32 accumulate: r+w)
    launches.append({"shape": [M, N, K, a, b], "kernel": r[col("Kernel Name")][:60], "split_k": len(grp) > 1,
                     "us": round(us, 2),
                     "dram_bytes": dram, "algorithmic_bytes": alg, "tflops": round(2.0 * M * N * K / (us * 1e-6) / 1e12, 1),
                     "tensor_active_pct": float(r[col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")])
                     if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in hdr else None})
res = {"source": "ncu --set full --clock-control none -k regex:k_gemm (scripts/roofline_shapes.py), one launch per "
                 "shape, cold caches", "avg_dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) / len(launches),
       "launches": launches}
with open(out, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}))
