"""Summarise an `ncu --set full -k regex:k_gemm` capture of scripts/roofline_shapes.py (one
launch per shape, in SHAPES order) into profiles/<name>_gemm_roofline_ncu.json: DRAM bytes
per launch (bench.py's roofline.traffic), duration, tensor-pipe activity, algorithmic bytes.

usage: python scripts/ncu_gemm_roofline.py gpurun_out/gemm12.ncu-rep profiles/r01m_gemm_roofline_ncu.json"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, "scripts")
from roofline_shapes import SHAPES  # noqa: E402

rep, out = sys.argv[1], sys.argv[2]
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


launches = []
for (M, N, K, a, b), r in zip(SHAPES, data):
    dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    us = val(r, "gpu__time_duration.sum")
    out_b = M * N * (4 if (a and b) else 2)
    alg = (M * K + N * K) * 2 + out_b * (2 if (a and b) else 1)  # operands once + output (fp32 accumulate: r+w)
    launches.append({"shape": [M, N, K, a, b], "kernel": r[col("Kernel Name")][:60], "us": round(us, 2),
                     "dram_bytes": dram, "algorithmic_bytes": alg, "tflops": round(2.0 * M * N * K / (us * 1e-6) / 1e12, 1),
                     "tensor_active_pct": float(r[col("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")])
                     if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in hdr else None})
res = {"source": "ncu --set full --clock-control none -k regex:k_gemm (scripts/roofline_shapes.py), one launch per "
                 "shape, cold caches", "avg_dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) / len(launches),
       "launches": launches}
with open(out, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}))
