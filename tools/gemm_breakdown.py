"""Per-shape breakdown of the GEMM DRAM traffic captured by tools/gemm_traffic.py
(ncu csv + shape dump): measured vs algorithmic bytes and time per product.

    python tools/gemm_breakdown.py gpurun_out/gemm_ncu.csv gpurun_out/gemm_shapes.csv
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
by, order = defaultdict(dict), []
for r in rows[1:]:
    i = r[h.index("ID")]
    if i not in by:
        order.append(i)
    by[i][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
shp = list(csv.DictReader(open(sys.argv[2])))
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, s in zip(order, shp):
    v = by[i]
    M, N, K, Z = (int(float(s[k])) for k in ("M", "N", "K", "batch"))
    if s["nsrc"] == "split":  # A [B | B2] and A2 B: two A operands, B and B2 once, C and C2
        ns = "split"
        alg = 4.0 * Z * (2 * M * K + N * K + M * N)
    elif s["nsrc"] == "twin":  # A B and A2 B + A B2: A, A2, B, B2 once, C and C2
        ns = "twin"
        alg = 4.0 * Z * (2 * M * K + 2 * N * K + 2 * M * N)
    else:
        ns = int(float(s["nsrc"]))
        alg = 4.0 * Z * (ns * (M * K + N * K) + M * N)
    a = agg[(M, N, K, Z, ns, s["a_mn"], s["b_mn"], s["causal"])]
    a[0] += 1
    a[1] += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
    a[2] += alg
    a[3] += v["gpu__time_duration.sum"]
print("M,N,K,batch,nsrc,a_mn,b_mn,kind | launches | measured GB | algorithmic GB | ratio | ms (ncu, serialised)")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(",".join(map(str, k)), "|", a[0], f"| {a[1] / 1e9:.2f} | {a[2] / 1e9:.2f} | {a[1] / a[2]:.2f} | {a[3] / 1e6:.2f}")
