"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per
launch) into a per-kernel markdown table and the GEMM traffic JSON."""
import csv, collections, json, sys
src, md_out, js_out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per, names = collections.defaultdict(dict), {}
for r in rows:
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    names[r[idi]] = r[ki].split("(")[0].replace("void ", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot += m.get("gpu__time_duration.sum", 0.0)
lines = [f"# Launch list summary ({src.split('/')[-1]})", "",
         f"{len(per)} launches, {tot / 1e3:.1f} ms summed kernel time (ncu-serialised, cold caches).", "",
         "DRAM GB/s = that kernel's DRAM bytes / its summed duration; % of the measured 6536.4 GB/s "
         "copy peak (MEASURED_PEAKS.json). For the HBM-bound kernels (Lanczos recurrence and reorth, "
         "elementwise R-op, softmax, CE) this is the roofline fraction; the GEMMs are tensor-bound.", "",
         "| kernel | launches | ms | share | DRAM GB | DRAM GB/s | % HBM peak |", "|---|---|---|---|---|---|---|"]
for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = b / (t * 1e-6) / 1e9 if t else 0.0
    lines.append(f"| `{k}` | {c} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {b / 1e9:.2f} | {gbs:.0f} | "
                 f"{100 * gbs / 6536.4:.0f}% |")
open(md_out, "w").write("\n".join(lines) + "\n")
g = [(c, t, b) for k, (c, t, b) in agg.items() if "k_gemm" in k]
n, t, b = sum(x[0] for x in g), sum(x[1] for x in g), sum(x[2] for x in g)
json.dump({"kernel": "k_gemm_pair / k_gemm_tf32 (3xTF32 tcgen05), all GEMM launches of one Lanczos step",
           "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none (launch list {src.split('/')[-1]})",
           "launches": n, "bytes_per_launch": b / n, "dram_bytes_total": b, "gemm_ms_serialised": t / 1e3,
           "gemm_share_of_step_serialised": t / tot}, open(js_out, "w"), indent=1)
print(open(md_out).read()[:1500])
