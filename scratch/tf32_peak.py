"""cuBLAS TF32 (and bf16 for reference) dense GEMM throughput on this B200:
burst (20 iterations) and sustained (~8 s loop), 8192^3."""
import time, torch, json, subprocess
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
out = {}
for name, dt in (("tf32", torch.float32), ("bf16", torch.bfloat16)):
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(5): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): a @ b
    e1.record(); torch.cuda.synchronize()
    burst = 2 * n**3 * 20 / (e0.elapsed_time(e1) / 1e3) / 1e12
    t0 = time.time(); it = 0
    e0.record()
    while time.time() - t0 < 8:
        for _ in range(20): a @ b
        it += 20
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    sus = 2 * n**3 * it / (e0.elapsed_time(e1) / 1e3) / 1e12
    out[name] = {"burst_tflops": burst, "sustained_tflops": sus}
    print(name, out[name], flush=True)
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
out["clocks_after"] = clk
print(json.dumps(out))
