import sys, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200._lib import lib, check
L = lib()
P = 124439808
def ev(f, it=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
s = torch.cuda.current_stream().cuda_stream
x = torch.randn(P, device="cuda"); y = torch.randn(P, device="cuda"); z = torch.randn(P, device="cuda")
plen = L.sd_partial_len(0, P, P)
part = torch.empty(128 * plen, dtype=torch.float64, device="cuda")
coef = torch.full((128,), 1e-3, dtype=torch.float64, device="cuda")
out = torch.empty(128, dtype=torch.float64, device="cuda")
vp = C.c_void_p
t = ev(lambda: check(L.sd_k_axpy_dot(vp(x.data_ptr()), vp(y.data_ptr()), vp(z.data_ptr()), vp(coef.data_ptr()), 0, P, P, 0, vp(part.data_ptr()), vp(s))))
print(f"axpy_dot(update+dot z): {t:.3f} ms  {16*P/t/1e6:.0f} GB/s")
t = ev(lambda: check(L.sd_k_axpy_dot(None, vp(y.data_ptr()), None, None, 0, P, P, 0, vp(part.data_ptr()), vp(s))))
print(f"self dot: {t:.3f} ms  {4*P/t/1e6:.0f} GB/s")
b = (C.c_uint64 * 1)(0); e = (C.c_uint64 * 1)(P)
for m in (1, 13, 50):
    t = ev(lambda: check(L.sd_k_combine(1, b, e, P, m, vp(part.data_ptr()), vp(out.data_ptr()), vp(s))))
    print(f"combine m={m}: {t:.3f} ms")
for j in (13, 30, 50, 100):
    Q = torch.randn(j, P, device="cuda")
    t = ev(lambda: check(L.sd_k_cgs(vp(Q.data_ptr()), P, j, vp(y.data_ptr()), None, 1, 0, P, P, 0, vp(part.data_ptr()), vp(s))), 3)
    print(f"cgs dots j={j}: {t:.3f} ms  {4*P*(j+1)/t/1e6:.0f} GB/s")
    t = ev(lambda: check(L.sd_k_cgs(vp(Q.data_ptr()), P, j, vp(y.data_ptr()), vp(coef.data_ptr()), 1, 0, P, P, 0, vp(part.data_ptr()), vp(s))), 3)
    print(f"cgs update+dots j={j}: {t:.3f} ms  {4*P*(2*j+3)/t/1e6:.0f} GB/s (2 passes)")
    t = ev(lambda: check(L.sd_k_cgs(vp(Q.data_ptr()), P, j, vp(y.data_ptr()), vp(coef.data_ptr()), 2, 0, P, P, 0, vp(part.data_ptr()), vp(s))), 3)
    print(f"cgs update+self j={j}: {t:.3f} ms  {4*P*(j+3)/t/1e6:.0f} GB/s")
    del Q
