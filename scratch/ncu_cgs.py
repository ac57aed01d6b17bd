import sys, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_2505_11564_b200 as sd
from paper_2505_11564_b200._lib import lib, check
L = lib()
P = 124439808
j = int(sys.argv[1]) if len(sys.argv) > 1 else 50
vp = C.c_void_p
Q = torch.randn(j, P, device="cuda") / 1e4
y = torch.randn(P, device="cuda")
coef = torch.randn(j, dtype=torch.float64, device="cuda") * 1e-3
part = torch.zeros(j * (P // 1024 + 2), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
check(L.sd_k_cgs(vp(Q.data_ptr()), P, j, vp(y.data_ptr()), vp(coef.data_ptr()), 1, 0, P, P, 0, vp(part.data_ptr()), vp(s)))
torch.cuda.synchronize()
print("ok")
