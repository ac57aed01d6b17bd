"""BASELINE C5 (R1-Distill-Llama-70B shape, bf16 weights, fp32 Lanczos) per-GPU
footprint and work on one B200: stage 4 of an 8-stage pipeline (10 layers,
8.56 B parameters) with the lean engine (bf16-valued weights, layer
recomputation, on-chip probe residuals) AND the three fp32 Lanczos vectors of
the 3-term recurrence resident, running its 1F1B compute for M micro-batches
with synthetic boundary messages."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
SEQ = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
S_, s = 8, int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = dict(gpt.LLAMA_70B, bf16_weights=1)
l0, l1 = gpt.pipeline_layers(cfg["n_layer"], S_)[s]
b, e = gpt.stage_params(cfg, l0, l1)
P = e - b
theta = torch.empty(P, device="cuda")
CH = 1 << 28
for i in range(0, P, CH):  # chunked: no full-size temporaries
    theta[i:i + CH].normal_(0, 0.02)
    theta[i:i + CH] = theta[i:i + CH].bfloat16().float()
lanczos = [torch.empty(P, device="cuda") for _ in range(3)]  # q_{k-1}, q_k, r of the 3-term recurrence
v, hv = lanczos[1].normal_(0, 1e-3), lanczos[2]
st = gpt.GptStage(cfg, 1, SEQ, M, l0, l1, theta, n_sets=min(M, S_ - s), recompute=True, probe_residual=False)
Td = SEQ * cfg["d"]
xin = [torch.randn(Td, device="cuda") for _ in range(2)]
gin = [torch.randn(Td, device="cuda") * 1e-4 for _ in range(2)]
ops = [(k, m) for k, m in gpt.pipeline_schedule(S_, s, M) if k in (gpt.PIPE_F, gpt.PIPE_B)]


def run():
    st.begin_pass(v, hv)
    for k, m in ops:
        if k == gpt.PIPE_F:
            st.forward(m, *(xin if s > 0 else (None, None)))
        else:
            st.backward(m, *(gin if s < S_ - 1 else (None, None)))


run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
free, total = torch.cuda.mem_get_info()
out = {"config": "C5 R1-Distill-Llama-70B shape, 8 stages, stage %d (layers %d-%d), micro-batch 1x%d, M=%d" % (s, l0, l1, SEQ, M),
       "stage_params": P, "workspace_gb": st.workspace.numel() / 1e9, "lanczos_vectors_gb": 3 * P * 4 / 1e9,
       "theta_gb": P * 4 / 1e9, "device_used_gb": (total - free) / 1e9, "device_total_gb": total / 1e9,
       "ms_per_pass": ms, "ms_per_microbatch": ms / M,
       "finite": all(bool(torch.isfinite(hv[i:i + CH]).all()) for i in range(0, P, CH))}
print(json.dumps(out))
