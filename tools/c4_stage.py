"""Per-GPU work of the C4 pipeline (Llama-2-7B shape, 8 stages, 1 x 1024-token
micro-batches) measured stage by stage on one B200: each stage runs its full
1F1B compute sequence for M micro-batches with synthetic boundary inputs
(the messages NCCL would deliver), timed with CUDA events."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_2505_11564_b200 import gpt
cfg = dict(gpt.LLAMA2_7B)
S_, M, B, SEQ = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 8, 1, 1024
ranges = gpt.pipeline_layers(cfg["n_layer"], S_)
out = {"config": "C4 Llama-2-7B, 8 stages, micro-batch 1x1024, M=%d" % M, "stages": []}
Td = B * SEQ * cfg["d"]
for s in (0, 4, 7):
    l0, l1 = ranges[s]
    b, e = gpt.stage_params(cfg, l0, l1)
    theta = torch.empty(e - b, device="cuda").normal_(0, 0.02)
    ns = min(M, S_ - s)
    st = gpt.GptStage(cfg, B, SEQ, M, l0, l1, theta, n_sets=ns)
    v = torch.randn(e - b, device="cuda") * 1e-3
    hv = torch.empty_like(v)
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
    out["stages"].append({"stage": s, "layers": [l0, l1], "params": e - b, "n_sets": ns,
                          "workspace_gb": st.workspace.numel() / 1e9, "ms_per_hvp": ms,
                          "max_mem_gb": torch.cuda.max_memory_allocated() / 1e9})
    print(out["stages"][-1], flush=True)
    del st, theta, v, hv
    torch.cuda.empty_cache(); torch.cuda.reset_peak_memory_stats()
worst = max(x["ms_per_hvp"] for x in out["stages"])
out["pipelined_hvp_ms_estimate"] = worst / M * (M + S_ - 1)
print(json.dumps(out))
