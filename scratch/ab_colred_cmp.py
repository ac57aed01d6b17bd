import torch
a, b = torch.load("gpurun_out/hv_scalar.pt"), torch.load("gpurun_out/hv_vec.pt")
print("bitwise equal:", torch.equal(a, b), "max abs diff", (a - b).abs().max().item(), "rel l2", ((a - b).norm() / a.norm()).item())
