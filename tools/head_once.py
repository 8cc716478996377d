import sys, torch
sys.path.insert(0, ".")
from paper_2503_06545_b200 import device as D
torch.manual_seed(0)
a = torch.randn(8192, 1152, device="cuda")
w = torch.randn(1152, 1152, device="cuda") / 1152 ** 0.5
hw = D.HeadWeights(w)
out = torch.empty(8192, 1152, device="cuda")
D.head_gemm(a, hw, out=out)
torch.cuda.synchronize()
