"""One cfg4-shaped core contraction (X x_0 Q^T, X 1000^3, Q 1000 x 50) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_11612_b200 as P  # noqa: E402
from paper_2303_11612_b200 import device  # noqa: E402

ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
dims = [1000, 1000, 1000]
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
m = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x = torch.randn(10 ** 9, dtype=torch.float64, device="cuda")
b = torch.randn(m, 1000, dtype=torch.float64, device="cuda")
for _ in range(2):
    y, _ = device.mode_n_product(x, dims, mode, b, ctx=ctx)
torch.cuda.synchronize()
print("ok", y.shape)
