import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_11612_b200 as P
from paper_2303_11612_b200 import device
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
shapes = [(1000, 60, 50), (200, 15, 10)] if len(sys.argv) < 2 else [tuple(map(int, sys.argv[1].split("x")))]
for I, s, mu in shapes:
    c = torch.randn(I * s, dtype=torch.float64, device="cuda")
    device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
torch.cuda.synchronize()
print("ok")
