import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2303_11612_b200 as P
from paper_2303_11612_b200 import device
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
for I, s, mu in [(16, 4, 2), (64, 15, 10), (128, 15, 10), (200, 15, 10), (60, 60, 50), (120, 50, 40), (500, 30, 20), (1000, 60, 50)]:
    c = torch.randn(I * s, dtype=torch.float64, device="cuda")
    try:
        u = device.leading_left_singular_vectors(c, I, s, mu, ctx=ctx)
        U = u.view(mu, I).T.cpu().numpy()
        import numpy as np
        C = c.view(s, I).T.cpu().numpy()
        Uo = np.linalg.svd(C, full_matrices=False)[0][:, :mu]
        print(I, s, mu, "ok", np.abs(U.T @ U - np.eye(mu)).max(), np.linalg.norm(Uo - U @ (U.T @ Uo), 2))
    except Exception as e:
        print(I, s, mu, "ERR", e)
