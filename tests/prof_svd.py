# profiling helper (not collected by pytest): one device SVD of a p x p arrow matrix
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_18966_b200 import svdsc as S
p = int(sys.argv[1]) if len(sys.argv) > 1 else 150
rng = np.random.default_rng(p)
k = p // 3
T = np.zeros((p, p))
T[np.arange(k), np.arange(k)] = np.sort(rng.uniform(1, 3, k))[::-1]
T[:k, k] = rng.uniform(-0.1, 0.1, k)
B = np.diag(rng.uniform(0.5, 2, p - k)) + np.diag(rng.uniform(0.1, 1, p - k - 1), 1)
T[k:, k:] = B
H = S.Handle()
Td = S.colmajor(p, p)
Td.copy_(torch.from_numpy(np.asfortranarray(T)).cuda())
for _ in range(2):
    U, s, V, sw = S.small_svd(H, Td)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
U, s, V, sw = S.small_svd(H, Td)
e1.record()
torch.cuda.synchronize()
print(f"p={p} sweeps={sw} ms={e0.elapsed_time(e1):.3f}")
