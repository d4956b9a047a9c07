"""Time one streaming CGS2 call shape through the C ABI (tuning aid).

    SVDSC_KTIMING=1 python tools/probe_cgs2.py N C [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def main():
    N, c = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    H = S.Handle()
    ld = -(-N // 32) * 32
    Q = torch.zeros((c, ld), device="cuda", dtype=torch.float64)
    Qc, _ = torch.linalg.qr(torch.randn(N, c, device="cuda", dtype=torch.float64))
    Q[:, :N] = Qc.t()
    Qm = Q.t()[:N, :]
    w = torch.randn(N, device="cuda", dtype=torch.float64)
    os.environ["SVDSC_OPCGS_FUSED"] = "1t"
    S.cgs2(H, Qm, w.clone())
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        x = w.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.cgs2(H, Qm, x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    print(f"{os.environ.get('SVDSC_LIB_VARIANT', 'libsvdsc.so')} N={N} c={c} median {us:.1f} us "
          f"({3 * 8 * N * c / us / 1e3:.0f} GB/s over 3 sweeps of Q)", flush=True)
    H.close()  # svdsc_destroy prints the SVDSC_KTIMING phase counters


if __name__ == "__main__":
    main()
