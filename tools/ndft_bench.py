"""FP64-pipe throughput of the direct NDFT kernels (a14) at compute-bound sizes.

Times gs_ndft_forward / gs_ndft_adjoint on device tensors with CUDA events and
reports algorithmic TFLOP/s (8 real flops per complex multiply-add term,
M x prod(N) terms per transform) against the measured FP64 peak
(profiles/fp64_peak.json).  Usage: python tools/ndft_bench.py [reps]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1607_04091_b200 as gs  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dmma_tflops"]
    rng = np.random.default_rng(5)
    out = []
    for dim, N, M in [(1, [1024], 4096), (1, [8192], 65536), (2, [128, 128], 65536), (2, [256, 256], 262144)]:
        pts = torch.from_numpy(rng.uniform(-0.5, 0.4999, M * dim)).cuda()
        nm = int(np.prod(N))
        x = torch.randn(nm, dtype=torch.complex128, device="cuda")
        y = torch.randn(M, dtype=torch.complex128, device="cuda")
        res = {"dim": dim, "N": N, "M": M}
        for name, fn, arg in (("forward", gs.ndft_forward, x), ("adjoint", gs.ndft_adjoint, y)):
            fn(dim, N, pts, arg)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn(dim, N, pts, arg)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            tf = 8.0 * M * nm / (ms / 1e3) / 1e12
            res[name] = {"ms": round(ms, 4), "tflops": round(tf, 3), "frac_fp64_peak": round(tf / peak, 4)}
        out.append(res)
        print(json.dumps(res), flush=True)
    return out


if __name__ == "__main__":
    main()
