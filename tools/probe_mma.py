"""Tensor-core summation probe (R10): runs tcgen05.mma kind::f16 (fp32 accumulate) through
ntbc_debug_mma on crafted fp16 inputs and saves A, B, C, D to an .npz for offline model fitting
(tools/fit_mma_model.py).  Measurement tool; not part of the product path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09543_b200 import ntbc  # noqa: E402


def rand_f16(rng, shape, lo, hi, p_zero=0.0, p_sub=0.0):
    mag = np.exp2(rng.uniform(lo, hi, shape)) * rng.choice([-1.0, 1.0], shape)
    x = mag.astype(np.float16)
    if p_sub:
        m = rng.random(shape) < p_sub
        x[m] = (rng.integers(1, 1024, m.sum()) * 2.0 ** -24 * rng.choice([-1, 1], m.sum())).astype(np.float16)
    if p_zero:
        x[rng.random(shape) < p_zero] = 0
    return x


def run(out_path, n_rounds=64, seed=0):
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    recs = {"A": [], "B": [], "C": [], "D": [], "K": [], "hasC": []}
    for rd in range(n_rounds):
        K = [16, 16, 32, 64][rd % 4]
        N = 16
        spread = [2, 6, 10, 14][(rd // 4) % 4]
        A = rand_f16(rng, (128, K), -spread, spread, p_zero=0.05, p_sub=0.02 if rd % 5 == 0 else 0.0)
        B = rand_f16(rng, (N, K), -spread, spread, p_zero=0.05)
        if rd % 7 == 3:  # cancellation: row pairs of opposite sign
            B[:, 1] = -B[:, 0]
            A[:, 1] = A[:, 0]
        hasC = rd % 2 == 1
        Cm = None
        if hasC:
            Cm = (rng.standard_normal((128, N)) * np.exp2(rng.uniform(-spread, spread, (128, N)))).astype(np.float32)
        At = torch.from_numpy(A).to(dev)
        Bt = torch.from_numpy(B).to(dev)
        Ct = torch.from_numpy(Cm).to(dev) if hasC else None
        D = ntbc.debug_mma(At, Bt, Ct, K, N).cpu().numpy()
        recs["A"].append(A); recs["B"].append(B)
        recs["C"].append(Cm if hasC else np.zeros((128, N), np.float32)); recs["D"].append(D)
        recs["K"].append(K); recs["hasC"].append(hasC)
    arrs = {"K": np.array(recs["K"]), "hasC": np.array(recs["hasC"]), "C": np.array(recs["C"]),
            "D": np.array(recs["D"])}
    for i, (a, b) in enumerate(zip(recs["A"], recs["B"])):
        arrs[f"A{i}"] = a
        arrs[f"B{i}"] = b
    np.savez_compressed(out_path, **arrs)
    # quick self-check: integer inputs must be exact for every model
    Ai = rng.integers(-8, 9, (128, 32)).astype(np.float16)
    Bi = rng.integers(-8, 9, (16, 32)).astype(np.float16)
    Di = ntbc.debug_mma(torch.from_numpy(Ai).to(dev), torch.from_numpy(Bi).to(dev), None, 32, 16).cpu().numpy()
    exact = Ai.astype(np.float64) @ Bi.astype(np.float64).T
    print("probe: integer MMA exact:", bool(np.array_equal(Di, exact)), "max err", float(np.abs(Di - exact).max()))
    return out_path


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    run(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mma_probe.npz")
