"""Analysis (test infrastructure, not a test): can the assignment GEMM drop the W_lo pass?

VERDICT r01 item 4 proposed one bf16 pass (score_j = x . bf16(W_j)) with an exact rescore of the
rows whose best-vs-second gap is within the bf16 rounding bound.  This script measures, on one
synthetic Wan2.1-14B 720p head (the bench workload's generator, N = 75,600, d = 128) and the
oracle's own Alg. 1 trace, how many rows such a scheme would flag:

    eps_cs(i)     = ||x_i|| * max_j ||W_lo_j||          (Cauchy-Schwarz, rigorous)
    eps_abs(i)    = max_j sum_c |x_ic| |W_lo_jc|          (elementwise, rigorous)
    flag(i)       = best_hi(i) - second_hi(i) < 2 eps(i)
    wrong(i)      = argmax_j x_i . bf16(W_j) != argmax_j x_i . W_j   (what one pass alone gets wrong)

    python tests/analysis/bf16_single_pass.py [kq kk]   -> one line per Alg. 1 half-step
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import svoo  # noqa: E402
from synthetic import config_workload  # noqa: E402


def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.float32).to(torch.bfloat16).double().numpy()


def main():
    kq, kk = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (100, 500)
    w = config_workload("wan14b_720p", H=1)
    Q = w.q[0, 0].double().numpy()
    K = w.k[0, 0].double().numpy()
    r = svoo.cocluster(Q, K, kq, kk, 2)
    for t in r.trace:
        X = K if t["side"] == "k" else Q
        Ca, Cs = t["C_anchor"], t["C_self"]
        P = Cs @ Ca.T
        W = ((Ca.T @ Ca) @ Cs.T).T / np.maximum(np.linalg.norm(P, axis=1), 1e-300)[:, None]
        Wh = bf16(W)
        Wl = W - Wh
        s_ex, s_hi = X @ W.T, X @ Wh.T
        top = np.sort(s_hi, 1)
        gap = top[:, -1] - top[:, -2]
        eps_cs = np.linalg.norm(X, axis=1) * np.linalg.norm(Wl, axis=1).max()
        eps_abs = (np.abs(X) @ np.abs(Wl).T).max(1)
        wrong = s_hi.argmax(1) != s_ex.argmax(1)
        out = {"kq": kq, "kk": kk, "iter": t["it"] + 1, "side": t["side"], "wrong": round(float(wrong.mean()), 5)}
        for name, eps in (("cs", eps_cs), ("abs", eps_abs)):
            flag = gap < 2 * eps
            assert not (wrong & ~flag).any()
            out[f"flag_{name}"] = round(float(flag.mean()), 4)
        print(out, flush=True)


if __name__ == "__main__":
    main()
