"""Mutation check of the oracle's pins.

Applies plausible one-line misreadings to a scratch copy of oracle/svoo.py and runs the CPU
oracle tests against each; every mutation must make at least one test fail.

    python scripts/mutate_oracle.py            # prints one line per mutation, exit 1 if one survives
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = [
    ("step B anchored on the old C_k", "rb = assign_step(Q, Ck_new, Cq)", "rb = assign_step(Q, Ck, Cq)"),
    ("step A anchor/self swapped", "ra = assign_step(K, Cq, Ck)", "ra = assign_step(K, Ck, Cq)"),
    ("pre-update centroids returned", "return CoclusterResult(Lq, Cq, Lk, Ck, trace)",
     "return CoclusterResult(Lq, trace[-1]['C_self'], Lk, trace[-2]['C_self'], trace)"),
    ("step B with a zeroed C_q^(i-1)", "rb = assign_step(Q, Ck_new, Cq)", "rb = assign_step(Q, Ck_new, 0 * Cq)"),
    ("n_rec rounded down", "n_rec = (int(c.sum()) + Kq_ne - 1) // Kq_ne", "n_rec = int(c.sum()) // Kq_ne"),
    ("n_rec over K_q instead of K_q'", "n_rec = (int(c.sum()) + Kq_ne - 1) // Kq_ne",
     "n_rec = (int(c.sum()) + Kq - 1) // Kq"),
    ("DENSITY branch on b > theta", "n = min(n_rec, n_b) if (1.0 - b) > th else max(n_rec, n_b)",
     "n = min(n_rec, n_b) if b > th else max(n_rec, n_b)"),
    ("gap on squared distances", "gap = (d2 - d1) / np.maximum(d2, 1e-300)",
     "gap = (d2 * d2 - d1 * d1) / np.maximum(d2 * d2, 1e-300)"),
    ("R4 side bit swapped", "(b * H + h) * 2 + side)", "(b * H + h) * 2 + (1 - side))"),
    ("R4 Floyd draw modulo j", "t = r % (j + 1)", "t = r % j if j else 0"),
    ("ties to the highest index", "labels = np.argmin(D, axis=1)     # first",
     "labels = D.shape[1] - 1 - np.argmin(D[:, ::-1], axis=1)     # first"),
    ("Norm skipped on Pbar", "Pbh = l2_normalize_rows(Pbar)", "Pbh = Pbar"),
    ("recall softmax without 1/sqrt(d)", "zs = A[a, o] / math.sqrt(d_head)", "zs = A[a, o]"),
    ("empty cluster reset to zero", "C = np.array(C_prev, dtype=np.float64, copy=True)",
     "C = np.zeros_like(np.asarray(C_prev, dtype=np.float64))"),
    ("kept not re-sorted ascending", "kept = np.stack([np.sort(o[:n]) for o in orders])",
     "kept = np.stack([o[:n] for o in orders])"),
    ("n_b without the -1e-3 guard", "n = math.ceil(float(r) * Kk - 1e-3)", "n = math.ceil(float(r) * Kk)"),
    ("attention scale sqrt(d) instead of 1/sqrt(d)", "scale = 1.0 / math.sqrt(d) if scale is None else scale",
     "scale = math.sqrt(d) if scale is None else scale"),
    ("attention over the query's own cluster label", "allowed = np.nonzero(np.isin(Lk, np.asarray(kept[a])))[0]",
     "allowed = np.nonzero(Lk == a)[0]"),
    ("counting sort scatter in reverse (unstable)", "    for i, c in enumerate(labels):\n        perm[pos[int(c)]] = i",
     "    for i, c in reversed(list(enumerate(labels))):\n        perm[pos[int(c)]] = i"),
    ("centroid mean over all tokens of the side", "C[j] = members.sum(axis=0) / members.shape[0]",
     "C[j] = members.sum(axis=0) / X.shape[0]"),
    ("n clamped to K_k instead of K_k'", "return int(min(max(n, 1), Kk_ne))", "return int(min(max(n, 1), Kk))"),
    ("Floyd inserts t on a collision", "chosen.add(j if t in chosen else t)", "chosen.add(t)"),
]


def main() -> int:
    src = open(os.path.join(ROOT, "oracle", "svoo.py")).read()
    survivors = 0
    for name, old, new in MUTATIONS:
        if src.count(old) < 1:
            print(f"[skip] {name}: pattern not found")
            survivors += 1
            continue
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("tests", "synthetic"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("__pycache__"))
            os.makedirs(os.path.join(tmp, "oracle"))
            open(os.path.join(tmp, "oracle", "__init__.py"), "w").close()
            open(os.path.join(tmp, "oracle", "svoo.py"), "w").write(src.replace(old, new, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "tests/test_oracle.py", "tests/test_oracle_pins.py"],
                               cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            survivors += not killed
            last = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
            print(f"[{'killed' if killed else 'SURVIVED'}] {name}" + (f"  <- {last[0][7:]}" if last else ""))
    print(f"{len(MUTATIONS) - survivors}/{len(MUTATIONS)} mutations killed")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
