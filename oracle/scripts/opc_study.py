"""Operator complexity of the oracle hierarchy under the readings the paper leaves open (DESIGN.md §3,
c.8 tie-break and c.12 ω norm), against Table 1c.

TEST INFRASTRUCTURE (oracle only): calls nothing but oracle/.  Output: oracle/opc_study.json.

    python oracle/scripts/opc_study.py 48 3 [96 3 ...]      (k p pairs; one oracle setup per variant)
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

VARIANTS = {
    "canonical": dict(),                         # tie (i asc, j asc), ω from K_f
    "tie_larger_index": dict(tie_break=1),       # each vertex prefers its larger-index partner
    "tie_hashed": dict(tie_break=2),             # fixed pseudo-random tie order (seed 0)
    "tie_hashed_s1": dict(tie_break=3),          # ... seeds 1, 2: the spread over arbitrary tie orders
    "tie_hashed_s2": dict(tie_break=4),
    "omega_unfiltered": dict(omega_norm=1),      # ω = 4/(3‖D⁻¹K‖∞) of K itself (A.2's wording)
}


def run(k: int, p: int, names):
    K = oracle.assemble(3, p, k)
    out = {}
    for name in names:
        t0 = time.perf_counter()
        H = oracle.setup(K, oracle.OParams.for_degree(p, **VARIANTS[name]))
        out[name] = dict(N=[L.N for L in H.levels], nnz=[int(L.K.nnz) for L in H.levels],
                         opc=round(H.opc(), 4), omega=[L.omega for L in H.levels[:-1]],
                         setup_s=round(time.perf_counter() - t0, 1))
        print(k, p, name, json.dumps(out[name]), flush=True)
        del H
    return out


def main():
    args = [int(a) for a in sys.argv[1:] if not a.startswith("--")]
    names = [a[2:] for a in sys.argv[1:] if a.startswith("--")] or list(VARIANTS)
    path = os.path.join(ROOT, "oracle", "opc_study.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for k, p in zip(args[0::2], args[1::2]):
        r = run(k, p, names)
        res.setdefault(f"k{k}_p{p}", {}).update(r)
        with open(path, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
