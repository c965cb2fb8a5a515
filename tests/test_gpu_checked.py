"""The checked build (libamg_b200_checked.so: device-side invariant checks compiled in, AMG_CHECKS in
kernels.cuh) on small cases in a subprocess: every SELL-VI variant (plain, forced tail splits,
windowed) and the CSR cores run their solves with the window / value-index / split-ticket / push
checks armed; a violated invariant traps the kernel and fails the subprocess.  The results agree with
the product build and with the oracle.  (compute-sanitizer is closed on the B200 pool.)
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2511_21268_b200 as amg
from paper_2511_21268_b200 import _lib
import amg_inputs
out = dict(lib=os.path.basename(_lib.LIB_PATH))
for case, (dim, p, n), fmt in [("C1", (2, 2, 16), 0), ("C2", (3, 2, 32), 0), ("C2", (3, 2, 32), 6),
                               ("c12", (3, 3, 12), 6), ("c10p4", (3, 4, 10), 0)]:
    K, F = amg.iga_poisson(dim, p, n, rhs=2 if dim == 3 else 0)
    H = amg.Hierarchy(K, amg.params(p, format=fmt, krylov=1 if dim == 3 else 0, coarse_solver=1 if dim == 3 else 0))
    Fd = torch.from_numpy(F).cuda()
    u, it, rr, hist, st = H.solve(Fd, rtol=1e-8, maxit=100)
    r = torch.from_numpy(amg_inputs.uniform_pm1(K.shape[0], seed=3)).cuda()
    z = H.vcycle(r)
    torch.cuda.synchronize()
    out[f"{{case}}_{{fmt}}"] = dict(it=it, st=st, u=u.cpu().numpy()[::7].tolist(), z=z.cpu().numpy()[::7].tolist(),
                                   l0=H.op_config(0, 0)["layout"])
print(json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0, (env_extra, r.stdout[-2000:], r.stderr[-4000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module", autouse=True)
def _need():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(os.path.join(ROOT, "paper_2511_21268_b200", "libamg_b200_checked.so")):
        pytest.fail("checked build missing: python -m paper_2511_21268_b200.build --checked")


@pytest.mark.parametrize("variant", [{}, {"AMG_SELLVIW_SPLIT": "2"}, {"AMG_SELLVI_WIN": "0", "AMG_SELLVI_PARTS": "2"},
                                     {"AMG_SELLVI_WIN": "0"}])
def test_checked_build_matches_product(variant):
    chk = _run(dict(variant, AMG_LIB="checked"))
    prod = _run(dict(variant))
    assert chk["lib"] == "libamg_b200_checked.so" and prod["lib"] == "libamg_b200.so"
    for key, c in chk.items():
        if key == "lib":
            continue
        p = prod[key]
        assert c["st"] == 0 and c["it"] == p["it"] and c["l0"] == p["l0"], (key, c["it"], p["it"])
        for f in ("u", "z"):
            a, b = np.array(c[f]), np.array(p[f])
            assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max(), (key, f)
    if variant.get("AMG_SELLVI_WIN") != "0":
        assert chk["C2_6"]["l0"] == "sellviw"  # the windowed core ran with its checks armed
