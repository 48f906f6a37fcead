"""Table I reproduction on the GPU (SPEC cmd_scan / cmd_table).

For each order n, an equally spaced grid of M points on [0, z_nb) is
evaluated by the sm_100a kernel and compared, every F_m, against the
extended-precision restatement of the reference oracle (oracle/boys_quad.c,
pinned to refmath in test_quad_reference.py).  M defaults to 2^16
(SPEC.md:406 desk scale); BOYS_TABLE1_POINTS=1048576 gives the paper's
density.  With BOYS_TABLE1_REPORT=<path> the measured table is written there.
"""

import json
import os

import numpy as np
import pytest
import torch

import accuracy as A
from paper_2504_07637_b200 import boys, coeffs as C

pytestmark = pytest.mark.gpu

M = int(os.environ.get("BOYS_TABLE1_POINTS", 1 << 16))


def _scan(oracle, profile, dtype):
    ds = C.load_default(profile)
    rows = {}
    for n in ds.orders():
        z = ds.records[n].z
        x = (np.arange(M, dtype=np.float64) * (z / M)).astype(dtype)
        ref = oracle.reference(n, x.astype(np.float64), "ld")
        got = boys(n, torch.from_numpy(x).cuda(), layout="aos").cpu().numpy()
        bits = [A.bits(A.rel_err(got[:, m], ref[:, m], dtype)) for m in range(n + 1)]
        rows[n] = {"N": ds.records[n].N, "eps_bar_0": bits[0],
                   "eps_bar_nm1": bits[n - 1] if n > 0 else None, "eps_bar_n": bits[n],
                   "eps_exact": ds.records[n].exact_bits, "per_m": bits}
        for m, b in enumerate(bits):
            assert b >= A.bar(n, m, dtype), f"{profile} n={n} m={m}: {b:.2f} < {A.bar(n, m, dtype)}"
        assert bits[0] >= bits[n] - 1          # acceptance 7
    return rows


def test_table1_double_and_single(oracle):
    out = {"points": M, "double53": _scan(oracle, "double53", np.float64),
           "single24": _scan(oracle, "single24", np.float32)}
    path = os.environ.get("BOYS_TABLE1_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
