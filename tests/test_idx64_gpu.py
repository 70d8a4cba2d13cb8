"""The 64-bit-offset kernels (taken when A or B has 2^31 or more nonzeros: the group
kernels' int64 row walker, the spilling block table + global recount for the top
symbolic bin, the ordered global-table heap tier) on inputs small enough to check:
SPGEMM_FORCE_IDX64=1 forces that path; the products must still equal the oracle
(bitwise: the 64-bit heap tier is the ordered one)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import numpy as np
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from oracle import oracle as O
from helpers import assert_matches_oracle, spill_pair
cases = [S.random_values(S.stencil3d_27pt(12), 1), S.random_values(S.rmat(12, 16, seed=5), 2),
         S.random_values(S.poisson2d_5pt(40), 3)]
for a in cases:
    out = sg.multiply(a, a)
    assert_matches_oracle(out.c, O.spgemm(a, a), bitwise=True)
a, b = spill_pair(20000, 200)
out = sg.multiply(a, b)
assert out.spilled_rows == 1
assert_matches_oracle(out.c, O.spgemm(a, b), bitwise=True)
a, b = spill_pair(6000, 60)
out = sg.multiply(S.random_values(a, 4), S.random_values(b, 5))
assert_matches_oracle(out.c, O.spgemm(S.random_values(a, 4), S.random_values(b, 5)), bitwise=True)
print("idx64 ok")
"""


def test_forced_64bit_offsets_match_oracle():
    env = dict(os.environ, SPGEMM_FORCE_IDX64="1")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "idx64 ok" in res.stdout, res.stdout[-2000:] + res.stderr[-3000:]
