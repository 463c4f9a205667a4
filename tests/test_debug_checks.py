"""Device-side invariant checks (csrc/debug_checks.cuh) in place of
compute-sanitizer, which is closed on this GPU pool.

lib_debug.so is libqcb200 built with QCB_DEBUG_CHECKS=1 (`bash
tools/debug_checks.sh build`): every shared-memory access through the cell /
table / I/O helpers is bounds- and alignment-checked against the CTA's
dynamic shared memory, the dynamic shared memory is poisoned before the
prologue (a read-before-write then shows up as an oracle mismatch), and every
CTA checks that its chunk lies inside the batch.  `tools/debug_checks.sh run`
runs the whole GPU suite and tools/sanitize_cases.py against it (logs under
profiles/).  Here: the debug library decodes bit-exactly like the oracle, and
the negative control -- QCB_DEBUG_INJECT makes each decoder family touch the
word just past its dynamic shared memory -- is caught (the launch traps).
Skipped when lib_debug.so has not been built.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
DEBUG_LIB = ROOT / "paper_2306_12063_b200" / "lib_debug.so"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not DEBUG_LIB.exists(), reason="lib_debug.so not built (tools/debug_checks.sh build)")]

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2306_12063_b200 as P
from oracle import oracle as O
from tests._util import noisy_llrs
code, fixed, w = ("%s", %d, "%s"), %d, %d
mm = P.get_model_matrix(*code)
llr, _, _ = noisy_llrs(mm, w, 2.5, seed=5, fixed=bool(fixed))
cfg = P.DecoderConfig(max_iterations=4, early_termination=True,
                      arithmetic=P.Arithmetic.Fixed16 if fixed else P.Arithmetic.Float32)
hard, it, conv = P.decode_batch(mm, torch.from_numpy(llr).cuda(), cfg)
torch.cuda.synchronize()
oh, oi, oc = O.decode_batch(P.expand(mm), llr, 4, True)
assert np.array_equal(hard.cpu().numpy(), oh) and np.array_equal(it.cpu().numpy(), oi)
print("decoded ok")
'''

# register kernel (f32), pair kernel (int16, TMEM tiers), TMEM message kernel (f32
# degree 20, forced below via the scaled plan: 1152 R5/6 f32 takes the register kernel,
# so QCB_TMEM=1 is set for it), int16 Z = 24 with CTA barriers
CASES = [("wimax", 2304, "1/2", 0, 5), ("wifi", 1944, "5/6", 1, 5), ("wimax", 1152, "5/6", 0, 5),
         ("wimax", 576, "1/2", 1, 5)]


def _run(case, inject):
    std, n, rate, fixed, w = case
    env = dict(os.environ, QCB_LIB=str(DEBUG_LIB))
    env.pop("QCB_DEBUG_INJECT", None)
    if inject:
        env["QCB_DEBUG_INJECT"] = "1"
    if (n, rate, fixed) == (1152, "5/6", 0):
        env["QCB_TMEM"] = "1"
    return subprocess.run([sys.executable, "-c", SCRIPT % (std, n, rate, fixed, w)], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}-{c[2]}-{'i16' if c[3] else 'f32'}")
def test_debug_library_decodes_like_the_oracle(case):
    res = _run(case, inject=False)
    assert res.returncode == 0 and "decoded ok" in res.stdout, res.stdout + res.stderr


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}-{c[2]}-{'i16' if c[3] else 'f32'}")
def test_debug_checks_catch_an_out_of_bounds_shared_access(case):
    res = _run(case, inject=True)
    assert res.returncode != 0 and "decoded ok" not in res.stdout, res.stdout + res.stderr
    assert "qcb debug: shared access site 99" in res.stdout + res.stderr, res.stdout + res.stderr
