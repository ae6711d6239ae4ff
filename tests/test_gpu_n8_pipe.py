"""The pipelined 8x8 kernel (expm8_pipe_kernel, MEXP_N8_VARIANT=12 dynamic
ticket / 15 static rounds) against the default kernel: the same arithmetic in
the same order, so e^A and the selection records must be bit-identical in
every rounding policy -- including non-finite matrices, an overflowing norm,
and a batch that is not a multiple of the four-matrix round.

The variant is read once per process, so each variant runs in a subprocess.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads
a = workloads.generate("cfg2", 0, 20003)          # odd: a partial last round
a[5, 2, 3] = np.nan
a[6, 0, 0] = -np.inf
a[7] = 1.7e308                                    # finite entries, the 1-norm overflows
a[11] *= 1e300                                    # a very large s
outs = []
for rounding in (mx.ROUND_REFERENCE, mx.ROUND_AUTO, mx.ROUND_FAST):
    for fam in (mx.Family.TaylorNew, mx.Family.TaylorPS):
        out, sel, st = mx.expm_batched_host(a, rounding=rounding, family=fam, raise_on_error=False)
        outs += [out.view(np.uint64), sel.view(np.uint8), np.array([st])]
np.savez(sys.argv[1], *outs)
"""


def run_variant(variant, path, **extra):
    env = dict(os.environ, MEXP_N8_VARIANT=str(variant), **extra)
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], check=True, env=env,
                   timeout=600)
    with np.load(path) as z:
        return [z[k] for k in z.files]


@pytest.mark.parametrize("variant,extra", [(12, {}), (15, {}), (12, {"MEXP_N8_STATIC_PCT": "50"})])
def test_pipelined_kernel_bitwise_equals_default(cuda, tmp_path, variant, extra):
    base = run_variant(0, str(tmp_path / "v0.npz"))
    got = run_variant(variant, str(tmp_path / f"v{variant}.npz"), **extra)
    assert len(base) == len(got) == 18
    for i, (b, g) in enumerate(zip(base, got)):
        assert np.array_equal(b, g), f"array {i} differs (variant {variant})"
    # the statuses of the planted matrices (first REFERENCE / TaylorNew call)
    import paper_1710_10989_b200 as mx
    sel = base[1].view(mx.SELECTION_DTYPE)
    assert sel["status"][5] == mx.ERR_NONFINITE and sel["status"][6] == mx.ERR_NONFINITE
    assert sel["status"][7] == mx.ERR_NORM_NONFINITE
    assert sel["status"][11] == mx.OK and sel["s"][11] > 900
