"""mexp_expm_batched_host_multi: the host call sharded by matrix across GPUs
(SURVEY.md 8(e)), one host thread and copy pipeline per device. On a
one-GPU box the same device is listed several times: the shards then run one
after another on it, which exercises the split, the per-shard offsets of A,
e^A and the records, and the global first-error index -- the results must
equal the single-device call bit for bit."""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x).view(np.uint8)


@pytest.mark.parametrize("devices", [None, [0], [0, 0], [0, 0, 0]])
def test_multi_equals_single_cfg2(cuda, devices):
    a = workloads.generate("cfg2", 0, 30001)
    out1, sel1, st1 = mx.expm_batched_host(a)
    out2, sel2, st2, first = mx.expm_batched_host_multi(a, devices=devices)
    assert st1 == st2 == mx.OK and first == -1
    assert np.array_equal(bits(out1), bits(out2))
    assert np.array_equal(bits(sel1), bits(sel2))


@pytest.mark.parametrize("n,dtype", [(13, np.float64), (32, np.float32), (96, np.float64)])
def test_multi_shards_other_sizes(cuda, n, dtype):
    rng = np.random.default_rng(n)
    norms = 10.0 ** rng.uniform(-3, 2, 7)
    a = rng.standard_normal((7, n, n))
    a = (a * (norms / workloads.one_norm_batched(a))[:, None, None]).astype(dtype)
    acc = mx.Accuracy.Single if dtype == np.float32 else mx.Accuracy.Double
    out1, sel1, _ = mx.expm_batched_host(a, accuracy=acc)
    out2, sel2, st, _ = mx.expm_batched_host_multi(a, devices=[0, 0, 0], accuracy=acc)
    assert st == mx.OK
    assert np.array_equal(bits(out1), bits(out2)) and np.array_equal(bits(sel1), bits(sel2))


def test_multi_first_error_is_global(cuda):
    a = workloads.generate("cfg2", 0, 999)
    a[700, 2, 3] = np.nan   # in the third of three shards [666, 999)
    a[400, 0, 0] = np.inf   # in the second [333, 666)
    out, sel, st, first = mx.expm_batched_host_multi(a, devices=[0, 0, 0], raise_on_error=False)
    assert st == mx.ERR_NONFINITE and first == 400
    assert sel["status"][400] == mx.ERR_NONFINITE and sel["status"][700] == mx.ERR_NONFINITE
    assert np.isnan(out[400]).all() and np.isnan(out[700]).all()
    ok = sel["status"] == 0
    ref, rsel, _ = mx.expm_batched_host(a, raise_on_error=False)
    assert np.array_equal(bits(out[ok]), bits(ref[ok]))


def test_multi_rejects_bad_device(cuda):
    with pytest.raises(ValueError, match="invalid argument"):
        mx.expm_batched_host_multi(np.zeros((4, 8, 8)), devices=[0, 99])
    assert mx.device_count() >= 1
