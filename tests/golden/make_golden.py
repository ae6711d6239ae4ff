"""Generate tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the oracle restatement and the GPU path on the GPU box,
where /root/reference is absent. Inputs are built from the reference's own
known-answer tests (proj/tests/test_expm.cpp, test_dense_matrix.cpp,
cli_smoke.sh) plus seeded cases that cover every degree m in {1,2,4,8,12,18},
the theta boundaries and s up to 7, at several n.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

THETA = {1: [2.22e-16, 2.58e-8, 3.40e-4, 4.99e-2, 2.99e-1, 1.09],
         0: [1.19e-7, 5.98e-4, 5.12e-2, 5.80e-1, 1.46, 3.01]}
# Family::TaylorPS (theta_tables.cpp:53-59)
THETA_PS = {1: [2.22e-16, 2.58e-8, 3.40e-4, 9.07e-3, 8.96e-2, 7.80e-1],
            0: [1.19e-7, 5.98e-4, 5.12e-2, 2.50e-1, 7.80e-1, 2.48]}


def select_cases():
    norms = [0.0, 1.0, 10.0, 2.18, 0.4, 1e-300, 5e-324, 1e300, 1.7976931348623157e308,
             np.pi, 100.0, 1e-4, 1e2, 333.0, 1.2, 3.7, 9.0, 40.0]
    for acc in (0, 1):
        for t in THETA[acc]:
            norms += [t, np.nextafter(t, 0.0), np.nextafter(t, np.inf)]
            for k in range(1, 12):
                v = np.ldexp(t, k)
                norms += [v, np.nextafter(v, 0.0), np.nextafter(v, np.inf)]
    return np.array(sorted(set(norms)), np.float64)


def random_with_norm(rng, n, norm):
    m = rng.uniform(-1.0, 1.0, size=(n, n))
    return m * (norm / workloads.one_norm_batched(m[None])[0])


def expm_cases():
    rng = np.random.default_rng(20171030)
    cases = []  # (name, matrix)
    pi = 3.141592653589793
    cases.append(("zero4", np.zeros((4, 4))))
    cases.append(("rot_pi", np.array([[0.0, pi], [-pi, 0.0]])))
    cases.append(("rot_1rad", np.array([[0.0, 1.0], [-1.0, 0.0]])))
    cases.append(("norm_kat", np.array([[1.0, -2.0], [3.0, 4.0]])))
    cases.append(("shear", np.array([[1.0, 1.0], [0.0, 1.0]])))
    cases.append(("ident3x2", 2.0 * np.eye(3)))
    cases.append(("one_by_one", np.array([[0.5]])))
    cases.append(("nilpotent", np.diag(np.ones(7), 1)))
    # every degree, and s from 1 to 7 (double table), at several n
    norms = [1e-17, 2.22e-16, 1e-9, 2.58e-8, 1e-5, 3.40e-4, 0.01, 4.99e-2, 0.1, 2.99e-1,
             0.5, 1.09, 2.18, 3.0, 10.0, 30.0, 50.0, 100.0]
    for n in (1, 2, 3, 5, 8, 13, 16, 24, 32, 40, 64):
        for norm in (norms if n <= 24 else [1e-9, 0.1, 1.09, 10.0, 100.0]):
            cases.append((f"n{n}_norm{norm:g}", random_with_norm(rng, n, norm)))
    return cases


def taylor_ps(ref):
    """tests/golden/taylor_ps.npz: Family::TaylorPS selection at every theta
    boundary and expm cases covering degrees {1, 2, 4, 6, 9, 16}, s up to 8."""
    norms = [0.0, 1.0, 10.0, 0.5, 1e-300, 1e300, 3.0, 100.0]
    for acc in (0, 1):
        for t in THETA_PS[acc]:
            norms += [t, np.nextafter(t, 0.0), np.nextafter(t, np.inf)]
            for k in range(1, 12):
                v = np.ldexp(t, k)
                norms += [v, np.nextafter(v, 0.0), np.nextafter(v, np.inf)]
    norms = np.array(sorted(set(norms)), np.float64)
    arrays = {"norms": norms}
    for acc in (0, 1):
        sel = np.array([ref.select(float(v), acc, 1) for v in norms], np.int32)
        arrays[f"status_acc{acc}"], arrays[f"degree_acc{acc}"], arrays[f"s_acc{acc}"] = sel.T
    rng = np.random.default_rng(19)
    case_norms = [1e-17, 1e-9, 1e-5, 3.40e-4, 5e-3, 9.07e-3, 0.05, 8.96e-2, 0.2, 0.78, 1.5,
                  2.48, 6.0, 40.0, 150.0]
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        a = np.stack([random_with_norm(rng, n, v) for v in case_norms])
        arrays[f"n{n}_a"] = a
        for acc in (0, 1):
            r = ref.expm_batch(a, accuracy=acc, family=1)
            arrays[f"n{n}_acc{acc}_out"] = r.out
            arrays[f"n{n}_acc{acc}_meta"] = np.stack(
                [r.degree, r.s, r.cost_thirds, r.status], axis=1).astype(np.int64)
            arrays[f"n{n}_acc{acc}_norm"] = r.norm_in
    np.savez_compressed(os.path.join(OUT, "taylor_ps.npz"), **arrays)
    print(f"wrote taylor_ps.npz: {len(norms)} select norms, {len(case_norms)} cases per n")


def pade(ref):
    """tests/golden/pade.npz: Family::PadeDiagonal selection at every theta
    boundary, pade_coeffs(1..13), and expm cases covering every order 2..26
    (both tables) with s up to 7."""
    theta = {1: [3.65e-8, 5.32e-4, 1.50e-2, 8.54e-2, 2.54e-1, 5.41e-1, 9.50e-1, 1.47, 2.10,
                 2.81, 3.60, 4.46, 5.37],
             0: [8.46e-4, 8.09e-2, 4.26e-1, 1.05, 1.88, 2.85, 3.93, 5.06, 6.25, 7.47, 8.71,
                 9.97, 11.2]}
    norms = [0.0, 1.0, 10.0, 0.5, 1e-300, 1e300, 3.0, 100.0]
    for acc in (0, 1):
        for t in theta[acc]:
            norms += [t, np.nextafter(t, 0.0), np.nextafter(t, np.inf)]
            for k in range(1, 8):
                v = np.ldexp(t, k)
                norms += [v, np.nextafter(v, 0.0), np.nextafter(v, np.inf)]
    norms = np.array(sorted(set(norms)), np.float64)
    arrays = {"norms": norms}
    for acc in (0, 1):
        sel = np.array([ref.select(float(v), acc, 2) for v in norms], np.int32)
        arrays[f"status_acc{acc}"], arrays[f"degree_acc{acc}"], arrays[f"s_acc{acc}"] = sel.T
    arrays["coeffs"] = np.stack([np.pad(ref.pade_coeffs(m), (0, 13 - m)) for m in range(1, 14)])
    rng = np.random.default_rng(26)
    case_norms = sorted(set(theta[1] + [1e-9, 4.0, 20.0, 300.0] +
                            [0.9 * t for t in theta[0]] + [0.9 * t for t in theta[1]]))
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        # every order of the double table (and s up to 6) at the large sizes
        nv = case_norms if n <= 16 else [0.9 * t for t in theta[1]] + [20.0, 300.0]
        a = np.stack([random_with_norm(rng, n, v) for v in nv])
        arrays[f"n{n}_a"] = a
        for acc in (0, 1):
            r = ref.expm_batch(a, accuracy=acc, family=2)
            arrays[f"n{n}_acc{acc}_out"] = r.out
            arrays[f"n{n}_acc{acc}_meta"] = np.stack(
                [r.degree, r.s, r.cost_thirds, r.status], axis=1).astype(np.int64)
            arrays[f"n{n}_acc{acc}_norm"] = r.norm_in
    np.savez_compressed(os.path.join(OUT, "pade.npz"), **arrays)
    print(f"wrote pade.npz: {len(norms)} select norms, {len(case_norms)} cases per n")


def main():
    ref = Reference()
    if "--only-ps" in sys.argv:
        taylor_ps(ref)
        return
    if "--only-pade" in sys.argv:
        pade(ref)
        return
    taylor_ps(ref)
    pade(ref)
    # selection
    norms = select_cases()
    sel = {}
    for acc in (0, 1):
        deg = np.zeros(len(norms), np.int32)
        s = np.zeros(len(norms), np.int32)
        st = np.zeros(len(norms), np.int32)
        for i, v in enumerate(norms):
            st[i], deg[i], s[i] = ref.select(float(v), acc)
        sel[f"degree_acc{acc}"] = deg
        sel[f"s_acc{acc}"] = s
        sel[f"status_acc{acc}"] = st
    np.savez_compressed(os.path.join(OUT, "select.npz"), norms=norms, **sel)

    # expm cases, grouped by n, both accuracy tables
    cases = expm_cases()
    arrays = {}
    names = []
    for idx, (name, a) in enumerate(cases):
        for acc in (1, 0):
            r = ref.expm_batch(a[None].astype(np.float64), accuracy=acc)
            key = f"c{idx}_acc{acc}"
            arrays[key + "_a"] = a.astype(np.float64)
            arrays[key + "_out"] = r.out[0]
            arrays[key + "_meta"] = np.array([r.degree[0], r.s[0], r.cost_thirds[0], r.status[0]],
                                             np.int64)
            arrays[key + "_norm"] = np.array([r.norm_in[0]])
            names.append(f"{key}:{name}")
    arrays["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "expm_cases.npz"), **arrays)

    # first 512 matrices of cfg2 and 64 of cfg3 (fp32 storage, double reference)
    a2 = workloads.generate("cfg2", 0, 512)
    r2 = ref.expm_batch(a2, accuracy=1)
    a3 = workloads.generate("cfg3", 32768 - 32, 64)  # straddles the dense/skew halves
    r3 = ref.expm_batch(a3, accuracy=0)
    np.savez_compressed(os.path.join(OUT, "cfg_slices.npz"),
                        cfg2_a=a2, cfg2_out=r2.out, cfg2_degree=r2.degree, cfg2_s=r2.s,
                        cfg2_norm=r2.norm_in, cfg2_cost=r2.cost_thirds,
                        cfg3_a=a3, cfg3_out=r3.out, cfg3_degree=r3.degree, cfg3_s=r3.s,
                        cfg3_norm=r3.norm_in)
    # reference coefficients as the library holds them
    t8, t12, t18a, t18b = ref.coefficients()
    np.savez_compressed(os.path.join(OUT, "coefficients.npz"), t8=t8, t12=t12, t18a=t18a,
                        t18b=t18b)
    print(f"wrote {len(norms)} select norms, {len(cases)} expm cases x2 tables, cfg slices")


if __name__ == "__main__":
    main()
