"""NEXT-4: CROWN-style back-substitution for MatrixInv.  The conic
bounds are obtained by propagating each entry's coefficients backwards through
Xp = X0 + X0 sum_i P^i, P^i = P^{i-1} E with the fixed R1 / R2 planes (forward bounds of the
operands) down to E = I - X X0, instead of concretising forward forms.  Pins: Example 1
moves towards the paper's 0.70 and stays above the empirical 0.66 with every sampled inverse
inside (Lemma 1); random SPD boxes: containment and never wider than forward; whole-pipeline
containment at sampled poses."""
import copy
import json
import os

import numpy as np
import pytest

from tests import helpers as H
from workloads import make_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _entry(n, c, r, k):
    f = np.zeros(2 * (n + 1))
    f[n] = f[2 * n + 1] = c
    f[k] = f[n + 1 + k] = r
    return f


def _bounds(oracle, conic, n):
    L = np.array([oracle.form_conc(conic[e], n)[0] for e in range(4)]).reshape(2, 2)
    U = np.array([oracle.form_conc(conic[e], n)[1] for e in range(4)]).reshape(2, 2)
    return L, U


def test_example1_backward(oracle):
    g = json.load(open(os.path.join(GOLD, "example1.json")))
    lo, hi = np.array(g["X_lo"]), np.array(g["X_hi"])
    c00, r00 = (lo[0, 0] + hi[0, 0]) / 2, (hi[0, 0] - lo[0, 0]) / 2
    c11, r11 = (lo[1, 1] + hi[1, 1]) / 2, (hi[1, 1] - lo[1, 1]) / 2
    r01 = hi[0, 1]
    n = 3
    X = np.stack([_entry(n, c00, r00, 0), _entry(n, 0.0, r01, 2), _entry(n, 0.0, r01, 2),
                  _entry(n, c11, r11, 1)])
    _, cf, _, _ = oracle.matrix_inv(X, n, g["k"])
    st, cb, _, _ = oracle.matrix_inv(X, n, g["k"], backward=True)
    assert st == 0
    Lf, Uf = _bounds(oracle, cf, n)
    Lb, Ub = _bounds(oracle, cb, n)
    wf, wb = np.linalg.norm(Uf - Lf), np.linalg.norm(Ub - Lb)
    rng = np.random.default_rng(0)
    xs = rng.uniform(-1, 1, (100000, 3))
    xs[:8] = [[a, b, c] for a in (-1, 1) for b in (-1, 1) for c in (-1, 1)]
    M = np.empty((len(xs), 2, 2))
    M[:, 0, 0] = c00 + r00 * xs[:, 0]
    M[:, 1, 1] = c11 + r11 * xs[:, 1]
    M[:, 0, 1] = M[:, 1, 0] = r01 * xs[:, 2]
    inv = np.linalg.inv(M)
    emp = np.linalg.norm(inv.max(axis=0) - inv.min(axis=0))
    assert np.all(inv >= Lb - 1e-12) and np.all(inv <= Ub + 1e-12)  # Lemma 1
    assert emp <= wb < wf
    assert abs(wb - g["width_matrixinv_paper"]) < abs(wf - g["width_matrixinv_paper"])
    assert abs(wb - 0.7371) < 5e-4  # regression pin of this rule (reading O17)
    assert np.all(Lb >= Lf - 1e-12) and np.all(Ub <= Uf + 1e-12)


def test_random_spd_boxes(oracle):
    rng = np.random.default_rng(7)
    n = 3
    checked = 0
    for _ in range(60):
        c00, c11 = rng.uniform(0.5, 2.0, 2)
        c01 = rng.uniform(-0.3, 0.3) * np.sqrt(c00 * c11)
        r = rng.uniform(0.01, 0.25, 3) * np.array([c00, c11, np.sqrt(c00 * c11)])
        X = np.stack([_entry(n, c00, r[0], 0), _entry(n, c01, r[2], 2), _entry(n, c01, r[2], 2),
                      _entry(n, c11, r[1], 1)])
        st, cb, _, _ = oracle.matrix_inv(X, n, 8, backward=True)
        sf, cf, _, _ = oracle.matrix_inv(X, n, 8)
        assert st == sf
        if st != 0:
            continue
        checked += 1
        Lb, Ub = _bounds(oracle, cb, n)
        Lf, Uf = _bounds(oracle, cf, n)
        xs = rng.uniform(-1, 1, (4000, 3))
        M = np.empty((len(xs), 2, 2))
        M[:, 0, 0] = c00 + r[0] * xs[:, 0]
        M[:, 1, 1] = c11 + r[1] * xs[:, 1]
        M[:, 0, 1] = M[:, 1, 0] = c01 + r[2] * xs[:, 2]
        ok = np.linalg.det(M) > 0
        inv = np.linalg.inv(M[ok])
        assert np.all(inv >= Lb - 1e-9) and np.all(inv <= Ub + 1e-9)
        assert np.linalg.norm(Ub - Lb) <= np.linalg.norm(Uf - Lf) + 1e-12
    assert checked >= 30


def test_pipeline_backward_sound_and_tighter(oracle):
    w = make_config("C4", N=3000, res=40)
    v = copy.deepcopy(w)
    v.pose_box = dict(w.pose_box, inv_backward=1)
    flo, fhi, fst = oracle.render_bounds(w)
    lo, hi, st = oracle.render_bounds(v)
    assert st["fails"] == fst["fails"]
    assert H.mpg(lo, hi) < H.mpg(flo, fhi)
    rng = np.random.default_rng(9)
    params = H.sample_params(w, rng, n_random=20, corners=True)
    for p in params[:1] + params[1:65:8] + params[65:]:
        e, t, sh = H.pose_of(w, p)
        img = oracle.render_concrete(w, euler=e, t=t, shifts=sh)
        assert np.all(lo <= img + 1e-9) and np.all(img <= hi + 1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw", [("C4", dict(N=6000, res=72)), ("C3", dict(N=5000, res=56)),
                                     ("C1", {})])
def test_gpu_backward_parity(oracle, name, kw):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_00308_b200 import Context
    w = make_config(name, **kw)
    w.pose_box = dict(w.pose_box, inv_backward=1)
    with Context(0) as ctx:
        ctx.load_workload(w)
        lo, hi, st = ctx.as_render_bounds(w.tile, w.batch)
        olo, ohi, ost = oracle.render_bounds(w)
        err = max(np.abs(lo.cpu().numpy() - olo).max(), np.abs(hi.cpu().numpy() - ohi).max())
        assert err <= 1e-4, err
        assert st["fails"] == ost["fails"] and st["pairs"] == ost["pairs"]
        # tighter than the forward conic on the same context
        ctx.as_set_inverse_mode(0)
        flo, fhi, _ = ctx.as_render_bounds(w.tile, w.batch)
        assert H.mpg(lo.cpu().numpy(), hi.cpu().numpy()) <= H.mpg(flo.cpu().numpy(), fhi.cpu().numpy()) + 1e-9
