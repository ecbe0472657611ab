"""Pins for the failure/repair branches of the oracle's Moller SCG (oracle/flmisr_oracle.c, orc_scg):
the rejected step (lambda_bar <- lambda, success <- 0), the delta re-use on the next pass, the
lambda raise lambda += delta (1 - Delta)/pp, the PD repair (delta <= 0), PR+'s beta < 0 clamp and
the FD-mode repair.  Cite: Moller's SCG (the [SCG] citation at P:186 / P:206), P:448 (runtime follows
the successful iterations), readings 10, 11, 13, 16; derivations in
tests/golden/scg_failure_branch.json.

Each expected value comes from a HAND-DERIVED reduction of the problem to one scalar line (the
derivation is in the golden file), evaluated here in 40-digit decimal arithmetic.  The reductions
eliminate lambda_bar altogether (the delta invariant of case A, the closed-form repair of case B),
so they do not restate the oracle's code: dropping lambda_bar <- lambda, flipping (1 - Delta),
recomputing delta after a rejection, dropping the repair or the PR+ clamp each turns a test red
(checked by tools/mutate_oracle.py; see its log in profiles/).  No GPU needed."""
import json
import os
from decimal import Decimal as Dec, getcontext

import numpy as np
import pytest

getcontext().prec = 40
GOLD = os.path.join(os.path.dirname(__file__), "golden", "scg_failure_branch.json")


def gold():
    with open(GOLD) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- case A
def charbonnier_line(n_pass, npix, eps, lam1, y, x0, pr_plus):
    """Closed form of case A (golden 'case_A_uniform_charbonnier'): per-pixel scalars, the delta
    invariant d = rho''(x) + lambda, trial point x + r/d.  Returns rows (f, rr, alpha, lambda, acc)."""
    eps, lam, y, x = Dec(eps), Dec(lam1), Dec(y), Dec(x0)
    n = Dec(npix)

    def rho(e):
        return (e * e + eps * eps).sqrt() - eps

    def r_of(e):                       # r = -rho'(e)
        return -e / (e * e + eps * eps).sqrt()

    def rho2(e):
        q = (e * e + eps * eps).sqrt()
        return eps * eps / (q * q * q)

    r = r_of(x - y)
    p = r
    rows = []
    for k in range(n_pass):
        d = rho2(x - y) + lam
        alpha = r / (d * p)
        xt = x + r / d
        Delta = 2 * d * (rho(x - y) - rho(xt - y)) / (r * r)
        acc = Delta >= 0
        if acc:
            r_new = r_of(xt - y)
            if (k + 1) % npix == 0:
                p = r_new
            else:
                beta = (r_new * r_new - r_new * r) / (p * r)
                if pr_plus and beta < 0:
                    beta = Dec(0)
                p = r_new + beta * p
            x, r = xt, r_new
            if Delta >= Dec("0.75"):
                lam = lam / 4
        if Delta < Dec("0.25"):
            lam = lam + d * (1 - Delta)
        rows.append((n * rho(x - y), n * r * r, alpha, lam, 1 if acc else 0))
        if r == 0:
            break
    return rows


def _case_a(orc, n_pass, rules, eps="1e-3", lam1="1e-6", x0=0):
    n = 8
    pb = orc.Problem(k=1, lr_h=n, lr_w=n, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     p_norm=1, eps=float(eps), lam=0.05, btv_alpha=0.4, btv_window=3)
    x, tr, st = orc.scg(pb, np.ones((1, n, n)), n_pass, x0=np.full((n, n), float(x0)), rules=rules,
                        lambda0=float(lam1))
    ref = charbonnier_line(n_pass, n * n, eps, lam1, 1, x0, pr_plus=bool(rules & 1))
    return x, tr, st, ref


def _check_rows(tr, ref, n_rows):
    for k in range(n_rows):
        f, rr, al, lam, _ = (float(v) for v in ref[k])
        row = tr[k + 1]
        for got, want, what in ((row[1], f, "f"), (row[2], rr, "rr"), (row[3], al, "alpha"), (row[4], lam, "lambda")):
            assert abs(got - want) <= 1e-10 * abs(want), (k + 1, what, got, want)


# passes 1..17 are far from fp64 rounding (f >= 5e-6); pass 18 lands within 1e-12 of y.
N_TIGHT = 17


@pytest.mark.parametrize("rules", [0, 1])
def test_reject_then_delta_reuse_trace(orc, rules):
    """Case A: 10 rejected passes (lambda_bar <- lambda, delta reused, lambda += delta(1-Delta)/pp),
    an accept, 4 more rejections, accepts.  alpha, lambda, f, <r,r> and the accept flags follow the
    closed form to 1e-10 relative for 17 passes (Moller / PR+)."""
    g = gold()["case_A_uniform_charbonnier"]
    x, tr, st, ref = _case_a(orc, 18, rules)
    flags = [int(v) for v in tr[1:, 5]]
    assert flags == g["accept_flags_first_18"] == [r[4] for r in ref[:18]]
    assert st["accepted"] == sum(flags)
    _check_rows(tr, ref, N_TIGHT)


def test_accept_with_small_and_middle_Delta(orc):
    """Case A2 (eps = 1e-2, lambda_1 = 0.3, x0 = 0.5): Delta = -1.40 (reject), 0.045 (ACCEPT with
    Delta < 0.25: lambda raised on an accepted step), 1.82, -1.37, 0.42 and 0.52 (accepts in
    [0.25, 0.75): lambda unchanged), ... -- the Delta thresholds 0, 0.25 and 0.75 of Moller's steps
    5-8 each decide a pass here (golden 'case_A2')."""
    g = gold()["case_A2_thresholds"]
    x, tr, st, ref = _case_a(orc, 8, 0, eps="1e-2", lam1="0.3", x0="0.5")
    flags = [int(v) for v in tr[1:, 5]]
    assert flags == g["accept_flags"] == [r[4] for r in ref]
    _check_rows(tr, ref, 8)
    assert tr[5, 4] == tr[4, 4] and tr[6, 4] == tr[5, 4]      # 0.25 <= Delta < 0.75: lambda kept
    assert tr[2, 4] > tr[1, 4]                                # accepted with Delta < 0.25: raised


def test_first_pass_by_hand(orc):
    """Case A, pass 1 as printed in the golden file: alpha_1 = 1/(rho''(-1) + 1e-6) = 500000.375 and
    the rejection raises lambda to ~7.0e-6 (Delta ~ -2)."""
    g = gold()["case_A_uniform_charbonnier"]
    _, tr, _, _ = _case_a(orc, 1, 0)
    assert tr[1, 5] == 0
    assert abs(tr[1, 3] - g["alpha_1"]) <= 1e-9 * g["alpha_1"]
    assert abs(tr[1, 4] - g["lambda_1_approx"]) <= 1e-5 * g["lambda_1_approx"]
    # rejected: f and <r,r> stay at their initial values
    assert tr[1, 1] == tr[0, 1] and tr[1, 2] == tr[0, 2]


def test_pr_plus_clamp_fires(orc):
    """Case A: beta < 0 at the accepted pass 16 (|r| shrinks without a sign change), so PR+ restarts
    p <- r and pass 17's alpha = r/(d p) = 1/d differs from Moller's; trial points (x + r/d) and
    hence f, <r,r> and the accept flags are the same for both rules."""
    _, tr0, _, ref0 = _case_a(orc, 18, 0)
    _, tr1, _, ref1 = _case_a(orc, 18, 1)
    assert float(ref0[16][2]) != pytest.approx(float(ref1[16][2]), rel=1e-3)       # the clamp matters
    assert abs(tr1[17, 3] - float(ref1[16][2])) <= 1e-10 * abs(float(ref1[16][2]))
    assert abs(tr0[17, 3] - float(ref0[16][2])) <= 1e-10 * abs(float(ref0[16][2]))
    np.testing.assert_array_equal(tr0[:, 5], tr1[:, 5])
    np.testing.assert_allclose(tr0[:N_TIGHT + 1, 1], tr1[:N_TIGHT + 1, 1], rtol=1e-12)
    # where beta >= 0 the rules agree exactly (passes 1..16)
    np.testing.assert_array_equal(tr0[:17, 3], tr1[:17, 3])


# ----------------------------------------------------------------------------- case B
A_B, C_LAMB, C_ALPHA, EPS_B = Dec("0.5"), Dec("-0.01"), Dec("0.4"), Dec("1e-3")


def _psi(t):
    return (t * t + EPS_B * EPS_B).sqrt() - EPS_B


def _dpsi(t):
    return t / (t * t + EPS_B * EPS_B).sqrt()


def _case_b(orc, curv_mode, lambda0=0.5, n_pass=1):
    pb = orc.Problem(k=1, lr_h=1, lr_w=2, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     p_norm=2, eps=float(EPS_B), lam=float(C_LAMB), btv_alpha=float(C_ALPHA), btv_window=2)
    y = np.array([[[float(A_B), -float(A_B)]]])
    return orc.scg(pb, y, n_pass, x0=np.zeros((1, 2)), curv_mode=curv_mode, sigma0=1e-4, lambda0=lambda0)


def _pass1_after_repair(h_abs):
    """Closed form after the repair: delta = |h| pp, lambda = 2|h|, alpha = 1/|h|, trial t = 2a/|h|."""
    c = C_LAMB * C_ALPHA
    a = A_B
    t = 2 * a / h_abs
    f0 = 2 * a * a
    fn = 2 * (t - a) ** 2 + c * _psi(2 * t)
    Delta = h_abs * (f0 - fn) / (4 * a * a)        # 2 delta (f0 - fn)/mu^2 with delta = |h| 2 (2a)^2, mu = 2 (2a)^2
    lam = 2 * h_abs
    acc = Delta >= 0
    if acc and Delta >= Dec("0.75"):
        lam = lam / 4
    if Delta < Dec("0.25"):
        lam = lam + h_abs * (1 - Delta)
    return 1 / h_abs, lam, (fn if acc else f0), acc, Delta


def test_pd_repair_exact_curvature(orc):
    """Case B: h = 2 + 2c/eps = -6 < 0, delta <= 0 -> lambda_bar = 2(lambda - delta/pp) = 12,
    delta = -delta + lambda pp = 6 pp, lambda = 12; alpha_1 = 1/6 exactly, accepted with Delta ~ 1.67,
    lambda -> 3 (golden 'case_B_pd_repair')."""
    g = gold()["case_B_pd_repair"]
    h = 2 + 2 * C_LAMB * C_ALPHA / EPS_B
    assert h == -6
    alpha, lam, f, acc, Delta = _pass1_after_repair(-h)
    x, tr, st = _case_b(orc, orc.CURV_EXACT)
    assert acc and abs(Delta - Dec("1.675")) < Dec("0.001")          # golden: Delta ~ 1.675
    assert abs(tr[1, 3] - g["alpha_1"]) <= 1e-15 and float(alpha) == pytest.approx(g["alpha_1"], rel=1e-15)
    assert tr[1, 4] == g["lambda_after_pass_1"] == float(lam)
    assert tr[1, 5] == 1
    assert abs(tr[1, 1] - float(f)) <= 1e-14 * float(f)
    np.testing.assert_allclose(x[0], [float(A_B) / 3, -float(A_B) / 3], rtol=1e-15)


@pytest.mark.parametrize("lambda0", [1e-6, 0.5, 5.9])
def test_pd_repair_independent_of_lambda(orc, lambda0):
    """The repaired delta = -h pp and lambda_bar = -2h do not depend on lambda as long as
    h + lambda <= 0 (golden derivation), so alpha_1 = 1/6 for every such lambda_1."""
    _, tr, _ = _case_b(orc, orc.CURV_EXACT, lambda0=lambda0)
    assert abs(tr[1, 3] - 1 / 6) <= 1e-15
    assert tr[1, 4] == 3.0


def test_pd_repair_fd_mode(orc):
    """Case B in the paper-literal FD probe (reading 16): the probe x + sigma p with
    sigma = sigma0/sqrt(pp) moves t by s = sigma0/sqrt(2), so h_FD = (g(s) - g(0))/s =
    2 + c psi'(2s)/s < 0 -> the same repair: alpha_1 = 1/|h_FD|, lambda from 2|h_FD| and the
    Delta rules."""
    # sigma = sigma0/sqrt(pp), pp = 2 (2a)^2; the probe moves t by sigma * 2a = sigma0/sqrt(2)
    s = Dec("1e-4") / Dec(2).sqrt()
    c = C_LAMB * C_ALPHA
    h_fd = 2 + c * _dpsi(2 * s) / s
    assert h_fd < 0
    alpha, lam, f, acc, _ = _pass1_after_repair(-h_fd)
    x, tr, st = _case_b(orc, orc.CURV_FD)
    assert abs(tr[1, 3] - float(alpha)) <= 1e-9 * float(alpha)
    assert abs(tr[1, 4] - float(lam)) <= 1e-9 * float(lam)
    assert tr[1, 5] == (1 if acc else 0)
