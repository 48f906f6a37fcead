"""Offline constrained minimax fit of the Boys Q-function approximation.

Build-time tooling only (never imported by the product path or the GPU box):
it needs the reference oracle ``boysfn.refmath`` from ``/root/reference``
(pure Python + mpmath) to sample Q_n(x).

What is fitted:

    Q~_n(x) = q0 + q1 x + q2 x^2 u(x)/v(x)                      (Eq. 12)

with q0 = Q_n(0), q1 = Q'_n(0), q2 = alpha_n - q1, u monic of degree N-1,
v monic of degree N.  This parameterisation builds in three of the four
constraints of SPEC.md:133 (value and slope at 0, slope alpha_n at
infinity); the fourth (intercept beta_n, Eq. 8) is the linear relation

    u_{N-2} = v_{N-1} + (beta_n - q0)/q2,

so 2N-2 coefficients are free, the same count as SPEC.md:145-148.

Objective (Eq. 15): the max relative error of
F~_n = c_n/(x + Q~^p e^-x)^p, p = n + 1/2, over [0, z_nb).  To first order
dF/F = -w dQ/Q with w = p^2 Q^p e^-x/(x + Q^p e^-x), so the
linearised residual at node x_i is

    e_i = w_i q2 x_i^2 (u(x_i) - g_i v(x_i)) / (v(x_i) Q_i),
    g_i = (Q_i - q0 - q1 x_i)/(q2 x_i^2).

It is minimised in the max-norm by Sanathanan-Koerner linearisation (divide
by the previous iterate's v) combined with Lawson's iteratively reweighted
least squares, solved as normal equations at 448-bit precision.  The true
(non-linearised) error is then measured on a dense grid against Q_n from
the reference oracle (``refmath.q_of_x``), and the worst points are added
to the node set (an exchange step) before refitting.
"""

from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass, field

from mpmath import mp

_REF = os.environ.get("BOYS_REFERENCE_SRC", "/root/reference/pkg/src")
if _REF not in sys.path:
    sys.path.insert(0, _REF)
from boysfn import refmath as R  # noqa: E402  (reference oracle, build-time only)

FIT_BITS = 448          # working precision of the linear algebra
SAMPLE_BITS = 192       # Precision() passed to the oracle for Q_n samples


@dataclass
class FitResult:
    n: int
    N: int
    bits_target: int               # 53 (double profile) or 24 (single)
    consts: R.AnalyticConstants
    z: object                      # cut-off z_{n,b} (mpf)
    u: list                        # monic u coefficients, ascending, in x
    v: list                        # monic v coefficients, ascending, in x
    exact_bits: float              # -log2 max |F~/F - 1| on the dense grid
    argmax: float
    u_quads: list = field(default_factory=list)   # [(y, a)]
    u_lins: list = field(default_factory=list)    # [y]
    v_quads: list = field(default_factory=list)   # [(z, b)]
    v_lins: list = field(default_factory=list)    # [z]
    grid_points: int = 0
    rescan_bits: float = 0.0


def _q_sample(n, x):
    return R.q_of_x(n, x, R.Precision(SAMPLE_BITS))


def _polyval(coeffs, x):
    """Horner, coefficients ascending."""
    acc = mp.mpf(0)
    for c in reversed(coeffs):
        acc = acc * x + c
    return acc


class _Problem:
    """Precomputed per-node quantities in the scaled variable t = x/S."""

    def __init__(self, n, N, consts, S, xs, Qs):
        self.n, self.N, self.S = n, N, S
        p = mp.mpf(2 * n + 1) / 2
        q0, q1 = consts.q0, consts.q1
        q2 = consts.alpha - q1
        self.kappa_t = (consts.beta - q0) / q2 / S
        self.rows = []
        for x, Q in zip(xs, Qs):
            t = x / S
            g_t = S * (Q - q0 - q1 * x) / (q2 * x * x)      # u~/v~ target
            E = mp.power(Q, p) * mp.exp(-x)
            w = p * p * E / (x + E)
            W = w * q2 * x * x / Q / S                       # rel-F per unit (u~-g v~)/v~
            self.rows.append((t, g_t, W))

    def unpack(self, theta):
        """theta -> (u~, v~) monic coefficient lists in t, ascending."""
        N = self.N
        nu = N - 2
        uc = list(theta[:nu])
        vc = list(theta[nu:nu + N - 1])
        vtop = theta[nu + N - 1]
        u = uc + [vtop + self.kappa_t, mp.mpf(1)]
        v = vc + [vtop, mp.mpf(1)]
        return u, v

    def design_row(self, t, g):
        N = self.N
        tp = [mp.mpf(1)]
        for _ in range(N):
            tp.append(tp[-1] * t)
        row = [tp[k] for k in range(N - 2)]
        row += [-g * tp[k] for k in range(N - 1)]
        row.append(tp[N - 2] - g * tp[N - 1])
        rhs = -(self.kappa_t * tp[N - 2] + tp[N - 1] - g * tp[N])
        return row, rhs

    def lin_errors(self, u, v):
        out = []
        for t, g, W in self.rows:
            vv = _polyval(v, t)
            out.append(W * (_polyval(u, t) - g * vv) / vv)
        return out


def _lawson(prob, iters=60, u0=None, v0=None):
    """SK-Lawson iteration. Returns (u~, v~, max linearised error)."""
    M = len(prob.rows)
    k = 2 * prob.N - 2
    lam = [mp.mpf(1) / M] * M
    vprev = [mp.mpf(1)] * M
    if v0 is not None:
        vprev = [_polyval(v0, t) for t, _, _ in prob.rows]
    design = [prob.design_row(t, g) for t, g, _ in prob.rows]
    best = None
    for it in range(iters):
        cols = [[None] * M for _ in range(k)]
        rhs = [None] * M
        for i, ((t, g, W), (row, b)) in enumerate(zip(prob.rows, design)):
            s = mp.sqrt(lam[i]) * W / vprev[i]
            for j in range(k):
                cols[j][i] = row[j] * s
            rhs[i] = b * s
        # column equilibration
        norms = [mp.sqrt(mp.fdot(c, c)) or mp.mpf(1) for c in cols]
        cols = [[e / nm for e in c] for c, nm in zip(cols, norms)]
        G = mp.matrix(k, k)
        r = mp.matrix(k, 1)
        for a in range(k):
            for b2 in range(a, k):
                G[a, b2] = G[b2, a] = mp.fdot(cols[a], cols[b2])
            r[a] = mp.fdot(cols[a], rhs)
        sol = mp.lu_solve(G, r)
        theta = [sol[j] / norms[j] for j in range(k)]
        u, v = prob.unpack(theta)
        err = prob.lin_errors(u, v)
        emax = max(abs(e) for e in err)
        if best is None or emax < best[2]:
            best = (u, v, emax)
        tot = mp.fsum(l * abs(e) for l, e in zip(lam, err))
        lam = [l * abs(e) / tot for l, e in zip(lam, err)]
        vprev = [_polyval(v, t) for t, _, _ in prob.rows]
    return best


def _to_x(u_t, v_t, S):
    """Monic coefficients in t = x/S -> monic coefficients in x."""
    du, dv = len(u_t) - 1, len(v_t) - 1
    u = [c * mp.power(S, du - j) for j, c in enumerate(u_t)]
    v = [c * mp.power(S, dv - j) for j, c in enumerate(v_t)]
    return u, v


def qtilde(consts, u, v, x):
    q2 = consts.alpha - consts.q1
    return consts.q0 + consts.q1 * x + q2 * x * x * _polyval(u, x) / _polyval(v, x)


def rel_f_error(n, consts, u, v, x, Q):
    """Exact F~/F - 1 given the true Q_n(x)."""
    p = mp.mpf(2 * n + 1) / 2
    ex = mp.exp(-x)
    Qt = qtilde(consts, u, v, x)
    if Qt <= 0:
        return mp.inf
    num = x + mp.power(Q, p) * ex
    den = x + mp.power(Qt, p) * ex
    return mp.power(num / den, p) - 1


def factorize(coeffs):
    """Monic polynomial (ascending coeffs) -> (quads [(y, a)], lins [y]),
    quads are complex-conjugate pairs (x-y)^2 + a with a = Im^2 > 0,
    each list sorted by real part ascending."""
    deg = len(coeffs) - 1
    roots = mp.polyroots(list(reversed(coeffs)), maxsteps=400, extraprec=2 * mp.prec)
    quads, lins = [], []
    used = [False] * deg
    scale = max(abs(r) for r in roots) if roots else 1
    for i, r in enumerate(roots):
        if used[i]:
            continue
        if abs(mp.im(r)) <= mp.mpf(2) ** (-mp.prec // 2) * (1 + scale):
            lins.append(mp.re(r))
            used[i] = True
            continue
        # find the conjugate
        j = min((j for j in range(deg) if not used[j] and j != i),
                key=lambda j: abs(roots[j] - mp.conj(r)))
        used[i] = used[j] = True
        y = (mp.re(r) + mp.re(roots[j])) / 2
        a = (abs(mp.im(r)) + abs(mp.im(roots[j]))) / 2
        quads.append((y, a * a))
    quads.sort(key=lambda q: q[0])
    lins.sort()
    return quads, lins


def expand(quads, lins):
    """Inverse of factorize (for the round-trip check)."""
    poly = [mp.mpf(1)]

    def mul(p, q):
        out = [mp.mpf(0)] * (len(p) + len(q) - 1)
        for i, a in enumerate(p):
            for j, b in enumerate(q):
                out[i + j] += a * b
        return out

    for y, a in quads:
        poly = mul(poly, [y * y + a, -2 * y, mp.mpf(1)])
    for y in lins:
        poly = mul(poly, [-y, mp.mpf(1)])
    return poly


def fit(n, N, bits_target, m_nodes=None, lawson_iters=60, exchange_rounds=2,
        grid=1500, verbose=False):
    """Fit Q~_n with denominator degree N for the b-bit profile."""
    with mp.workprec(FIT_BITS):
        consts = R.constants(n, R.Precision(256))
        z = R.cutoff_solve(n, bits_target, R.Precision(256))
        X = z * mp.mpf("1.02")
        S = X / 2
        M = m_nodes or (12 * N + 96)
        nodes = [X / 2 * (1 - mp.cos(mp.pi * (i + mp.mpf(1) / 2) / M)) for i in range(M)]
        qs = [_q_sample(n, x) for x in nodes]
        # dense validation grid on (0, z): equally spaced, as PAPER.md:235-238
        gx = [z * (i + 1) / (grid + 1) for i in range(grid)]
        gq = [_q_sample(n, x) for x in gx]
        u_t = v_t = None
        for rnd in range(exchange_rounds + 1):
            prob = _Problem(n, N, consts, S, nodes, qs)
            u_t, v_t, lmax = _lawson(prob, iters=lawson_iters, v0=v_t)
            u, v = _to_x(u_t, v_t, S)
            errs = [rel_f_error(n, consts, u, v, x, q) for x, q in zip(gx, gq)]
            aerr = [abs(e) for e in errs]
            emax = max(aerr)
            imax = aerr.index(emax)
            if verbose:
                print(f"  n={n} N={N} round {rnd}: lin {float(-mp.log(lmax, 2)):.2f} bits,"
                      f" grid {float(-mp.log(emax, 2)):.2f} bits at x={float(gx[imax]):.4g}",
                      flush=True)
            if rnd == exchange_rounds:
                break
            # exchange: add local maxima of the grid error that exceed the node max
            add = []
            for i in range(1, len(aerr) - 1):
                if aerr[i] >= aerr[i - 1] and aerr[i] >= aerr[i + 1] and aerr[i] > lmax:
                    add.append(gx[i])
            if not add:
                break
            for x in add:
                nodes.append(x)
                qs.append(_q_sample(n, x))
        res = FitResult(n=n, N=N, bits_target=bits_target, consts=consts, z=z, u=u, v=v,
                        exact_bits=float(-mp.log(emax, 2)), argmax=float(gx[imax]),
                        grid_points=grid)
        res.u_quads, res.u_lins = factorize(u)
        res.v_quads, res.v_lins = factorize(v)
        return res


def rescan_bits(res, factor=4):
    """-log2 max |F~/F - 1| re-derived on a fresh grid `factor` times denser
    than the fit's ("re-derives exact_error_bits on a fresh 4x
    denser grid"): equally spaced midpoints of factor * grid_points cells of
    [0, z), none of them a point of the fit's own grid."""
    with mp.workprec(FIT_BITS):
        M = factor * max(1, res.grid_points)
        worst = mp.mpf(0)
        for i in range(M):
            x = res.z * (2 * i + 1) / (2 * M)
            e = abs(rel_f_error(res.n, res.consts, res.u, res.v, x, _q_sample(res.n, x)))
            worst = max(worst, e)
        return float(-mp.log(worst, 2)) if worst > 0 else float("inf")


def validate(res, rescan=4, drift_bits=0.5):
    """SPEC.md:182-190 checks. Returns a list of violation strings.

    rescan: density factor of the fresh-grid re-derivation of exact_bits
    (0 skips it); a drift of more than drift_bits below the recorded value
    means the fit grid under-resolved the error curve."""
    bad = []
    with mp.workprec(FIT_BITS):
        v0 = res.v[0]
        if not v0 > 0:
            bad.append("B_N <= 0 (v(0) <= 0): rejected by the paper's section III rule "
                       "(PAPER.md:163-164, solutions with B_N < 0 are rejected)")
        for zr in res.v_lins:
            if zr >= 0:
                bad.append(f"pole of v on [0, inf): real root {zr}")
        for _, b in res.v_quads:
            if not b > 0:
                bad.append("v quadratic factor with b <= 0")
        for _, a in res.u_quads:
            if not a > 0:
                bad.append("u quadratic factor with a <= 0")
        L, lu = len(res.u_quads), len(res.u_lins)
        M, lv = len(res.v_quads), len(res.v_lins)
        if 2 * L + lu != res.N - 1:
            bad.append("degree(u) != N-1")
        if 2 * M + lv != res.N:
            bad.append("degree(v) != N")
        # factored vs coefficient form
        ue = expand(res.u_quads, res.u_lins)
        ve = expand(res.v_quads, res.v_lins)
        for k in range(1, 11):
            x = res.z * k / 10
            for a, b in ((ue, res.u), (ve, res.v)):
                pa, pb = _polyval(a, x), _polyval(b, x)
                if abs(pa - pb) > abs(pb) * mp.mpf(2) ** (-200):
                    bad.append(f"factored/coefficient mismatch at x={float(x)}")
        # Q~ > 0 on [0, z] (needed for the half-integer power)
        for k in range(0, 201):
            x = res.z * k / 200
            if not qtilde(res.consts, res.u, res.v, x) > 0:
                bad.append(f"Q~ <= 0 at x={float(x)}")
                break
    if rescan and not bad:
        rb = rescan_bits(res, rescan)
        res.rescan_bits = rb
        if rb < res.exact_bits - drift_bits:
            bad.append(f"grid-refinement drift: {rescan}x denser grid gives {rb:.2f} bits vs "
                       f"{res.exact_bits:.2f} recorded (> {drift_bits} bit): under-resolved grid")
    return bad


if __name__ == "__main__":
    import time
    n, N, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    t0 = time.time()
    r = fit(n, N, b, verbose=True)
    print(f"n={n} N={N} b={b}: exact {r.exact_bits:.2f} bits; "
          f"u {len(r.u_quads)}q+{len(r.u_lins)}l v {len(r.v_quads)}q+{len(r.v_lins)}l; "
          f"{time.time() - t0:.1f}s; violations={validate(r)}")
