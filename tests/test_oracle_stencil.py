"""Pins for the oracle's stencil (oracle_coeffs / oracle_step / oracle_incore).

Each test checks the oracle against something other than itself: the order-8
moment system solved independently with exact rationals, closed forms
(constant, linear, quadratic fields), a brute-force 25-term impulse response,
and invariants (translation equivariance, touch-only-region, determinism).
SPEC references: S:L122-123.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle

R = oracle.R


def _solve_fraction(A, b):
    n = len(A)
    M = [row[:] + [bb] for row, bb in zip(A, b)]
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col] / M[col][col]
                M[r] = [a - f * c for a, c in zip(M[r], M[col])]
    return [M[i][n] / M[i][i] for i in range(n)]


def test_coeffs_solve_the_order8_moment_system():
    # f''(0) ~ c0 f(0) + sum c_m (f(m)+f(-m)) exact for x^0, x^2, x^4, x^6, x^8
    A, b = [], []
    for p in range(5):
        row = [Fraction(1 if p == 0 else 0)] + [Fraction(2 * m ** (2 * p)) for m in range(1, 5)]
        A.append(row)
        b.append(Fraction(2 if p == 1 else 0))
    exact = _solve_fraction(A, b)
    assert exact == [Fraction(-205, 72), Fraction(8, 5), Fraction(-1, 5), Fraction(8, 315), Fraction(-1, 560)]
    c = oracle.coeffs()
    for ce, co in zip(exact, c):
        assert abs(float(ce) - co) <= 1e-16 * abs(float(ce))
    # and the m^10 moment is the first non-zero one (order exactly 8)
    assert sum(Fraction(2 * m ** 10) * exact[m] for m in range(1, 5)) != 0


def _grid(nx, ny, nz):
    return (nz + 2 * R, ny + 2 * R, nx + 2 * R)


def test_constant_and_zero_fields_are_fixed_points():
    rng = np.random.default_rng(0)
    shp = _grid(10, 9, 8)
    vel = rng.uniform(1.0, 3.0, size=shp).astype(np.float32)
    for cval in [0.0, 1.0, -3.75, 1e-30, 123456.78]:
        p_curr = np.full(shp, cval, dtype=np.float32)
        p_prev = p_curr.copy()
        oracle.step(vel, p_prev, p_curr, 0.13, R, shp[0] - R)
        assert np.array_equal(p_prev, p_curr), cval


def test_linear_field_is_unchanged():
    shp = _grid(12, 11, 10)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shp], indexing="ij")
    f = (7 + 3 * x - 2 * y + 5 * z).astype(np.float32)
    vel = np.full(shp, 2.0, dtype=np.float32)
    p_prev = f.copy()
    oracle.step(vel, p_prev, f, 0.2, R, shp[0] - R)
    assert np.array_equal(p_prev, f)


def test_quadratic_field_closed_form_in_time():
    # f = x^2+y^2+z^2 has Lap25 f = 6 exactly (stencil exact to degree 9);
    # with p_{-1} = p_0 = f and uniform c = (v dt)^2: p_n = f + 3 c n (n+1)
    # on cells whose distance to the fixed boundary is >= n R.
    nx = ny = nz = 40
    shp = _grid(nx, ny, nz)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) - n / 2 for n in shp], indexing="ij")
    f = (x * x + y * y + z * z).astype(np.float32)
    v, dt = np.float32(1.5), np.float32(0.25)
    c = (float(v) * float(dt)) ** 2
    vel = np.full(shp, v, dtype=np.float32)
    p_prev, p_curr = f.copy(), f.copy()
    steps = 3
    oracle.incore(vel, p_prev, p_curr, dt, steps)
    d = steps * R
    sl = (slice(R + d, shp[0] - R - d), slice(R + d, shp[1] - R - d), slice(R + d, shp[2] - R - d))
    want = f.astype(np.float64) + 3 * c * steps * (steps + 1)
    np.testing.assert_allclose(p_curr[sl], want[sl], rtol=2e-7, atol=0)
    want_prev = f.astype(np.float64) + 3 * c * (steps - 1) * steps
    np.testing.assert_allclose(p_prev[sl], want_prev[sl], rtol=2e-7, atol=0)


def test_unit_impulse_matches_bruteforce_25_terms():
    shp = _grid(9, 9, 9)
    cz, cy, cx = shp[0] // 2, shp[1] // 2, shp[2] // 2
    p_curr = np.zeros(shp, dtype=np.float32)
    p_curr[cz, cy, cx] = 1.0
    p_prev = np.zeros(shp, dtype=np.float32)
    dt = np.float32(0.4)
    vel = np.ones(shp, dtype=np.float32)
    cc = (1.0 * float(dt)) ** 2
    coef = [Fraction(-205, 72), Fraction(8, 5), Fraction(-1, 5), Fraction(8, 315), Fraction(-1, 560)]
    want = np.zeros(shp, dtype=np.float64)
    want[cz, cy, cx] = 2.0 + cc * 3 * float(coef[0])
    for m in range(1, 5):
        for dz, dy, dx in [(m, 0, 0), (-m, 0, 0), (0, m, 0), (0, -m, 0), (0, 0, m), (0, 0, -m)]:
            want[cz + dz, cy + dy, cx + dx] = cc * float(coef[m])
    oracle.step(vel, p_prev, p_curr, dt, R, shp[0] - R)
    assert np.count_nonzero(p_prev) == 25
    np.testing.assert_allclose(p_prev, want.astype(np.float32), rtol=1e-7, atol=0)


def test_translation_equivariance_and_region():
    rng = np.random.default_rng(3)
    shp = _grid(8, 8, 12)
    vel = rng.uniform(1, 3, size=shp).astype(np.float32)
    pc = rng.normal(size=shp).astype(np.float32)
    pp = rng.normal(size=shp).astype(np.float32)
    # step planes [6, 10) of the buffer, then the same physics shifted down one plane
    a = pp.copy()
    oracle.step(vel, a, pc, 0.1, 6, 10)
    b = np.roll(pp, -1, axis=0).copy()
    oracle.step(np.roll(vel, -1, axis=0).copy(), b, np.roll(pc, -1, axis=0).copy(), 0.1, 5, 9)
    assert np.array_equal(a[6:10], b[5:9])
    # touch-only-region: everything outside planes [6,10) and the x/y halo is unchanged
    mask = np.zeros(shp, dtype=bool)
    mask[6:10, R:-R, R:-R] = True
    assert np.array_equal(a[~mask], pp[~mask])
    assert not np.array_equal(a[mask], pp[mask])


def test_incore_zero_steps_identity_and_determinism():
    rng = np.random.default_rng(5)
    shp = _grid(8, 8, 8)
    vel = rng.uniform(1, 3, size=shp).astype(np.float32)
    p0 = rng.normal(size=shp).astype(np.float32)
    a, b = p0.copy(), p0.copy()
    oracle.incore(vel, a, b, 0.1, 0)
    assert np.array_equal(a, p0) and np.array_equal(b, p0)
    r1 = oracle.incore(vel, p0.copy(), p0.copy(), 0.1, 5)
    r2 = oracle.incore(vel, p0.copy(), p0.copy(), 0.1, 5)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])
    # odd step counts return levels (T-1, T): one more step from (4,5) state equals 6 steps
    s5p, s5c = oracle.incore(vel, p0.copy(), p0.copy(), 0.1, 5)
    s6p, s6c = oracle.incore(vel, p0.copy(), p0.copy(), 0.1, 6)
    oracle.step(vel, s5p, s5c, 0.1, R, shp[0] - R)
    assert np.array_equal(s5p, s6c)


# ---- non-uniform velocity: the c = (v dt)^2 factor is taken at the updated cell -----------------------
def test_bruteforce_25_terms_nonuniform_velocity():
    """Random fields and a strongly varying random velocity: every updated cell against the 25-term sum
    written out with exact rationals from the fp32 inputs (p_next = 2p - p_prev + v^2 dt^2 Lap25),
    rounded once to fp32.  A velocity taken at a neighbour, c = v^2 dt or c = v dt^2 all fail."""
    rng = np.random.default_rng(11)
    shp = _grid(5, 4, 3)
    vel = rng.uniform(0.5, 3.0, size=shp).astype(np.float32)
    pc = rng.normal(size=shp).astype(np.float32)
    pp = rng.normal(size=shp).astype(np.float32)
    dt = np.float32(0.13)
    out = pp.copy()
    oracle.step(vel, out, pc, dt, R, shp[0] - R)
    coef = [Fraction(-205, 72), Fraction(8, 5), Fraction(-1, 5), Fraction(8, 315), Fraction(-1, 560)]
    F = lambda a: Fraction(float(a))
    n_checked = 0
    for z in range(R, shp[0] - R):
        for y in range(R, shp[1] - R):
            for x in range(R, shp[2] - R):
                lap = 3 * coef[0] * F(pc[z, y, x])
                for m in range(1, 5):
                    lap += coef[m] * (F(pc[z, y, x + m]) + F(pc[z, y, x - m]) + F(pc[z, y + m, x]) + F(pc[z, y - m, x])
                                      + F(pc[z + m, y, x]) + F(pc[z - m, y, x]))
                c = (F(vel[z, y, x]) * F(dt)) ** 2
                want = 2 * F(pc[z, y, x]) - F(pp[z, y, x]) + c * lap
                got = F(out[z, y, x])
                # the oracle rounds its fp64 sum once to fp32: within one fp32 ulp of the exact value
                ulp = np.spacing(np.float32(abs(float(want))))
                assert abs(float(got - want)) <= float(ulp), (z, y, x, float(got), float(want))
                # and distinguishable from the plausible mistakes
                wrong_c = [(F(wv) * F(dt)) ** 2 for wv in (vel[z, y, x + 1], vel[z + 1, y, x], vel[z, y - 1, x])]
                wrong_c += [F(vel[z, y, x]) ** 2 * F(dt), F(vel[z, y, x]) * F(dt) ** 2]
                for wc in wrong_c:
                    if abs(float((wc - c) * lap)) > 4 * float(ulp):
                        assert abs(float(got - (2 * F(pc[z, y, x]) - F(pp[z, y, x]) + wc * lap))) > float(ulp)
                n_checked += 1
    assert n_checked == 5 * 4 * 3


def test_quadratic_field_closed_form_with_varying_velocity():
    """f = x^2+y^2+z^2, p_-1 = p_0 = f, and a velocity with v^2 linear in x, y and z (so that
    c = (v dt)^2 is linear and Lap25 c = 0, the stencil being exact to degree 9): then
    p_n = f + 3 n (n+1) c(x,y,z) pointwise, on cells at distance >= nR from the fixed boundary.
    With c varying by ~3e-3 per plane a velocity index off by one cell in any axis is ~10^3 ulps off."""
    nx = ny = nz = 36
    shp = _grid(nx, ny, nz)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shp], indexing="ij")
    f = ((x - shp[2] / 2) ** 2 + (y - shp[1] / 2) ** 2 + (z - shp[0] / 2) ** 2).astype(np.float32)
    vel = np.sqrt(1.0 + 0.5 * z + 0.3 * x + 0.2 * y).astype(np.float32)
    dt = np.float32(0.05)
    c = (vel.astype(np.float64) * float(dt)) ** 2  # exactly the oracle's c (fp64 from fp32 v, dt)
    assert vel.max() * float(dt) < 0.4529  # CFL (Q1)
    p_prev, p_curr = f.copy(), f.copy()
    steps = 3
    oracle.incore(vel, p_prev, p_curr, dt, steps)
    d = steps * R
    sl = (slice(R + d, shp[0] - R - d), slice(R + d, shp[1] - R - d), slice(R + d, shp[2] - R - d))
    for n, got in ((steps, p_curr), (steps - 1, p_prev)):
        want = f.astype(np.float64) + 3 * n * (n + 1) * c
        np.testing.assert_allclose(got[sl], want[sl], rtol=3e-7, atol=0)
        # c shifted by one cell along any axis is far outside that tolerance
        for ax_ in range(3):
            wrong = f.astype(np.float64) + 3 * n * (n + 1) * np.roll(c, 1, axis=ax_)
            assert np.max(np.abs(got[sl] - wrong[sl]) / np.abs(wrong[sl])) > 1e-5, (n, ax_)
