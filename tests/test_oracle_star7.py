"""Pins for the oracle's STAR7 stencil (oracle_step7; oocs.h OOCS_STENCIL_STAR7, SURVEY §8(b) "STAR7 (R=1)
for small exact tests").

Checked against things other than the oracle: the textbook 7-point Laplacian written out term by term on
a unit impulse with a non-uniform velocity (brute force), its Fourier symbol 2cos(theta) - 2 per axis on
plane waves (closed form), the quadratic closed form in time, linear and constant fixed points, and the
pipeline's temporal-blocking validity (blocked == in-core bitwise with the Identity codec).
"""
import numpy as np
import pytest

import oracle

R = oracle.R
S7 = oracle.STENCIL_STAR7


def _grid(nx, ny, nz):
    return (nz + 2 * R, ny + 2 * R, nx + 2 * R)


def test_impulse_bruteforce_7_terms_nonuniform_velocity():
    shp = _grid(9, 9, 9)
    rng = np.random.default_rng(7)
    vel = rng.uniform(1.0, 3.0, size=shp).astype(np.float32)
    dt = 0.11
    c0 = (R + 4, R + 4, R + 4)
    p_curr = np.zeros(shp, dtype=np.float32)
    p_curr[c0] = 1.0
    p_prev = rng.uniform(-1, 1, size=shp).astype(np.float32)
    pp0 = p_prev.copy()
    oracle.step(vel, p_prev, p_curr, dt, R, shp[0] - R, stencil=S7)
    # written out: p_next = 2 f0 - p_prev + (v dt)^2 * sum_axes (f[+1] + f[-1] - 2 f0), each cell's own v
    for z in range(R, shp[0] - R):
        for y in range(R, shp[1] - R):
            for x in range(R, shp[2] - R):
                f = lambda dz, dy, dx: float(p_curr[z + dz, y + dy, x + dx])
                lap = (f(0, 0, 1) + f(0, 0, -1) - 2 * f(0, 0, 0)) + (f(0, 1, 0) + f(0, -1, 0) - 2 * f(0, 0, 0)) \
                    + (f(1, 0, 0) + f(-1, 0, 0) - 2 * f(0, 0, 0))
                c = (float(vel[z, y, x]) * float(np.float32(dt))) ** 2
                want = np.float32(2 * f(0, 0, 0) - float(pp0[z, y, x]) + c * lap)
                assert p_prev[z, y, x] == want, (z, y, x)
    # the centre and its six neighbours are the only cells the impulse reaches
    cz, cy, cx = c0
    vc = (float(vel[c0]) * float(np.float32(dt))) ** 2
    assert p_prev[c0] == np.float32(2 - float(pp0[c0]) - 6 * vc)
    for d in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
        i = (cz + d[0], cy + d[1], cx + d[2])
        assert p_prev[i] == np.float32(-float(pp0[i]) + (float(vel[i]) * float(np.float32(dt))) ** 2)
    far = (cz + 2, cy, cx)
    assert p_prev[far] == np.float32(-float(pp0[far]))


@pytest.mark.parametrize("theta", [0.3, 1.0, 2.2])
def test_plane_wave_symbol(theta):
    # f = cos(theta x): Lap7 f = (2 cos theta - 2) f exactly (textbook symbol of the 3-point second
    # difference); the 25-point stencil's symbol is c0 + 2 sum c_m cos(m theta) -- they differ, so a
    # swapped stencil fails here
    shp = _grid(16, 6, 6)
    x = np.arange(shp[2], dtype=np.float64)
    f = np.broadcast_to(np.cos(theta * x), shp).astype(np.float32).copy()
    vel = np.ones(shp, dtype=np.float32)
    zero = np.zeros(shp, dtype=np.float32)
    dt = 0.25
    p_prev = zero.copy()
    oracle.step(vel, p_prev, f, dt, R, shp[0] - R, stencil=S7)
    sl = (slice(R, -R), slice(R, -R), slice(R, -R))
    # exact symbol applied to the fp32 samples themselves (cos(theta(x+-1)) rounded), in fp64
    fd = f.astype(np.float64)
    lap = np.roll(fd, 1, 2) + np.roll(fd, -1, 2) - 2 * fd
    want = 2 * fd + (dt * dt) * lap
    assert np.max(np.abs(p_prev[sl] - want[sl])) <= 4e-7
    # and the continuum-symbol form: (2 + dt^2 (2cos theta - 2)) cos(theta x), to fp32 sampling error
    cont = (2 + dt * dt * (2 * np.cos(theta) - 2)) * np.cos(theta * x)
    assert np.max(np.abs(p_prev[sl] - np.broadcast_to(cont, shp)[sl])) <= 2e-6
    # not the 25-point symbol: the two predictions differ by far more than the tolerance above
    c = oracle.coeffs()
    s25 = c[0] + 2 * sum(c[m] * np.cos(m * theta) for m in range(1, 5))
    assert abs(s25 - (2 * np.cos(theta) - 2)) * dt * dt > 50 * 4e-7


def test_constant_linear_fixed_points():
    shp = _grid(10, 9, 8)
    rng = np.random.default_rng(1)
    vel = rng.uniform(1.0, 3.0, size=shp).astype(np.float32)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shp], indexing="ij")
    for f in [np.full(shp, 2.5, dtype=np.float32), (7 + 3 * x - 2 * y + 5 * z).astype(np.float32)]:
        p_prev = f.copy()
        oracle.step(vel, p_prev, f, 0.2, R, shp[0] - R, stencil=S7)
        assert np.array_equal(p_prev, f)


def test_quadratic_closed_form_in_time():
    # Lap7 (x^2+y^2+z^2) = 6 exactly: p_n = f + 3 c n (n+1) on cells at distance >= n from the boundary
    n_steps, shp = 5, _grid(24, 24, 24)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) - n / 2 for n in shp], indexing="ij")
    f = (x * x + y * y + z * z).astype(np.float32)
    dt, v = 0.25, 1.5
    vel = np.full(shp, v, dtype=np.float32)
    a, b = oracle.incore(vel, f.copy(), f.copy(), dt, n_steps, stencil=S7)
    c = (v * float(np.float32(dt))) ** 2
    m = R + n_steps
    sl = (slice(m, -m), slice(m, -m), slice(m, -m))
    want = f.astype(np.float64) + 3 * c * n_steps * (n_steps + 1)
    assert np.max(np.abs(b[sl] - want[sl])) <= 1e-5 * np.abs(want[sl]).max()


@pytest.mark.parametrize("n,k", [(1, 1), (2, 3), (4, 2), (3, 1)])
def test_identity_pipeline_bitwise_equals_incore(n, k):
    nx = ny = 12
    nz = 48
    shp = _grid(nx, ny, nz)
    rng = np.random.default_rng(n * 10 + k)
    vel = rng.uniform(1.0, 2.0, size=shp).astype(np.float32)
    p0 = np.zeros(shp, dtype=np.float32)
    p0[R:-R, R:-R, R:-R] = rng.standard_normal((nz, ny, nx)).astype(np.float32)
    steps = 2 * k
    S = [oracle.encode_planes(a, 0, 0) for a in (vel, p0, p0)]
    oracle.pipeline(shp[2], shp[1], nz, n, k, 0.3, steps, 0, 0, *S, stencil=S7)
    a, b = oracle.incore(vel, p0.copy(), p0.copy(), 0.3, steps, stencil=S7)
    got_c = oracle.decode_planes(S[2], shp[2], shp[1], shp[0], 0, 0)
    assert np.array_equal(got_c, b)
    # and the result differs from the 25-point stencil's (the stencil argument reached the steps)
    a25, b25 = oracle.incore(vel, p0.copy(), p0.copy(), 0.3, steps)
    assert not np.array_equal(b25, b)
