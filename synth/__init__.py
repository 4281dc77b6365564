"""Seeded synthetic inputs shaped like the paper's workload (shared by tests, smoke and bench).

This module holds NO arithmetic of the method (no stencil, no codec, no
decomposition).  It only produces the initial fields that both the oracle and
the CUDA path consume, as a pure function of (seed, global cell coordinate), so
any z-slab can be generated independently and the result is identical at any
rank count.  Recipe:

* grid: interior nx*ny*nz, allocated (nx+2R, ny+2R, nz+2R), R = 4
  (Table 1 "(1152+2xHALO)^3, HALO=4");
* velocity (read-only dataset): layered smooth model
  v = 1 + 2 z/(nz-1) + 0.1 sin(2 pi x/nx) sin(2 pi y/ny) on the interior,
  edge-replicated into the halo; v_max = 3.1;
* pressure p_0 = p_{-1} (two read-write datasets, zero initial time
  derivative): 8 Gaussian pulses of amplitude 1 and sigma = max(2, nx/32)
  cells at counter-hash-seeded positions, plus a 0.05-amplitude background of
  4 separable standing waves with wavelengths 16..64 cells (so no codec block
  is constant); pressure is 0 in the R-cell boundary halo (Dirichlet);
* dt = 0.4 / v_max (CFL 0.4; the 3D limit of this stencil is 0.4529, Q1).

``kind="gaussian"`` gives SPEC's default single centred Gaussian with v = 1
(S:L164).
"""
from __future__ import annotations

import math

import numpy as np

R = 4
SEED = 11315
V_MAX = 3.1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def _u01(seed: int, counter: int) -> float:
    return (_splitmix64(seed * 0x1000193 + counter) >> 11) / float(1 << 53)


def dt_for(kind: str = "layered") -> np.float32:
    return np.float32(0.4 / (V_MAX if kind == "layered" else 1.0))


def _axis(n: int, lo: int, hi: int) -> np.ndarray:
    """Interior coordinates of allocated indices [lo, hi) (allocated i -> i - R)."""
    return np.arange(lo, hi, dtype=np.float64) - R


def fields(nx: int, ny: int, nz: int, z_lo: int = 0, z_hi: int | None = None,
           seed: int = SEED, kind: str = "layered"):
    """Return (vel, p0) float32 arrays of shape (z_hi-z_lo, ny+2R, nx+2R) for allocated planes [z_lo, z_hi)."""
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    if z_hi is None:
        z_hi = az
    X = _axis(nx, 0, ax)
    Y = _axis(ny, 0, ay)
    Z = _axis(nz, z_lo, z_hi)
    # clamp coordinates into the interior for edge replication of v
    Xc, Yc, Zc = np.clip(X, 0, nx - 1), np.clip(Y, 0, ny - 1), np.clip(Z, 0, nz - 1)
    if kind == "gaussian":
        vel = np.ones((len(Z), ay, ax), dtype=np.float32)
        sig = max(2.0, nx / 16.0)
        gx = np.exp(-((X - (nx - 1) / 2) ** 2) / (2 * sig * sig))
        gy = np.exp(-((Y - (ny - 1) / 2) ** 2) / (2 * sig * sig))
        gz = np.exp(-((Z - (nz - 1) / 2) ** 2) / (2 * sig * sig))
        p = (gz[:, None, None] * gy[None, :, None]) * gx[None, None, :]
    else:
        vz = 1.0 + 2.0 * Zc / max(nz - 1, 1)
        vxy = 0.1 * np.outer(np.sin(2 * np.pi * Yc / ny), np.sin(2 * np.pi * Xc / nx))
        vel = (vz[:, None, None] + vxy[None, :, :]).astype(np.float32)
        sig = max(2.0, nx / 32.0)
        p = np.zeros((len(Z), ay, ax), dtype=np.float64)
        for j in range(8):
            cx = nx * (0.125 + 0.75 * _u01(seed, 3 * j + 0))
            cy = ny * (0.125 + 0.75 * _u01(seed, 3 * j + 1))
            cz = nz * (0.125 + 0.75 * _u01(seed, 3 * j + 2))
            gx = np.exp(-((X - cx) ** 2) / (2 * sig * sig))
            gy = np.exp(-((Y - cy) ** 2) / (2 * sig * sig))
            gz = np.exp(-((Z - cz) ** 2) / (2 * sig * sig))
            p += (gz[:, None, None] * gy[None, :, None]) * gx[None, None, :]
        for j in range(4):
            lam = [16.0 + 48.0 * _u01(seed, 100 + 6 * j + a) for a in range(3)]
            ph = [2 * np.pi * _u01(seed, 103 + 6 * j + a) for a in range(3)]
            wx = np.sin(2 * np.pi * X / lam[0] + ph[0])
            wy = np.sin(2 * np.pi * Y / lam[1] + ph[1])
            wz = np.sin(2 * np.pi * Z / lam[2] + ph[2])
            p += 0.05 * (wz[:, None, None] * wy[None, :, None]) * wx[None, None, :]
    # Dirichlet halo: pressure 0 outside the interior
    inx = (X >= 0) & (X < nx)
    iny = (Y >= 0) & (Y < ny)
    inz = (Z >= 0) & (Z < nz)
    p = p * (inz[:, None, None] & iny[None, :, None] & inx[None, None, :])
    return np.ascontiguousarray(vel, dtype=np.float32), np.ascontiguousarray(p, dtype=np.float32)


def fields_torch(nx: int, ny: int, nz: int, z_lo: int = 0, z_hi: int | None = None,
                 seed: int = SEED, device: str = "cuda"):
    """Same recipe as fields(kind="layered"), evaluated with torch (float64) on `device` -- for
    BASELINE-sized grids where numpy would take minutes.  Values agree with fields() to ~1 ulp
    (different libm); tests that compare against the oracle feed both sides the same arrays."""
    import torch

    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    if z_hi is None:
        z_hi = az
    f64 = dict(dtype=torch.float64, device=device)
    X = torch.arange(0, ax, **f64) - R
    Y = torch.arange(0, ay, **f64) - R
    Z = torch.arange(z_lo, z_hi, **f64) - R
    Xc, Yc, Zc = X.clamp(0, nx - 1), Y.clamp(0, ny - 1), Z.clamp(0, nz - 1)
    vz = 1.0 + 2.0 * Zc / max(nz - 1, 1)
    vxy = 0.1 * torch.outer(torch.sin(2 * math.pi * Yc / ny), torch.sin(2 * math.pi * Xc / nx))
    vel = (vz[:, None, None] + vxy[None]).to(torch.float32)
    sig = max(2.0, nx / 32.0)
    p = torch.zeros((len(Z), ay, ax), **f64)
    for j in range(8):
        cx = nx * (0.125 + 0.75 * _u01(seed, 3 * j + 0))
        cy = ny * (0.125 + 0.75 * _u01(seed, 3 * j + 1))
        cz = nz * (0.125 + 0.75 * _u01(seed, 3 * j + 2))
        gx = torch.exp(-((X - cx) ** 2) / (2 * sig * sig))
        gy = torch.exp(-((Y - cy) ** 2) / (2 * sig * sig))
        gz = torch.exp(-((Z - cz) ** 2) / (2 * sig * sig))
        p += gz[:, None, None] * torch.outer(gy, gx)[None]
    for j in range(4):
        lam = [16.0 + 48.0 * _u01(seed, 100 + 6 * j + a) for a in range(3)]
        ph = [2 * math.pi * _u01(seed, 103 + 6 * j + a) for a in range(3)]
        wx = torch.sin(2 * math.pi * X / lam[0] + ph[0])
        wy = torch.sin(2 * math.pi * Y / lam[1] + ph[1])
        wz = torch.sin(2 * math.pi * Z / lam[2] + ph[2])
        p += 0.05 * wz[:, None, None] * torch.outer(wy, wx)[None]
    inx = ((X >= 0) & (X < nx)).to(torch.float64)
    iny = ((Y >= 0) & (Y < ny)).to(torch.float64)
    inz = ((Z >= 0) & (Z < nz)).to(torch.float64)
    p *= inz[:, None, None] * torch.outer(iny, inx)[None]
    return vel, p.to(torch.float32)


def random_blocks(n_blocks: int, seed: int = 1, special: bool = True) -> np.ndarray:
    """(n_blocks, 64) float32 codec test blocks: mixed scales/offsets, optionally with
    +-0, subnormals, constant blocks and sentinel extremes."""
    rng = np.random.default_rng(seed)
    scale = 10.0 ** rng.uniform(-30, 30, size=(n_blocks, 1))
    off = rng.normal(size=(n_blocks, 1)) * scale * rng.choice([0.0, 1.0, 100.0], size=(n_blocks, 1))
    x = (rng.normal(size=(n_blocks, 64)) * scale + off).astype(np.float32)
    if special and n_blocks >= 8:
        x[0] = 0.0
        x[1, ::2] = -0.0
        x[2] = np.float32(3.25)
        x[3] = np.float32(1e-40) * np.arange(64, dtype=np.float32)  # subnormals
        x[4, :] = np.arange(64, dtype=np.float32)
        x[5] = rng.uniform(-1, 1, size=64).astype(np.float32)
        x[6, 0] = np.float32(2.0 ** 125)
        x[6, 1] = -np.float32(2.0 ** 125)
        x[7] = np.float32(-7.5)
        x[7, 17] = np.float32(-7.5) + np.float32(2 ** -20)
    return x
