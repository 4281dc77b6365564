"""Parity at the configurations the bench quotes: BASELINE.json configs[2] (c3 = 2048^3, 16 chunks) at
(k, r) = (4, 16) [the bench line], (8, 8) and (4, 24), and configs[3]'s per-GPU slab c4slab (4096^2 x 512,
8 chunks of W = 64, kR/W = 1/4), in the launch configuration bench.py times (single working buffer,
Algorithm 1 over 2 lanes as bench.py runs it, host dispatcher; pinned host store, and for (4, 16) also the
HBM-resident store).

The oracle cannot run these grids, so it recomputes 256 sampled 4x4x4 output blocks one by one
(decode, k steps, encode, in the paper's order).  To cover the cross-sweep hazards
(a10) and the device store's double buffering, the GPU runs TWO sweeps in one oocs_run (2k steps, from
S_0), and the oracle starts each sample from the GPU's S_1 (a separate k-step run from the same S_0:
the GPU path is deterministic, so that run's S_1 is the one the 2-sweep run produced internally) and
runs the second sweep: decode the dependency cone (+-kR cells; the fixed Dirichlet halo where it meets
the domain edge), k in-core steps (temporal-blocking validity: a chunk's owned planes equal the
in-core result), encode the block, compare with the GPU's record in S_2.

Samples: blocks on both sides of every chunk seam, of the stencil kernel's CTA tile edges in x (64
cells) and y (16 rows), of the kernel's z-split planes (placement only: the split rule is mirrored from
kernels.cu's launch_stencil), the domain's edge blocks, and random blocks.  Tolerances: the quantiser's
bin (codes may flip where the GPU's fp32 stencil and the oracle's fp64 one straddle a bin edge) plus the
stencil's 1e-6 per step per element; the records' fp32 headers (block min / max, themselves stencil
outputs) within the stencil tolerance; at most 1% of the codes one bin off where a bin is wider than
the stencil's tolerance (q <= 16).  (Records are often not
bit-identical here: a one-ulp difference in a block's min or max, common after k fp32 steps, changes the
header bytes although every code agrees -- the codec's own bit-exactness on identical inputs is
test_gpu_parity's.)  With OOCS_REPORT_DIR set,
every case writes its exact-record fraction and the histogram of per-element differences in units of
the bin width (the codec-level form of SURVEY Q16's ulp histogram) there."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import bench  # noqa: E402
import paper_2204_11315_b200 as oocs  # noqa: E402

R = 4
N_SAMPLES = 256
# name: (nx, ny, nz, chunks, k, rate, stores)
CASES = {
    "c3_k4_r16": (2048, 2048, 2048, 16, 4, 16, ("host", "device")),
    "c3_k8_r8": (2048, 2048, 2048, 16, 8, 8, ("host",)),
    "c3_k4_r24": (2048, 2048, 2048, 16, 4, 24, ("host",)),
    "c4slab": (4096, 4096, 512, 8, 4, 16, ("host",)),
}
PARAMS = [(c, s) for c, v in CASES.items() for s in v[6]]


def _zsplit_planes(Z, nx, ny):
    """Interior-plane offsets (from the launch's z_lo) where launch_stencil splits a Z-plane step across
    CTAs (mirror of kernels.cu's wave-efficiency rule, TY = 16, 2 CTAs/SM): sample placement only."""
    gx, gy = (nx + 63) // 64, (ny + 15) // 16
    tiles, res = gx * gy, 148 * 2
    best, best_eff = 1, 0.0
    for nzc in range(1, 17):
        chunk = (Z + nzc - 1) // nzc
        if nzc > 1 and chunk < 24:
            break
        items = tiles * ((Z + chunk - 1) // chunk)
        waves = items / res
        eff = waves / np.ceil(waves) * chunk / (chunk + 4.0)
        if eff > best_eff + 1e-3:
            best_eff, best = eff, nzc
    chunk = (Z + best - 1) // best
    return [j * chunk for j in range(1, (Z + chunk - 1) // chunk)]


def _samples(nx, ny, nz, nb, k, rng):
    """(bx, by, bz) allocated block coordinates of the sampled output blocks (interior blocks only)."""
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    nbx, nby, nbz = ax // 4, ay // 4, az // 4
    W, kR = nz // nb, k * R
    zs = {1, nbz - 2}
    for i in range(1, nb):  # chunk seams: last block of chunk i-1, first block of chunk i
        zs |= {(i * W) // 4, (i * W) // 4 + 1}
    for i in (0, nb // 2, nb - 1):  # CTA z-split planes of every step of three chunks
        ext_lo, ext_hi = max(-R, i * W - kR), min(nz + R, (i + 1) * W + kR)
        for s in range(1, k + 1):
            lo = 0 if ext_lo == -R else ext_lo + s * R
            hi = nz if ext_hi == nz + R else ext_hi - s * R
            for off in _zsplit_planes(hi - lo, nx, ny):
                z = lo + off  # first plane of a CTA's z range: blocks holding z and z-1
                zs |= {(z + R) // 4, (z - 1 + R) // 4}
    zs = sorted(b for b in zs if 1 <= b <= nbz - 2)
    rng.shuffle(zs)
    zs = zs[:12] + [int(b) for b in rng.integers(1, nbz - 1, 4)]
    # x: tile edges at interior x = 64 m -> blocks 16 m (last of a tile) and 16 m + 1 (first of the next)
    xs = [1, nbx - 2] + [16 * m + d for m in (1, (nbx - 2) // 32, (nbx - 2) // 16 - 1) for d in (0, 1)]
    # y: tile edges every 16 rows -> blocks 4 m and 4 m + 1
    ys = [1, nby - 2] + [4 * m + d for m in (1, nby // 8, nby // 4 - 1) for d in (0, 1)]
    out = []
    per_z = N_SAMPLES // len(zs)
    for bz in zs:
        for j in range(per_z):
            if j < len(xs) and rng.random() < 0.5:
                bx, by = xs[j % len(xs)], int(rng.integers(1, nby - 1))
            elif j < len(ys) and rng.random() < 0.5:
                bx, by = int(rng.integers(1, nbx - 1)), ys[j % len(ys)]
            else:
                bx, by = int(rng.integers(1, nbx - 1)), int(rng.integers(1, nby - 1))
            out.append((min(max(bx, 1), nbx - 2), min(max(by, 1), nby - 2), bz))
    return out


def _cone(S1_slabs, vel_slabs, rec, nbx, nby, bx, by, bz, kR, nbz):
    """Decode the dependency cone of block (bx, by, bz) from S_1 records: blocks within kR/4 of it."""
    m = kR // 4
    x0, x1 = max(0, bx - m), min(nbx, bx + m + 1)
    y0, y1 = max(0, by - m), min(nby, by + m + 1)
    z0, z1 = max(0, bz - m), min(nbz, bz + m + 1)
    arrs = []
    for src in (vel_slabs, S1_slabs[0], S1_slabs[1]):
        sub = np.concatenate([src[z][:, y0:y1, x0:x1] for z in range(z0, z1)], axis=0).reshape(-1)
        arrs.append(sub)
    return arrs, (x0, y0, z0), (4 * (x1 - x0), 4 * (y1 - y0), 4 * (z1 - z0))


@pytest.mark.parametrize("case,store", PARAMS)
def test_sampled_blocks_second_sweep(case, store):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nx, ny, nz, nb, k, rate, _ = CASES[case]
    q, kR = rate - 1, k * R
    rec = 8 * rate
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    nbx, nby, nbz = ax // 4, ay // 4, az // 4
    dt = float(synth.dt_for())
    plan = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nb, tb_depth=k, codec="blockquant",
                                      rate_bits=rate, mode="swb", store=store, n_lanes=2))  # bench.py --lanes 2
    try:
        rng = np.random.default_rng(11315 + len(case))
        samples = _samples(nx, ny, nz, nb, k, rng)
        assert len(samples) >= N_SAMPLES - 16
        zneed = sorted({z for (_, _, bz) in samples for z in range(max(0, bz - kR // 4), min(nbz, bz + kR // 4 + 1))})
        # sweep 1 (a k-step run from S_0) -> S_1 on the cones
        bench.load_state(plan, nx, ny, nz, 0)
        plan.run(k)
        slab = lambda a, z: plan.read_raw(a, 4 * z, 4 * z + 4).reshape(nby, nbx, rec)[None]
        S1 = [{z: slab(a, z) for z in zneed} for a in (1, 2)]
        V = {z: slab(0, z) for z in zneed}
        # two sweeps in one run from the same S_0 -> S_2
        bench.load_state(plan, nx, ny, nz, 0)
        st = plan.run(2 * k)
        pb = plan.info.plane_bytes
        if store == "host":  # fixed-rate transfer identities over 2 sweeps
            assert st.bytes_h2d == 2 * 3 * (nz + 2 * R) * pb
            assert st.bytes_d2h == 2 * 2 * nz * pb
        assert st.cell_updates == nx * ny * nz * 2 * k
        out_slabs = {}
        exact = n = 0
        hist = np.zeros(6, dtype=np.int64)  # |diff| / bin in [0, .5), [.5, 1.5), [1.5, 2.5), ... , >= 4.5
        worst = 0.0
        for (bx, by, bz) in samples:
            arrs, (x0, y0, z0), (sx, sy, sz) = _cone(S1, V, rec, nbx, nby, bx, by, bz, kR, nbz)
            v, pp, pc = (oracle.decode_planes(a, sx, sy, sz, 1, q) for a in arrs)
            pp, pc = oracle.incore(v, pp, pc, dt, k)
            lx, ly, lz = 4 * (bx - x0), 4 * (by - y0), 4 * (bz - z0)
            for arr, want in ((1, pp), (2, pc)):
                if (arr, bz) not in out_slabs:
                    out_slabs[(arr, bz)] = plan.read_raw(arr, 4 * bz, 4 * bz + 4).reshape(nby, nbx, rec)
                r = out_slabs[(arr, bz)][by, bx].tobytes()
                blk = np.ascontiguousarray(want[lz:lz + 4, ly:ly + 4, lx:lx + 4]).reshape(64)
                ref_rec = oracle.encode_block(blk, q)
                exact += r == ref_rec
                n += 1
                got = oracle.decode_block(r, q).astype(np.float64)
                ref = oracle.decode_block(ref_rec, q).astype(np.float64)
                mn, mx = np.frombuffer(ref_rec[:8], dtype=np.float32)
                step = (float(mx) - float(mn)) / 2 ** q
                amax = max(float(np.abs(ref).max()), 1e-30)
                tol = 1.01 * step + k * 1e-6 * amax + 4 * float(np.spacing(np.float32(amax)))
                d = np.abs(got - ref)
                assert np.all(d <= tol), (case, store, bx, by, bz, arr, float(d.max()), tol)
                hdr_g = np.frombuffer(r[:8], dtype=np.float32).astype(np.float64)
                assert np.all(np.abs(hdr_g - np.array([mn, mx], dtype=np.float64)) <= k * 1e-6 * amax + 1e-30), (
                    case, store, bx, by, bz, arr, hdr_g, mn, mx)
                if step > 0:
                    u = d / step
                    worst = max(worst, float(u.max()))
                    hist += np.histogram(np.minimum(u, 5.0), bins=[0, .5, 1.5, 2.5, 3.5, 4.5, 5.01])[0]
        report = {"case": case, "store": store, "nx": nx, "ny": ny, "nz": nz, "chunks": nb, "k": k, "rate": rate,
                  "sweeps_run": 2, "samples": len(samples), "records_compared": n, "records_bit_identical": exact,
                  "diff_over_bin_hist": {"bins": ["<0.5", "1", "2", "3", "4", ">=4.5"], "counts": hist.tolist()},
                  "max_diff_over_bin": worst}
        rd = os.environ.get("OOCS_REPORT_DIR")
        if rd:
            os.makedirs(rd, exist_ok=True)
            with open(os.path.join(rd, f"fullsize_{case}_{store}.json"), "w") as f:
                json.dump(report, f, indent=1)
        if q <= 16:  # bins far wider than the stencil's tolerance: at most 1% of the codes one bin off
            assert hist[1:].sum() <= 0.01 * hist.sum() and hist[2:].sum() == 0, report
        # q = 23: a bin is ~1 ulp of the block's values, narrower than the stencil's own k x 1e-6; the
        # per-element tolerance above is then the whole bar (the histogram is reported)
    finally:
        plan.close()


@pytest.mark.parametrize("nx,ny", [(2048, 2048), (2040, 2044)])
def test_full_plane_step_vs_oracle(nx, ny):
    """One stencil step over whole c3-sized planes (2048^2, and a ragged 2040 x 2044 whose last CTA tiles
    are partial) against the oracle, every cell: normwise <= 1e-6 (Q16) and the per-element ulp histogram
    (written to $OOCS_REPORT_DIR/fullplane_ulp_<nx>x<ny>.json)."""
    from test_gpu_parity import _rel_err, _ulp_distance, from_ws, stream, to_ws
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nz = 24
    vel, p0 = synth.fields(nx, ny, nz)
    rng = np.random.default_rng(nx + ny)
    pprev = (p0 * np.float32(0.97) + rng.normal(scale=1e-3, size=p0.shape).astype(np.float32)).astype(np.float32)
    pprev[:R], pprev[-R:], pprev[:, :R], pprev[:, -R:], pprev[:, :, :R], pprev[:, :, -R:] = 0, 0, 0, 0, 0, 0
    pprev = np.ascontiguousarray(pprev)
    dt = synth.dt_for()
    az, ay, ax = p0.shape
    o = pprev.copy()
    oracle.step(vel, o, p0, dt, R, az - R)
    tv, tp, tc = to_ws(vel), to_ws(pprev), to_ws(p0)
    oocs.oocs_step(tv.data_ptr(), tp.data_ptr(), tc.data_ptr(), ax, ay, az, oocs.pitch_for(ax), dt, R, az - R,
                   stream())
    torch.cuda.synchronize()
    g = from_ws(tp, ax)
    sl = (slice(R, az - R), slice(R, ay - R), slice(R, ax - R))
    rel = _rel_err(g[sl], o[sl].astype(np.float64))
    d = _ulp_distance(g[sl], o[sl]).ravel()
    counts = np.histogram(d, bins=[0, 1, 2, 3, 5, 9, 17, 65, 1 << 62])[0].tolist()
    rd = os.environ.get("OOCS_REPORT_DIR")
    if rd:
        os.makedirs(rd, exist_ok=True)
        with open(os.path.join(rd, f"fullplane_ulp_{nx}x{ny}.json"), "w") as f:
            json.dump({"cells": int(d.size), "bins_ulp": ["0", "1", "2", "3-4", "5-8", "9-16", "17-64", ">64"],
                       "counts": counts, "median_ulp": float(np.median(d)), "p99_ulp": float(np.percentile(d, 99)),
                       "max_ulp": int(d.max()), "normwise_rel_err": rel}, f, indent=1)
    assert rel <= 1e-6
    # untouched outside the updated region
    assert np.array_equal(g[:R], pprev[:R]) and np.array_equal(g[:, :R], pprev[:, :R])
    assert np.array_equal(g[:, :, ax - R:], pprev[:, :, ax - R:])


def test_sampled_blocks_second_sweep_zfp():
    """The paper's codec (ZFP fixed rate, NEXT-1) at c3 (2048^3, 16 chunks, k = 4, rate 12), two sweeps,
    host store, 2 lanes: 256 sampled blocks of S_2 against the oracle's second sweep from the GPU's S_1
    (ZFP records: 8 * rate bytes per 4x4x4 block, slab-major like BlockQuant's).  Per element within
    twice the oracle's own ZFP round-trip error on the block plus the stencil's 1e-6 per step; bit-identical
    records counted (ZFP's embedded planes carry the stencil's last-ulp differences, so fewer are)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nx = ny = nz = 2048
    nb, k, rate = 16, 4, 12
    kR, rec = k * R, 8 * rate
    ax, ay, az = nx + 2 * R, ny + 2 * R, nz + 2 * R
    nbx, nby, nbz = ax // 4, ay // 4, az // 4
    dt = float(synth.dt_for())
    plan = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=dt, n_blocks=nb, tb_depth=k, codec="zfp",
                                      rate_bits=rate, mode="swb", store="host", n_lanes=2))
    try:
        samples = _samples(nx, ny, nz, nb, k, np.random.default_rng(2204))
        zneed = sorted({z for (_, _, bz) in samples for z in range(max(0, bz - kR // 4), min(nbz, bz + kR // 4 + 1))})
        bench.load_state(plan, nx, ny, nz, 0)
        plan.run(k)
        slab = lambda a, z: plan.read_raw(a, 4 * z, 4 * z + 4).reshape(nby, nbx, rec)[None]
        S1 = [{z: slab(a, z) for z in zneed} for a in (1, 2)]
        V = {z: slab(0, z) for z in zneed}
        bench.load_state(plan, nx, ny, nz, 0)
        st = plan.run(2 * k)
        assert st.bytes_h2d == 2 * 3 * (nz + 2 * R) * plan.info.plane_bytes
        out_slabs, exact, n = {}, 0, 0
        for (bx, by, bz) in samples:
            arrs, (x0, y0, z0), (sx, sy, sz) = _cone(S1, V, rec, nbx, nby, bx, by, bz, kR, nbz)
            v, pp, pc = (oracle.decode_planes(a, sx, sy, sz, 2, rate) for a in arrs)
            pp, pc = oracle.incore(v, pp, pc, dt, k)
            lx, ly, lz = 4 * (bx - x0), 4 * (by - y0), 4 * (bz - z0)
            for arr, want in ((1, pp), (2, pc)):
                if (arr, bz) not in out_slabs:
                    out_slabs[(arr, bz)] = plan.read_raw(arr, 4 * bz, 4 * bz + 4).reshape(nby, nbx, rec)
                r = out_slabs[(arr, bz)][by, bx].tobytes()
                blk = np.ascontiguousarray(want[lz:lz + 4, ly:ly + 4, lx:lx + 4]).reshape(64)
                ref_rec = oracle.zfp_encode_block(blk, rate)
                exact += r == ref_rec
                n += 1
                got = oracle.zfp_decode_block(r, rate).astype(np.float64)
                ref = oracle.zfp_decode_block(ref_rec, rate).astype(np.float64)
                amax = max(float(np.abs(blk).max()), 1e-30)
                err = float(np.abs(ref - blk.astype(np.float64)).max())
                tol = 2 * err + 4 * k * 1e-6 * amax + 4 * float(np.spacing(np.float32(amax)))
                assert np.all(np.abs(got - blk.astype(np.float64)) <= tol), (bx, by, bz, arr)
        rd = os.environ.get("OOCS_REPORT_DIR")
        if rd:
            os.makedirs(rd, exist_ok=True)
            with open(os.path.join(rd, "fullsize_c3_zfp_k4_r12_host.json"), "w") as f:
                json.dump({"case": "c3 zfp k4 r12", "records_compared": n, "records_bit_identical": exact}, f)
    finally:
        plan.close()


@pytest.mark.parametrize("store", ["device", "host"])
def test_fused_first_step_full_size_bitwise(store):
    """The decode -> first step fusion (OOCS_FLAG_FUSE_DECODE) at the bench's c3 configuration, two sweeps
    from the same S_0: sampled slabs of S_2 (every chunk seam, the domain's edge slabs, random slabs; both
    pressures) bitwise equal to the unfused run's."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nx = ny = nz = 2048
    nb, k, rate = 16, 4, 16
    rec = 8 * rate
    nbx = nby = (nx + 2 * R) // 4
    nbz = (nz + 2 * R) // 4
    W = nz // nb
    rng = np.random.default_rng(2204)
    zs = sorted({1, nbz - 2} | {(i * W) // 4 for i in range(1, nb)} | {(i * W) // 4 + 1 for i in range(1, nb, 3)}
                | {int(z) for z in rng.integers(1, nbz - 1, 6)})
    got = {}
    for fuse in (False, True):
        plan = oocs.Plan(oocs.make_config(nx=nx, ny=ny, nz=nz, dt=float(synth.dt_for()), n_blocks=nb, tb_depth=k,
                                          codec="blockquant", rate_bits=rate, mode="swb", store=store, n_lanes=2,
                                          fuse_decode=fuse))
        try:
            bench.load_state(plan, nx, ny, nz, 0)
            plan.run(2 * k)
            got[fuse] = {(a, z): plan.read_raw(a, 4 * z, 4 * z + 4) for a in (1, 2) for z in zs}
        finally:
            plan.close()
    for key in got[False]:
        assert got[False][key].size == nby * nbx * rec
        assert np.array_equal(got[False][key], got[True][key]), (store, key)
