"""CPU tests of the C-ABI library: symbols, validation, decomposition and the lowered schedule.

No compute calls (no GPU here).  The schedule tests run the exact op list
oocs_run issues through tests/schedule_check.py: every pair of operations that
touch the same bytes (one writing) must be ordered by stream order or events
(SPEC validate_exclusive S:L409-417, acceptance #2 S:L655), Algorithm 1's
paper-visible sequence must match the hand-unrolled golden file (acceptance #8
S:L661), and deleting the paper's working-buffer waits must create a race.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2204_11315_b200 as oocs
import schedule_check as sc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "oocs.h")).read()
    names = set(re.findall(r"^\s*(?:oocs_status|const char \*|int32_t)\s*(oocs_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 17
    L = ctypes.CDLL(oocs.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n
    assert oocs.lib().oocs_abi_version() == 2


def cfg(**kw):
    base = dict(nx=64, ny=64, nz=64, dt=0.1, n_blocks=4, tb_depth=2)
    base.update(kw)
    return oocs.make_config(**base)


@pytest.mark.parametrize("kw", [
    dict(nx=63), dict(nz=0), dict(n_blocks=17), dict(tb_depth=4), dict(rate_bits=25), dict(rate_bits=1),
    dict(mode="baseline", codec="blockquant"), dict(world=3), dict(rank=4, world=4), dict(dt=-1.0),
    dict(region_sharing=False, store="host"), dict(codec=7), dict(codec="trunc16", rate_bits=8),
    dict(codec="zfp", rate_bits=33), dict(codec="zfp", rate_bits=0), dict(decoded_velocity=True, store="host"),
    dict(mode="baseline", codec="identity", world=2, rank=0),
    dict(stencil=2), dict(v_max=-1.0), dict(v_max=float("nan")),
    dict(dt=0.1, v_max=4.53),            # 0.453 > 2/sqrt(3*2048/315) = 0.45286 (ACOUSTIC25 CFL, Q1)
    dict(dt=0.1, v_max=5.78, stencil="star7"),  # 0.578 > 2/sqrt(12) = 0.57735
    # the decode -> first step fusion: BlockQuant at an even rate <= 16, codec modes, the 25-point stencil
    dict(fuse_decode=True, rate_bits=24), dict(fuse_decode=True, rate_bits=15), dict(fuse_decode=True, codec="zfp"),
    dict(fuse_decode=True, mode="baseline", codec="identity"), dict(fuse_decode=True, stencil="star7"),
])
def test_config_errors(kw):
    with pytest.raises(oocs.OocsError) as e:
        oocs.oocs_plan_table(cfg(**kw))
    assert e.value.status == 2


@pytest.mark.parametrize("rate", [8, 12, 16])
def test_fuse_decode_accepted(rate):
    oocs.oocs_plan_table(cfg(fuse_decode=True, rate_bits=rate))


@pytest.mark.parametrize("stencil,vdt", [("acoustic25", 0.4528), ("star7", 0.4529), ("star7", 0.5773)])
def test_cfl_limit_accepts_below(stencil, vdt):
    # the limits are 2/sqrt(3 |L1(pi)|): 25-point |L1(pi)| = 2048/315 (exact rationals), 7-point 4
    from fractions import Fraction
    sym25 = Fraction(205, 72) + 2 * (Fraction(8, 5) + Fraction(1, 5) + Fraction(8, 315) + Fraction(1, 560))
    assert sym25 == Fraction(2048, 315)
    assert vdt < 2 / (3 * float(sym25 if stencil == "acoustic25" else 4)) ** 0.5
    oocs.oocs_plan_table(cfg(dt=0.1, v_max=vdt / 0.1, stencil=stencil))


def test_struct_size_is_checked():
    c = cfg()
    c.struct_size = 8
    with pytest.raises(oocs.OocsError):
        oocs.oocs_plan_table(c)


@pytest.mark.parametrize("nz,n,k", [(1152, 8, 12), (64, 4, 2), (128, 8, 3), (40, 3, 2), (16, 1, 3), (96, 5, 1)])
def test_decomposition_matches_oracle(nz, n, k):
    # the library's planner and the oracle's are written independently
    got = np.array(oocs.oocs_plan_table(cfg(nz=nz, n_blocks=n, tb_depth=k)))
    want = oracle.plan(nz, n, k)
    assert np.array_equal(got, want)


def test_encoded_bytes_fixed_rate_law():
    # rate 16 = half of fp32 (P:L170's 1/2); identity = 4 B/value
    c16 = cfg(rate_bits=16)
    c_id = cfg(codec="identity")
    ax = 72
    assert oocs.oocs_encoded_bytes(c16, 4) * 2 == oocs.oocs_encoded_bytes(c_id, 4) == 4 * ax * ax * 4
    for r in (8, 12, 24):
        assert oocs.oocs_encoded_bytes(cfg(rate_bits=r), 8) == 8 * ax * ax * r // 8
        assert oocs.oocs_encoded_bytes(cfg(codec="zfp", rate_bits=r), 8) == 8 * ax * ax * r // 8
    # Truncate-16: raw bf16 planes, the same bytes as rate-16 BlockQuant
    assert oocs.oocs_encoded_bytes(cfg(codec="trunc16", rate_bits=16), 4) == oocs.oocs_encoded_bytes(c16, 4)
    for codec, r in (("trunc16", 16), ("zfp", 12)):
        assert oocs.oocs_encoded_bytes(cfg(codec=codec, rate_bits=r), 12) == 12 * oracle.plane_bytes(
            ax, ax, {"trunc16": 3, "zfp": 2}[codec], r)


def _geo(c, blocks):
    L = c.n_lanes or 3
    n_ws = {0: L, 1: L, 2: 1, 3: 2}[c.mode] if c.store == 0 else 1
    return dict(k=c.tb_depth, n_ws=n_ws, lanes=L, mode={0: "baseline"}.get(c.mode, "codec"), nz=c.nz,
                max_ext=max(b[3] - b[2] for b in blocks), max_own=max(b[1] - b[0] for b in blocks),
                resident_velocity=bool(c.flags & oocs.FLAG_RESIDENT_VELOCITY),
                fuse_decode=bool(c.flags & oocs.FLAG_FUSE_DECODE))


def _check(c, steps):
    ops = oocs.oocs_schedule(c, steps)
    blocks = oocs.oocs_plan_table(c)
    return ops, sc.violations(ops, blocks, _geo(c, blocks))


MODES = [("swb", "blockquant"), ("dwb", "blockquant"), ("compress", "blockquant"), ("baseline", "identity"),
         ("swb", "identity"), ("swb", "trunc16")]


@pytest.mark.parametrize("sched", ["alg1", "dag", "dag_func"])
@pytest.mark.parametrize("lanes", [0, 2, 4])
@pytest.mark.parametrize("mode,codec", MODES)
@pytest.mark.parametrize("n,k,nz", [(1, 1, 16), (2, 1, 32), (3, 2, 48), (4, 2, 64), (5, 3, 80), (8, 1, 64),
                                    (12, 1, 96)])
def test_schedule_is_race_free(mode, codec, n, k, nz, lanes, sched):
    c = cfg(nz=nz, n_blocks=n, tb_depth=k, mode=mode, codec=codec, n_lanes=lanes, schedule=sched)
    ops, bad = _check(c, 3 * k)  # three sweeps: exercises the cross-sweep host-store hazards
    assert bad == [], bad[:5]
    # every chunk of every sweep is decoded/computed/encoded exactly once per step
    assert sum(o["kind"] == "STEP" for o in ops) == 3 * n * k


@pytest.mark.parametrize("sched", ["alg1", "dag", "dag_func"])
@pytest.mark.parametrize("lanes", [0, 2, 4])
@pytest.mark.parametrize("mode", ["swb", "dwb", "compress"])
@pytest.mark.parametrize("resident", [False, True])
@pytest.mark.parametrize("n,k,nz", [(1, 1, 16), (3, 2, 48), (5, 3, 80), (12, 1, 96)])
def test_schedule_is_race_free_with_fused_first_step(mode, n, k, nz, lanes, sched, resident):
    # OOCS_FLAG_FUSE_DECODE adds a read of the staging buffer (p_{t-1}'s records) to every chunk's first step
    c = cfg(nz=nz, n_blocks=n, tb_depth=k, mode=mode, n_lanes=lanes, schedule=sched, fuse_decode=True,
            resident_velocity=resident)
    ops, bad = _check(c, 3 * k)
    assert bad == [], bad[:5]


def test_fused_first_step_read_is_guarded():
    # the model sees the fused read: deleting the waits that order the next H2D into a staging slot after
    # that slot's chunk is done (its D2H) exposes the first step's read, not only the decode's
    c = cfg(nz=64, n_blocks=4, tb_depth=2, mode="swb", fuse_decode=True)
    ops = oocs.oocs_schedule(c, 4)
    blocks = oocs.oocs_plan_table(c)
    geo = _geo(c, blocks)
    assert sc.violations(ops, blocks, geo) == []
    fused_reads = [i for i, o in enumerate(ops) if o["kind"] == "STEP" and o["arg"] == 1]
    assert fused_reads and any(r[0] == ("hf", ops[fused_reads[0]]["g"] % 3)
                               for r in sc.footprint(ops[fused_reads[0]], blocks, geo))


def test_algorithm1_golden_n3():
    c = cfg(nz=48, n_blocks=3, tb_depth=1, mode="swb")
    ops = oocs.oocs_schedule(c, 1)
    seq = []
    for o in ops:
        if o["kind"] in ("H2D", "DECODE", "STEP", "ENCODE", "D2H"):
            seq.append(f"{o['kind']} {o['lane']} {o['block']}")
        elif o["kind"] in ("RECORD", "WAIT") and o["ev"] == "ENC":
            seq.append(f"{o['kind']} {o['lane']} {o['block']} ENC")
    gold = [l.strip() for l in open(os.path.join(ROOT, "tests", "golden", "alg1_n3.txt"))
            if l.strip() and not l.startswith("#")]
    # Algorithm 1's meaning is its per-stream programs plus its record -> wait pairs; the interleaving
    # of different streams in the listing is not (the library issues H2D(i) before chunk i-1's tail,
    # which runs on another stream: DESIGN.md §8).  Compare every stream's program, and that each wait
    # follows the record it waits for.
    per_lane = lambda s: {ln: [x for x in s if x.split()[1] == ln] for ln in "012"}
    assert per_lane(seq) == per_lane(gold)
    assert sorted(seq) == sorted(gold)
    for q in (seq, gold):
        for j, x in enumerate(q):
            if x.startswith("WAIT"):
                blk = int(x.split()[2])
                assert f"RECORD {(blk - 1) % 3} {blk - 1} ENC" in q[:j], (x, q)
    # lanes cycle 0,1,2,0 and waits connect lanes cyclically 0->1->2
    c4 = cfg(nz=64, n_blocks=4, tb_depth=1, mode="swb")
    ops4 = oocs.oocs_schedule(c4, 1)
    assert [o["lane"] for o in ops4 if o["kind"] == "H2D"] == [0, 1, 2, 0]
    waits = [(o["lane"], o["ev_g"] % 3) for o in ops4 if o["kind"] == "WAIT" and o["ev"] == "ENC"]
    assert waits == [(1, 0), (2, 1), (0, 2)]


@pytest.mark.parametrize("mode", ["swb", "dwb"])
def test_deleting_a_working_buffer_wait_creates_a_race(mode):
    c = cfg(nz=64, n_blocks=4, tb_depth=2, mode=mode)
    ops = oocs.oocs_schedule(c, 4)
    blocks = oocs.oocs_plan_table(c)
    geo = _geo(c, blocks)
    assert sc.violations(ops, blocks, geo) == []
    idx = [i for i, o in enumerate(ops) if o["kind"] == "WAIT" and o["ev"] == "ENC"]
    assert idx
    for i in idx:
        mutated = ops[:i] + ops[i + 1:]
        assert sc.violations(mutated, blocks, geo, limit=1), f"deleting op {i} went unnoticed"


def test_deleting_carry_and_cross_sweep_waits_is_detected():
    c = cfg(nz=64, n_blocks=4, tb_depth=2, mode="swb")
    ops = oocs.oocs_schedule(c, 4)
    blocks = oocs.oocs_plan_table(c)
    geo = _geo(c, blocks)
    # the carry runs on the previous chunk's stream right after its H2D and steps, so it needs no H2D
    # wait; it waits for the destination buffer's last D2H, and the next chunk's decode waits for it
    assert not [o for o in ops if o["kind"] == "WAIT" and o["ev"] == "H2D"]
    idx = [i for i, o in enumerate(ops) if o["kind"] == "WAIT" and o["ev"] == "D2H"]
    assert sum(bool(sc.violations(ops[:i] + ops[i + 1:], blocks, geo, limit=1)) for i in idx) >= 1
    # the decode's carry wait: implied by the working-buffer wait under SWB (the previous chunk's encode
    # follows the carry on its stream), a real edge with 2 or 3 working sets (also with 2kR > W)
    for mode, nz, n, k in (("dwb", 64, 4, 2), ("compress", 64, 4, 2), ("dwb", 80, 5, 3), ("swb", 80, 5, 3)):
        c = cfg(nz=nz, n_blocks=n, tb_depth=k, mode=mode)
        ops = oocs.oocs_schedule(c, 2 * k)
        blocks = oocs.oocs_plan_table(c)
        geo = _geo(c, blocks)
        assert sc.violations(ops, blocks, geo) == []
        idx = [i for i, o in enumerate(ops) if o["kind"] == "WAIT" and o["ev"] == "CARRY"]
        caught = sum(bool(sc.violations(ops[:i] + ops[i + 1:], blocks, geo, limit=1)) for i in idx)
        assert caught == (len(idx) if mode != "swb" else 0), (mode, caught, len(idx))


def test_transfer_byte_identities():
    # region sharing: each interior chunk transfers exactly 2kR planes fewer per dataset
    for n, k in [(4, 2), (8, 1), (3, 3)]:
        c = cfg(nz=96, n_blocks=n, tb_depth=k)
        t = oocs.oocs_plan_table(c)
        body = sum(b[7] - b[6] for b in t)
        ext = sum(b[3] - b[2] for b in t)
        assert ext - body == (n - 1) * 2 * k * oocs.R
        # and the H2D planes of one sweep cover [-R, nz+R) exactly once
        assert body == 96 + 2 * oocs.R


def _al(b):
    return (b + 255) // 256 * 256


@pytest.mark.parametrize("rate", [8, 16, 24])
def test_memory_accounting_paper_units(rate):
    """baseline = 1 x datasets x 3 streams working buffers; compressed + SWB = 0.5 x 3 x 3 + 1 x
    datasets.  Our datasets are 3 (the write-only 4th is removed, Q21), so in units of one
    array's (unpadded) working buffer: baseline 9, COMPRESS 9 + 9r/32, SWB 3 + 9r/32 (= 7.5 at r = 16,
    the paper's printed figure), DWB 6 + 9r/32."""
    nx = ny = 100  # ax = 108: working rows padded to 160 floats, compressed planes are not
    base = dict(nx=nx, ny=ny, nz=256, dt=0.1, n_blocks=4, tb_depth=4, rate_bits=rate)
    info = {m: oocs.oocs_plan_estimate(cfg(mode=m, codec="identity" if m == "baseline" else "blockquant", **base))
            for m in ("baseline", "compress", "swb", "dwb")}
    i = info["swb"]
    E, ax, ay, pitch = i.max_ext_planes, i.ax, i.ay, i.pitch
    U_ws = _al(E * ay * pitch * 4)                # one array's working buffer as allocated
    U_c = E * i.plane_bytes                         # one array's compressed (half-size at r = 16) buffer
    assert i.plane_bytes * 32 == ax * ay * 4 * rate  # fixed-rate law: r/32 of the fp32 plane
    assert info["baseline"].arena_bytes == 9 * U_ws + 256
    assert info["swb"].arena_bytes == 3 * U_ws + 3 * _al(3 * U_c) + 256
    assert info["dwb"].arena_bytes == 6 * U_ws + 3 * _al(3 * U_c) + 256
    assert info["compress"].arena_bytes == 9 * U_ws + 3 * _al(3 * U_c) + 256
    # the same numbers in the paper's units (unpadded working buffer = 1)
    U = E * ax * ay * 4
    units = {m: 3 * info[m].n_working_sets + info[m].staging_bytes / U for m in info}
    assert units["baseline"] == 9
    assert units["swb"] == pytest.approx(3 + 9 * rate / 32, abs=0.01)
    if rate == 16:
        assert units["swb"] == pytest.approx(7.5, abs=0.01)  # "0.5x3x3 + 1x3" (P:L245 prints 7.5)
        assert 1 - units["swb"] / units["baseline"] == pytest.approx(1 / 6, abs=1e-3)


def test_decoded_velocity_accounting():
    """OOCS_FLAG_DECODED_VELOCITY adds exactly one fp32 array over the rank's store planes (allocated
    rows, pitch) to the device-store arena, and nothing else."""
    kw = dict(nx=1024, ny=1024, nz=1024, dt=0.1, n_blocks=8, tb_depth=4, rate_bits=16, store="device")
    for world, rank in ((1, 0), (4, 1)):
        a = oocs.oocs_plan_estimate(cfg(world=world, rank=rank, **kw))
        b = oocs.oocs_plan_estimate(cfg(world=world, rank=rank, decoded_velocity=True, **kw))
        planes = a.store_hi - a.store_lo
        assert b.arena_bytes - a.arena_bytes == _al(planes * a.ay * a.pitch * 4)


def test_plan_estimate_c5_swb_vs_dwb():
    # BASELINE configs[4]: 4096x4096x8192, 128 chunks, at 8 B200 -- per-rank arena, SWB vs DWB (no allocation)
    kw = dict(nx=4096, ny=4096, nz=8192, dt=0.1, n_blocks=128, tb_depth=4, rate_bits=16, world=8)
    swb = [oocs.oocs_plan_estimate(cfg(mode="swb", rank=r, **kw)) for r in range(8)]
    dwb = [oocs.oocs_plan_estimate(cfg(mode="dwb", rank=r, **kw)) for r in range(8)]
    for s, d in zip(swb, dwb):
        assert d.arena_bytes - s.arena_bytes == s.working_set_bytes  # exactly one more working set
        assert s.store_bytes > 100e9  # ~104 GB compressed state per rank: truly out of core


@pytest.mark.parametrize("mode", ["swb", "dwb", "compress"])
def test_dag_schedule_derives_no_more_waits_than_alg1(mode):
    # the DAG + Kahn + events recipe reproduces Algorithm 1's operation order and needs at most
    # as many cross-stream waits as the hand-lowered Algorithm 1 with its hazard repairs
    c1 = cfg(nz=128, n_blocks=8, tb_depth=2, mode=mode)
    c2 = cfg(nz=128, n_blocks=8, tb_depth=2, mode=mode, schedule="dag")
    a, d = oocs.oocs_schedule(c1, 6), oocs.oocs_schedule(c2, 6)
    core = lambda ops: [(o["kind"], o["lane"], o["g"], o["arg"]) for o in ops if o["kind"] not in ("WAIT", "RECORD")]
    assert core(a) == core(d)
    assert sum(o["kind"] == "WAIT" for o in d) <= sum(o["kind"] == "WAIT" for o in a)
    blocks = oocs.oocs_plan_table(c2)
    geo = _geo(c2, blocks)
    idx = [i for i, o in enumerate(d) if o["kind"] == "WAIT"]
    caught = sum(bool(sc.violations(d[:i] + d[i + 1:], blocks, geo, limit=1)) for i in idx)
    assert caught >= len(idx) * 3 // 4  # (almost) every derived wait is load-bearing


def test_create_in_rejects_null_arena_without_a_gpu():
    # argument checks come before any CUDA call, so this runs on a CPU-only box
    with pytest.raises(oocs.OocsError) as e:
        oocs.oocs_plan_create_in(cfg(), 0, 1 << 20)
    assert e.value.status == 2


def test_binding_structs_mirror_the_header():
    out = (ctypes.c_int64 * 6)()
    oocs.lib().oocs_abi_sizes(out)
    mine = [ctypes.sizeof(t) for t in (oocs.Config, oocs.Stats, oocs.PlanInfo, oocs.Block, oocs.Op, oocs.Span)]
    assert list(out) == mine


# ---- multi-GPU (world > 1): the per-rank schedule with in-library peer sends ------------------------
@pytest.mark.parametrize("sched", ["alg1", "dag", "dag_func"])
@pytest.mark.parametrize("mode", ["swb", "dwb", "compress"])
@pytest.mark.parametrize("world,n,k", [(2, 4, 2), (3, 3, 1), (4, 8, 3)])
def test_multirank_schedule_race_free_with_sends(world, n, k, mode, sched):
    """Every rank's op list is race-free over 3 sweeps (the SEND reads the encoded edge planes before the
    lane's next H2D overwrites them), has no host barrier, and sends each edge once per sweep: the
    first chunk's lower kR planes to rank-1 (arg bit 0), the last chunk's upper planes to rank+1 (bit 1).
    Sweeps stay pipelined back to back: the only cross-rank dependencies are device-side flags."""
    nz = 16 * n
    for r in range(world):
        c = cfg(nz=nz * world, n_blocks=n * world, tb_depth=k, mode=mode, schedule=sched, rank=r, world=world)
        ops, bad = _check(c, 3 * k)
        assert bad == [], (r, bad[:3])
        sends = [o for o in ops if o["kind"] == "SEND"]
        first, last = r * n, (r + 1) * n - 1
        want = []
        for t in range(3):
            for blk in sorted({first, last}):
                m = (1 if blk == first and r > 0 else 0) | (2 if blk == last and r + 1 < world else 0)
                if m:
                    want.append((t, blk, m))
        assert sorted((o["sweep"], o["block"], o["arg"]) for o in sends) == sorted(want)
        # the send follows its chunk's encode and precedes its D2H on the same lane
        for o in sends:
            lane_ops = [(i, x["kind"]) for i, x in enumerate(ops) if x["g"] == o["g"] and x["kind"] in ("ENCODE", "SEND", "D2H")]
            assert [k_ for _, k_ in lane_ops] == ["ENCODE", "SEND", "D2H"]


def test_multirank_device_store_sends_after_every_sweep():
    """The device store sends too, after every sweep including the last one (the next oocs_run starts from
    the neighbours' current edge planes: run(a); run(b) == run(a + b))."""
    for r in range(3):
        c = cfg(nz=96, n_blocks=6, tb_depth=2, store="device", rank=r, world=3)
        ops = oocs.oocs_schedule(c, 2)  # one sweep
        sends = [(o["block"], o["arg"]) for o in ops if o["kind"] == "SEND"]
        want = {0: [(1, 2)], 1: [(2, 1), (3, 2)], 2: [(4, 1)]}[r]
        assert sorted(sends) == want


def test_multirank_exchange_region_accounting():
    """world > 1 adds exactly one exchange region to the device peak -- 256 B of flags plus 2 sides x 2
    parities x 2 pressures ghost slots of kR planes -- and nothing else (host store: the rank's arena
    equals a one-rank plan of the same chunk geometry)."""
    kw = dict(nx=256, ny=256, dt=0.1, tb_depth=4, rate_bits=16)
    b = oocs.oocs_plan_estimate(cfg(nz=512, n_blocks=8, world=2, rank=1, **kw))
    one = oocs.oocs_plan_estimate(cfg(nz=256, n_blocks=4, **kw))
    assert (b.max_ext_planes, b.working_set_bytes, b.staging_bytes) == (one.max_ext_planes, one.working_set_bytes,
                                                                      one.staging_bytes)
    slot = _al(4 * oocs.R * b.plane_bytes)
    assert b.arena_bytes - one.arena_bytes == _al(256 + 8 * slot)


def test_schedule_race_free_random_configs():
    """Seeded random configurations beyond the grid above (chunk counts with remainders, 2kR > W, up to 8
    lanes, resident velocity, 2-4 sweeps): every lowered schedule is race-free under stream + event
    semantics, and every chunk is decoded, stepped and encoded exactly once per sweep."""
    rng = np.random.default_rng(2204)
    done = 0
    while done < 60:
        n = int(rng.integers(1, 13))
        k = int(rng.integers(1, 5))
        units = int(rng.integers(n, 4 * n + 6))
        nz = 4 * units
        mode = ["swb", "dwb", "compress", "baseline"][int(rng.integers(0, 4))]
        codec = "identity" if mode == "baseline" else ["blockquant", "zfp", "trunc16"][int(rng.integers(0, 3))]
        rate = {"identity": 32, "blockquant": 16, "zfp": 12, "trunc16": 16}[codec]
        lanes = [0, 2, 4, 8][int(rng.integers(0, 4))]
        sched = ["alg1", "dag", "dag_func"][int(rng.integers(0, 3))]
        resv = mode != "baseline" and bool(rng.integers(0, 2))
        c = cfg(nz=nz, n_blocks=n, tb_depth=k, mode=mode, codec=codec, rate_bits=rate, n_lanes=lanes,
                schedule=sched, resident_velocity=resv)
        try:
            oocs.oocs_plan_table(c)
        except oocs.OocsError:
            continue  # k*R >= W for some chunk: rejected, not a schedule
        sweeps = int(rng.integers(2, 5))
        ops, bad = _check(c, sweeps * k)
        assert bad == [], (n, k, nz, mode, codec, lanes, sched, resv, bad[:3])
        for kind, per in (("DECODE", 1), ("STEP", k), ("ENCODE", 1)):
            if mode == "baseline" and kind != "STEP":
                continue
            assert sum(o["kind"] == kind for o in ops) == sweeps * n * per
        done += 1


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("mode", ["swb", "dwb", "compress"])
@pytest.mark.parametrize("n,k,nz,lanes", [(4, 2, 64, 0), (16, 1, 128, 2), (2, 1, 32, 0), (5, 3, 80, 2), (1, 1, 16, 0)])
def test_chained_runs_are_race_free(mode, n, k, nz, lanes, fuse):
    """oocs_run_async issues a run while the previous one drains: the dispatcher sees the two op lists
    back to back (lane programs and events continue across them).  Their concatenation must be race-free
    under stream + event semantics, and the second run's first H2Ds must carry the cross-sweep waits on
    the first run's write-backs -- deleting them is a detected race."""
    c = cfg(nz=nz, n_blocks=n, tb_depth=k, mode=mode, n_lanes=lanes, fuse_decode=fuse)
    s1, s2, s3 = 2 * k, k, 3 * k
    ops = (oocs.oocs_schedule(c, s1) + oocs.oocs_schedule(c, s2, first_sweep=s1 // k)
           + oocs.oocs_schedule(c, s3, first_sweep=(s1 + s2) // k))
    blocks = oocs.oocs_plan_table(c)
    geo = _geo(c, blocks)
    assert sc.violations(ops, blocks, geo) == []
    assert sum(o["kind"] == "STEP" for o in ops) == n * (s1 + s2 + s3)
    # the chunk counter continues: every global chunk is decoded exactly once
    dec = [o["g"] for o in ops if o["kind"] == "DECODE"]
    assert dec == list(range(n * (s1 + s2 + s3) // k))
    n1 = len(oocs.oocs_schedule(c, s1))
    cross = [i for i, o in enumerate(ops) if i >= n1 and o["kind"] == "WAIT" and o["ev"] == "D2H"
             and o["ev_g"] < (s1 // k) * n]
    assert cross, "the second run must wait on the first run's write-backs"
    caught = sum(bool(sc.violations(ops[:i] + ops[i + 1:], blocks, geo, limit=1)) for i in cross)
    assert caught >= 1


def test_schedule_at_is_a_restart_where_runs_cannot_chain():
    # DAG schedules, the BASELINE mode, the device store and multi-rank plans restart at chunk 0
    for kw in (dict(schedule="dag"), dict(mode="baseline", codec="identity", rate_bits=32), dict(store="device"),
               dict(world=2, rank=0)):
        c = cfg(nz=64, n_blocks=4, tb_depth=2, **kw)
        assert oocs.oocs_schedule(c, 4, first_sweep=3) == oocs.oocs_schedule(c, 4)
