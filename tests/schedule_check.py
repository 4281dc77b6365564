"""Structural race checker for lowered pipeline schedules (test tooling; SPEC validate_exclusive S:L409-417).

Builds the happens-before relation of an op list (lane FIFO order, RECORD -> WAIT
event edges) and the memory footprint of every op
(buffer, array, plane range, read/write), then reports every pair of ops that
touch overlapping memory with at least one write but are not ordered.
"""
from __future__ import annotations

R = 4


def footprint(op, blocks, geo):
    """list of (resource, lo, hi, is_write)."""
    k = geo["k"]
    n_ws = geo["n_ws"]
    mode = geo["mode"]
    g = op["g"]
    b = blocks[op["block"]]
    own_lo, own_hi, ext_lo, ext_hi, c_lo, c_hi, body_lo, body_hi = b
    L = geo.get("lanes", 3)
    s = g % L
    w = g % n_ws
    E = ext_hi - ext_lo
    out = []
    kind = op["kind"]
    up_last = 1 if k % 2 else 2
    if mode == "baseline":
        if kind == "H2D":
            for a in range(3):
                out.append((("host", a), body_lo, body_hi, False))
                out.append((("ws", s, a), body_lo - ext_lo, ext_hi - ext_lo, True))
        elif kind == "CARRY":  # op.g is the receiving chunk
            pb = blocks[op["block"] - 1]
            sp = (g - 1) % L
            for a in range(3):
                out.append((("ws", sp, a), c_lo - pb[2], c_hi - pb[2], False))
                out.append((("ws", s, a), c_lo - ext_lo, c_hi - ext_lo, True))
        elif kind == "STEP":
            st = op["arg"]
            lo = 0 if ext_lo == -R else ext_lo + st * R
            hi = geo["nz"] if ext_hi == geo["nz"] + R else ext_hi - st * R
            up = 1 if st % 2 else 2
            for a in (0, 3 - up):
                out.append((("ws", s, a), lo - R - ext_lo, hi + R - ext_lo, False))
            out.append((("ws", s, up), lo - ext_lo, hi - ext_lo, True))
        elif kind == "D2H":
            for a in (1, 2):
                out.append((("ws", s, a), own_lo - ext_lo, own_hi - ext_lo, False))
                out.append((("host", a), own_lo, own_hi, True))
        return out
    # one half-size buffer per lane (hf_buf[s]), in plane units: incoming array a at
    # [a*ME, a*ME + E), outgoing owned planes of pressure j at [j*MO, j*MO + W)
    ME, MO = geo["max_ext"], geo["max_own"]
    # OOCS_FLAG_RESIDENT_VELOCITY: the velocity never passes through the staging buffers (its compressed
    # planes stay in HBM, read-only, and the decode reads them there)
    a0 = 1 if geo.get("resident_velocity") else 0
    if kind == "H2D":
        for a in range(a0, 3):
            out.append((("host", a), body_lo, body_hi, False))
            out.append((("hf", s), a * ME + body_lo - ext_lo, a * ME + ext_hi - ext_lo, True))
    elif kind == "CARRY":
        pb = blocks[op["block"] - 1]
        sp = (g - 1) % L
        for a in range(a0, 3):
            out.append((("hf", sp), a * ME + c_lo - pb[2], a * ME + c_hi - pb[2], False))
            out.append((("hf", s), a * ME + c_lo - ext_lo, a * ME + c_hi - ext_lo, True))
    elif kind == "DECODE":
        for a in range(3):
            if a >= a0:
                out.append((("hf", s), a * ME, a * ME + E, False))
            out.append((("ws", w, a), 0, E, True))
    elif kind == "STEP":
        st = op["arg"]
        lo = 0 if ext_lo == -R else ext_lo + st * R
        hi = geo["nz"] if ext_hi == geo["nz"] + R else ext_hi - st * R
        up = 1 if st % 2 else 2
        for a in (0, 3 - up):
            out.append((("ws", w, a), lo - R - ext_lo, hi + R - ext_lo, False))
        out.append((("ws", w, up), lo - ext_lo, hi - ext_lo, True))
        if st == 1 and geo.get("fuse_decode"):
            # OOCS_FLAG_FUSE_DECODE: the first step reads p_{t-1} from its compressed records in the staging
            # buffer (the decode then writes only p_{t-1}'s ring, still modelled as the whole array)
            out.append((("hf", s), ME, ME + E, False))
    elif kind == "ENCODE":
        for a in (1, 2):
            out.append((("ws", w, a), own_lo - ext_lo, own_hi - ext_lo, False))
        for j in range(2):
            out.append((("hf", s), j * MO, j * MO + own_hi - own_lo, True))
    elif kind == "D2H":
        for j in range(2):
            out.append((("hf", s), j * MO, j * MO + own_hi - own_lo, False))
            out.append((("host", 1 + j), own_lo, own_hi, True))
    elif kind == "SEND":  # multi-GPU: reads edge planes of the encoded output (peer side: device flags)
        for j in range(2):
            out.append((("hf", s), j * MO, j * MO + own_hi - own_lo, False))
    return out


def happens_before(ops):
    """Return (nodes, reach) where reach[i] is a bitmask of nodes j that happen after node i."""
    n = len(ops)
    succ = [set() for _ in range(n)]
    last_on_lane = {}
    last_record = {}
    for i, op in enumerate(ops):
        l = op["lane"]
        if l in last_on_lane:
            succ[last_on_lane[l]].add(i)
        last_on_lane[l] = i
        if op["kind"] == "RECORD":
            last_record[(op["ev"], op["ev_g"])] = i
        elif op["kind"] == "WAIT":
            key = (op["ev"], op["ev_g"])
            if key in last_record:  # waiting on a never-recorded event is a no-op (CUDA semantics)
                succ[last_record[key]].add(i)
    reach = [0] * n
    for i in range(n - 1, -1, -1):  # ops only point forward in list order
        m = 0
        for j in succ[i]:
            m |= (1 << j) | reach[j]
        reach[i] = m
    return reach


def violations(ops, blocks, geo, limit=50):
    reach = happens_before(ops)
    fps = [footprint(op, blocks, geo) if op["kind"] not in ("WAIT", "RECORD") else [] for op in ops]
    bad = []
    idx = [i for i, f in enumerate(fps) if f]
    for ii, i in enumerate(idx):
        for j in idx[ii + 1:]:
            if (reach[i] >> j) & 1:
                continue
            for (ra, lo_a, hi_a, wa) in fps[i]:
                hit = False
                for (rb, lo_b, hi_b, wb) in fps[j]:
                    if ra == rb and (wa or wb) and lo_a < hi_b and lo_b < hi_a:
                        bad.append((i, j, ra))
                        hit = True
                        break
                if hit:
                    break
            if len(bad) >= limit:
                return bad
    return bad
