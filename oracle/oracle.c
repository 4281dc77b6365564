/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path of
 * arXiv 2204.11315 ("Compression-Based Optimizations for Out-of-Core GPU
 * Stencil Computation") computes.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2204_11315_b200/ (neither includes nor links the other).
 *
 * Citation convention: "P:L<n>" = /root/reference/PAPER.md line n (section),
 * "S:L<n>" = SPEC.md line n (module.op).  Readings of the paper where it is
 * silent are listed in DESIGN.md §3 (Q-numbers follow SURVEY.md §8(c)).
 *
 * Contents (each pinned by tests/test_oracle_*.py, -m "not gpu"):
 *   oracle_coeffs            8th-order central-difference weights (Q1)
 *   oracle_step              one leapfrog step of the 25-point acoustic wave
 *                            stencil over a plane range, fp64 arithmetic,
 *                            fp32 storage ("25-point stencil ... acoustic
 *                            wave propagation")
 *   oracle_step7             the same step with the 2nd-order 7-point Laplacian (STAR7,
 *                            small exact tests); oracle_step_s / _incore_s /
 *                            _pipeline_s take the stencil (0 = 25-point, 1 = STAR7)
 *   oracle_incore            T plain steps over the whole interior
 *   oracle_bq_encode_block / oracle_bq_decode_block
 *                            fixed-rate BlockQuant codec on one 4x4x4 block
 *                            (the codec SPEC.md fixes, S:L182, S:L196-219,
 *                            S:L242-244, adapted to fp32 -- DESIGN.md §3 Q11-Q14)
 *   oracle_encode_planes / oracle_decode_planes
 *                            array-level codec over whole 4-plane slabs
 *                            (identity, BlockQuant, ZFP, Truncate-16), slab-major block order
 *   oracle_tr16_encode / oracle_tr16_decode
 *                            Truncate-16: fp32 -> bfloat16 round-to-nearest-even
 *   oracle_plan              z-chunk decomposition with temporal-blocking halo
 *                            and region-sharing overlap (§3.1)
 *   oracle_pipeline          the out-of-core method, step by step in the
 *                            paper's order: for every sweep, for every chunk:
 *                            decompress its extended extent, k temporally
 *                            blocked steps, compress the owned planes
 *                            (Alg. 1)
 *
 * Floating point: IEEE binary32/binary64, round-to-nearest-even, no FMA
 * contraction (built with -ffp-contract=off), no flush-to-zero.  fmaf() is
 * the C99 correctly-rounded fused multiply-add.
 *
 *   oracle_zfp_*             NEXT-1: the ZFP fixed-rate codec (cuZFP's algorithm,
 *                            P:L116), codec 2 in the array-level calls
 *                            and the pipeline (the codec argument `q` is the rate)
 *
 * Everything here is pinned; see DESIGN.md §5 for the pin list.  Nothing is
 * "parity unpinned" except what DESIGN.md names (ZFP bitstream compatibility
 * with the zfp library itself).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Host threads for the OpenMP plane loops (timing only: results do not depend on it, every
 * parallel loop writes disjoint planes). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

#define R 4 /* stencil radius: 25-point star = centre + 3 axes x 2 sides x 4 (Table 1 HALO=4) */

/* Status codes (mirror the SPEC exit-code table S:L641 plus a data error S:L200). */
#define ORACLE_OK 0
#define ORACLE_ERR_CONFIG 2
#define ORACLE_ERR_DATA 6

/* ------------------------------------------------------------------ */
/* Stencil                                                            */
/* ------------------------------------------------------------------ */

/* Central-difference weights of d^2/dx^2 with accuracy order 8, unit spacing:
 *   f''(x) ~ c0 f(x) + sum_{m=1..4} c_m (f(x+m) + f(x-m)).
 * The paper gives no formula; SPEC adopts the standard 8th-order
 * scheme.  Values are the exact rationals of the order-8 system. */
void oracle_coeffs(double c[5]) {
    c[0] = -205.0 / 72.0;
    c[1] = 8.0 / 5.0;
    c[2] = -1.0 / 5.0;
    c[3] = 8.0 / 315.0;
    c[4] = -1.0 / 560.0;
}

/* One leapfrog step:
 *   p_next = 2 p_curr - p_prev + v^2 dt^2 Lap25(p_curr),
 *   Lap25  = sum over axes x,y,z of [c0 f0 + sum_m c_m (f(+m) + f(-m))], h = 1.
 * Arrays are (planes, ay, ax), x fastest, allocated layout with an R-cell
 * halo on the x and y faces.  Updates interior x in [R, ax-R), y in [R, ay-R)
 * for buffer planes z in [z_lo, z_hi); the result overwrites p_prev
 * (pointwise, so in place is exact).  Arithmetic in binary64, stored as
 * binary32 (one rounding per cell per step). */
void oracle_step(int64_t ax, int64_t ay, int64_t planes, const float *vel,
                 float *p_prev, const float *p_curr, float dt, int64_t z_lo,
                 int64_t z_hi) {
    double c[5];
    oracle_coeffs(c);
    const int64_t sy = ax, sz = ax * ay;
    (void)planes;
#pragma omp parallel for schedule(static)
    for (int64_t z = z_lo; z < z_hi; ++z) {
        for (int64_t y = R; y < ay - R; ++y) {
            for (int64_t x = R; x < ax - R; ++x) {
                const int64_t i = z * sz + y * sy + x;
                const double f0 = p_curr[i];
                double lap = 0.0;
                /* x axis */
                lap += c[0] * f0;
                for (int m = 1; m <= R; ++m)
                    lap += c[m] * ((double)p_curr[i + m] + (double)p_curr[i - m]);
                /* y axis */
                lap += c[0] * f0;
                for (int m = 1; m <= R; ++m)
                    lap += c[m] * ((double)p_curr[i + m * sy] + (double)p_curr[i - m * sy]);
                /* z axis */
                lap += c[0] * f0;
                for (int m = 1; m <= R; ++m)
                    lap += c[m] * ((double)p_curr[i + m * sz] + (double)p_curr[i - m * sz]);
                const double v = vel[i];
                const double vdt = v * (double)dt;
                const double next = 2.0 * f0 - (double)p_prev[i] + vdt * vdt * lap;
                p_prev[i] = (float)next;
            }
        }
    }
}

/* STAR7 (oocs.h OOCS_STENCIL_STAR7, SURVEY §8(b) "STAR7 (R=1) for small exact tests"): the same leapfrog
 * with the textbook 2nd-order 7-point Laplacian,
 *   Lap7 = sum over axes x,y,z of [f(+1) + f(-1) - 2 f0],  h = 1,
 * on the same allocated layout (R = 4 halo; only the first halo cell is read).  Binary64 arithmetic,
 * stored as binary32. */
void oracle_step7(int64_t ax, int64_t ay, int64_t planes, const float *vel, float *p_prev,
                  const float *p_curr, float dt, int64_t z_lo, int64_t z_hi) {
    const int64_t sy = ax, sz = ax * ay;
    (void)planes;
#pragma omp parallel for schedule(static)
    for (int64_t z = z_lo; z < z_hi; ++z) {
        for (int64_t y = R; y < ay - R; ++y) {
            for (int64_t x = R; x < ax - R; ++x) {
                const int64_t i = z * sz + y * sy + x;
                const double f0 = p_curr[i];
                double lap = 0.0;
                lap += (double)p_curr[i + 1] + (double)p_curr[i - 1] - 2.0 * f0;
                lap += (double)p_curr[i + sy] + (double)p_curr[i - sy] - 2.0 * f0;
                lap += (double)p_curr[i + sz] + (double)p_curr[i - sz] - 2.0 * f0;
                const double vdt = (double)vel[i] * (double)dt;
                p_prev[i] = (float)(2.0 * f0 - (double)p_prev[i] + vdt * vdt * lap);
            }
        }
    }
}

/* stencil 0 = the 25-point acoustic stencil (oracle_step), 1 = STAR7 (oracle_step7) */
void oracle_step_s(int stencil, int64_t ax, int64_t ay, int64_t planes, const float *vel,
                   float *p_prev, const float *p_curr, float dt, int64_t z_lo, int64_t z_hi) {
    if (stencil == 1)
        oracle_step7(ax, ay, planes, vel, p_prev, p_curr, dt, z_lo, z_hi);
    else
        oracle_step(ax, ay, planes, vel, p_prev, p_curr, dt, z_lo, z_hi);
}

/* T plain steps over the whole interior.  Dirichlet boundary:
 * the R-cell halo on all six faces keeps its initial values.
 * On return p_prev holds time level T-1 and p_curr level T. */
void oracle_incore_s(int stencil, int64_t ax, int64_t ay, int64_t az, const float *vel,
                     float *p_prev, float *p_curr, float dt, int64_t steps) {
    float *a = p_prev, *b = p_curr; /* a = level t-1, b = level t */
    for (int64_t t = 0; t < steps; ++t) {
        oracle_step_s(stencil, ax, ay, az, vel, a, b, dt, R, az - R); /* a <- level t+1 */
        float *tmp = a;
        a = b;
        b = tmp;
    }
    if (a != p_prev) { /* odd number of steps: roles are swapped */
        const size_t n = (size_t)(ax * ay * az);
        float *tmp = (float *)malloc(n * sizeof(float));
        memcpy(tmp, a, n * sizeof(float));
        memcpy(p_curr, b, n * sizeof(float));
        memcpy(p_prev, tmp, n * sizeof(float));
        free(tmp);
    }
}

void oracle_incore(int64_t ax, int64_t ay, int64_t az, const float *vel,
                   float *p_prev, float *p_curr, float dt, int64_t steps) {
    oracle_incore_s(0, ax, ay, az, vel, p_prev, p_curr, dt, steps);
}

/* ------------------------------------------------------------------ */
/* BlockQuant fixed-rate codec (fp32)                                 */
/* ------------------------------------------------------------------ */
/* Block record, 8(q+1) bytes, rate r = q+1 bits/value (Q13):
 *   [mn: f32 LE][mx: f32 LE][P_{q-1}: u64 LE] ... [P_0: u64 LE]
 * P_b bit j = bit b of code_j, j = xi + 4 yi + 16 zi (x fastest).
 * Quantiser (Q12): canonicalise -0 -> +0; mn/mx = block min/max;
 *   range = fl(mx - mn); step = fl(range * 2^-q);
 *   if step < FLT_MIN: every code 0
 *   else scale = fl(2^q / range), code = min(2^q - 1, floor(fl(fl(x - mn) * scale)))
 * Reconstruction: x^ = fmaf((float)code + 0.5f, step, mn)  (bin centres).
 * Rejects NaN/Inf and |x| >= 2^126. */

static int bq_reject(float x) { return !isfinite(x) || fabsf(x) >= 0x1p126f; }

int oracle_bq_encode_block(const float *x_in, int q, uint8_t *rec) {
    float x[64];
    for (int j = 0; j < 64; ++j) {
        if (bq_reject(x_in[j])) return ORACLE_ERR_DATA;
        x[j] = x_in[j] + 0.0f; /* -0 -> +0 */
    }
    float mn = x[0], mx = x[0];
    for (int j = 1; j < 64; ++j) {
        if (x[j] < mn) mn = x[j];
        if (x[j] > mx) mx = x[j];
    }
    const float range = mx - mn;
    const float step = range * ldexpf(1.0f, -q);
    uint32_t code[64];
    if (step < 0x1p-126f) {
        for (int j = 0; j < 64; ++j) code[j] = 0;
    } else {
        const float scale = ldexpf(1.0f, q) / range;
        const uint32_t cmax = (1u << q) - 1u;
        for (int j = 0; j < 64; ++j) {
            const float a = x[j] - mn;
            const float t = a * scale;
            uint32_t cj = (uint32_t)floorf(t);
            code[j] = cj > cmax ? cmax : cj;
        }
    }
    memcpy(rec, &mn, 4);
    memcpy(rec + 4, &mx, 4);
    for (int b = q - 1; b >= 0; --b) {
        uint64_t plane = 0;
        for (int j = 0; j < 64; ++j) plane |= (uint64_t)((code[j] >> b) & 1u) << j;
        uint8_t *dst = rec + 8 + 8 * (q - 1 - b);
        for (int byte = 0; byte < 8; ++byte) dst[byte] = (uint8_t)(plane >> (8 * byte));
    }
    return ORACLE_OK;
}

void oracle_bq_decode_block(const uint8_t *rec, int q, float *x) {
    float mn, mx;
    memcpy(&mn, rec, 4);
    memcpy(&mx, rec + 4, 4);
    const float range = mx - mn;
    const float step = range * ldexpf(1.0f, -q);
    uint32_t code[64];
    for (int j = 0; j < 64; ++j) code[j] = 0;
    for (int b = q - 1; b >= 0; --b) {
        const uint8_t *src = rec + 8 + 8 * (q - 1 - b);
        uint64_t plane = 0;
        for (int byte = 0; byte < 8; ++byte) plane |= (uint64_t)src[byte] << (8 * byte);
        for (int j = 0; j < 64; ++j) code[j] |= (uint32_t)((plane >> j) & 1u) << b;
    }
    for (int j = 0; j < 64; ++j) x[j] = fmaf((float)code[j] + 0.5f, step, mn);
}

int oracle_zfp_encode_planes(int64_t ax, int64_t ay, int64_t planes, const float *src, int rate, uint8_t *dst);

/* Truncate-16 (SURVEY.md §8(b) codec enum, §8(c) C-3 "Truncate-16: fp32 -> bf16 RNE (the upper 16 bits
 * after RNE rounding; NaN -> quiet NaN)").  Written out on the bit pattern: bfloat16 keeps the sign,
 * the 8 exponent bits and the top 7 fraction bits of binary32, so rounding to nearest-even is adding
 * half an ulp of the kept part (0x7FFF, plus the kept lsb to break ties towards even) to the 32-bit
 * pattern and keeping the upper half; a carry out of the fraction correctly bumps the exponent (up to
 * Inf).  NaN becomes 0x7FC0, the canonical quiet NaN (torch's convention).  Decoding appends 16 zero
 * bits, which is exact. */
uint16_t oracle_tr16_encode(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if (x != x) return 0x7FC0u;
    const uint32_t lsb = (u >> 16) & 1u;
    return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

float oracle_tr16_decode(uint16_t h) {
    const uint32_t u = (uint32_t)h << 16;
    float x;
    memcpy(&x, &u, 4);
    return x;
}
void oracle_zfp_decode_planes(int64_t ax, int64_t ay, int64_t planes, const uint8_t *src, int rate, float *dst);

/* Bytes of one compressed plane-slab-row: an allocated xy plane of ax*ay
 * values costs ax*ay*rate_bits/8 bytes; identity (codec 0) costs 4 B/value. */
int64_t oracle_plane_bytes(int64_t ax, int64_t ay, int codec, int q) {
    if (codec == 0) return ax * ay * 4;
    if (codec == 3) return ax * ay * 2; /* Truncate-16: q unused (rate 16) */
    if (codec == 2) return (ax / 4) * (ay / 4) * 8 * q / 4; /* ZFP: q is the rate (bits/value) */
    return (ax / 4) * (ay / 4) * 8 * (q + 1) / 4;
}

/* Array-level codec over `planes` allocated planes (a multiple of 4), source
 * laid out (planes, ay, ax).  Blocks ordered slab (z/4) major, then y/4, then
 * x/4, so any 4-aligned plane range is one contiguous byte range -- which is
 * what makes the overlap area independently decodable ("we compress
 * the overlapped area of a chunk separately").  codec 0 = identity (raw fp32
 * bytes), 1 = BlockQuant with q = rate_bits - 1. */
int oracle_encode_planes(int64_t ax, int64_t ay, int64_t planes, const float *src,
                         int codec, int q, uint8_t *dst) {
    if (codec == 0) {
        memcpy(dst, src, (size_t)(ax * ay * planes) * 4);
        return ORACLE_OK;
    }
    if (codec == 3) { /* raw bf16 planes, x fastest, little-endian */
        for (int64_t i = 0; i < ax * ay * planes; ++i) {
            const uint16_t h = oracle_tr16_encode(src[i]);
            dst[2 * i] = (uint8_t)(h & 0xFFu);
            dst[2 * i + 1] = (uint8_t)(h >> 8);
        }
        return ORACLE_OK;
    }
    if (codec == 2) return oracle_zfp_encode_planes(ax, ay, planes, src, q, dst);
    if (ax % 4 || ay % 4 || planes % 4) return ORACLE_ERR_CONFIG;
    const int64_t nbx = ax / 4, nby = ay / 4, nbz = planes / 4;
    const int64_t rec_bytes = 8 * (q + 1);
    int err = ORACLE_OK;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (int64_t bz = 0; bz < nbz; ++bz) {
        float blk[64];
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                for (int zi = 0; zi < 4; ++zi)
                    for (int yi = 0; yi < 4; ++yi)
                        for (int xi = 0; xi < 4; ++xi)
                            blk[xi + 4 * yi + 16 * zi] =
                                src[((4 * bz + zi) * ay + 4 * by + yi) * ax + 4 * bx + xi];
                uint8_t *rec = dst + ((bz * nby + by) * nbx + bx) * rec_bytes;
                err |= oracle_bq_encode_block(blk, q, rec);
            }
    }
    return err ? ORACLE_ERR_DATA : ORACLE_OK;
}

void oracle_decode_planes(int64_t ax, int64_t ay, int64_t planes, const uint8_t *src,
                          int codec, int q, float *dst) {
    if (codec == 0) {
        memcpy(dst, src, (size_t)(ax * ay * planes) * 4);
        return;
    }
    if (codec == 3) {
        for (int64_t i = 0; i < ax * ay * planes; ++i)
            dst[i] = oracle_tr16_decode((uint16_t)(src[2 * i] | (src[2 * i + 1] << 8)));
        return;
    }
    if (codec == 2) {
        oracle_zfp_decode_planes(ax, ay, planes, src, q, dst);
        return;
    }
    const int64_t nbx = ax / 4, nby = ay / 4, nbz = planes / 4;
    const int64_t rec_bytes = 8 * (q + 1);
#pragma omp parallel for schedule(static)
    for (int64_t bz = 0; bz < nbz; ++bz) {
        float blk[64];
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                oracle_bq_decode_block(src + ((bz * nby + by) * nbx + bx) * rec_bytes, q, blk);
                for (int zi = 0; zi < 4; ++zi)
                    for (int yi = 0; yi < 4; ++yi)
                        for (int xi = 0; xi < 4; ++xi)
                            dst[((4 * bz + zi) * ay + 4 * by + yi) * ax + 4 * bx + xi] =
                                blk[xi + 4 * yi + 16 * zi];
            }
    }
}

/* ------------------------------------------------------------------ */
/* Decomposition                                                      */
/* ------------------------------------------------------------------ */
/* Chunk i of n over interior planes [0, nz) ("decomposes the original
 * data into smaller data chunks").  Owned intervals partition
 * [0, nz) in 4-plane units, the remainder going to leading chunks (Q5).
 * Temporal blocking piggybacks k*R halo planes per side, clamped at
 * the physical boundary [-R, nz+R).  With region sharing chunk i>0
 * finds carry_i = ext_{i-1} ∩ ext_i already on the device and transfers only
 * body_i = ext_i \ carry_i.
 * out[i*8 + 0..7] = own_lo, own_hi, ext_lo, ext_hi, carry_lo, carry_hi,
 *                   body_lo, body_hi (interior plane coordinates). */
int oracle_plan(int64_t nz, int64_t n, int64_t k, int sharing, int64_t *out) {
    if (n < 1 || k < 1 || nz % 4 || nz / 4 < n) return ORACLE_ERR_CONFIG;
    const int64_t units = nz / 4, base = units / n, rem = units % n;
    int64_t lo = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t w = 4 * (base + (i < rem ? 1 : 0));
        if (k * R >= w) return ORACLE_ERR_CONFIG; /* halo would span a non-neighbour */
        const int64_t own_lo = lo, own_hi = lo + w;
        int64_t ext_lo = own_lo - k * R, ext_hi = own_hi + k * R;
        if (ext_lo < -R) ext_lo = -R;
        if (ext_hi > nz + R) ext_hi = nz + R;
        int64_t *o = out + 8 * i;
        o[0] = own_lo;
        o[1] = own_hi;
        o[2] = ext_lo;
        o[3] = ext_hi;
        if (i > 0 && sharing) {
            o[4] = own_lo - k * R; /* = ext_i lo; ext_{i-1} reaches own_lo + kR */
            o[5] = own_lo + k * R;
            o[6] = o[5];
        } else {
            o[4] = o[5] = ext_lo;
            o[6] = ext_lo;
        }
        o[7] = ext_hi;
        lo = own_hi;
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* The out-of-core method                                             */
/* ------------------------------------------------------------------ */
/* Stores hold the whole allocated grid (az = nz + 2R planes of ax*ay values)
 * compressed slab by slab (oracle_encode_planes layout).  One sweep advances
 * the domain by k steps: for every chunk i, decompress ext_i of the velocity
 * and of both pressure time levels from S_t ("Decompress data in
 * hf_buf[si] to fl_buf"), apply k leapfrog steps on the shrinking trapezoid
 * ("Compute on data in fl_buf"), compress the owned planes of
 * the two read-write datasets into S_{t+1} (P:L155 write-back to
 * chk).  The velocity is read-only and never re-compressed.  The
 * oracle double-buffers S (reads S_t, writes S_{t+1}) so chunk order does not
 * matter; boundary planes [-R,0) and [nz,nz+R) are never written (Dirichlet,
 * S:L102).  Region sharing only changes which bytes cross PCIe, not values,
 * so the oracle has no notion of it.
 * steps must be a multiple of k.  Returns ORACLE_OK or an error. */
int oracle_pipeline_s(int stencil, int64_t ax, int64_t ay, int64_t nz, int64_t n, int64_t k,
                      float dt, int64_t steps, int codec, int q, const uint8_t *S_vel,
                      uint8_t *S_prev, uint8_t *S_curr) {
    if (k < 1 || steps % k) return ORACLE_ERR_CONFIG;
    int64_t *plan = (int64_t *)malloc((size_t)n * 8 * sizeof(int64_t));
    int rc = oracle_plan(nz, n, k, 1, plan);
    if (rc) {
        free(plan);
        return rc;
    }
    const int64_t az = nz + 2 * R;
    const int64_t pb = oracle_plane_bytes(ax, ay, codec, q); /* bytes per plane */
    const size_t store_bytes = (size_t)(pb * az);
    uint8_t *N_prev = (uint8_t *)malloc(store_bytes), *N_curr = (uint8_t *)malloc(store_bytes);
    int64_t max_ext = 0;
    for (int64_t i = 0; i < n; ++i)
        if (plan[8 * i + 3] - plan[8 * i + 2] > max_ext) max_ext = plan[8 * i + 3] - plan[8 * i + 2];
    const size_t buf_vals = (size_t)(ax * ay * max_ext);
    float *v = (float *)malloc(buf_vals * 4), *pa = (float *)malloc(buf_vals * 4),
          *pbuf = (float *)malloc(buf_vals * 4);
    for (int64_t sweep = 0; sweep < steps / k && rc == ORACLE_OK; ++sweep) {
        memcpy(N_prev, S_prev, store_bytes); /* boundary planes carried over bytewise */
        memcpy(N_curr, S_curr, store_bytes);
        for (int64_t i = 0; i < n && rc == ORACLE_OK; ++i) {
            const int64_t own_lo = plan[8 * i], own_hi = plan[8 * i + 1];
            const int64_t ext_lo = plan[8 * i + 2], ext_hi = plan[8 * i + 3];
            const int64_t E = ext_hi - ext_lo;
            const int64_t a0 = ext_lo + R; /* allocated plane index of buffer plane 0 */
            oracle_decode_planes(ax, ay, E, S_vel + a0 * pb, codec, q, v);
            oracle_decode_planes(ax, ay, E, S_prev + a0 * pb, codec, q, pa);
            oracle_decode_planes(ax, ay, E, S_curr + a0 * pb, codec, q, pbuf);
            float *prev = pa, *curr = pbuf;
            for (int64_t s = 1; s <= k; ++s) {
                /* step s is valid on [lo_s, hi_s): the halo shrinks by R per step
                 * except at the physical boundary (Fig. 1(b)) */
                const int64_t lo = (ext_lo == -R) ? 0 : ext_lo + s * R;
                const int64_t hi = (ext_hi == nz + R) ? nz : ext_hi - s * R;
                oracle_step_s(stencil, ax, ay, E, v, prev, curr, dt, lo - ext_lo, hi - ext_lo);
                float *t = prev;
                prev = curr;
                curr = t;
            }
            const int64_t ob = own_lo - ext_lo, W = own_hi - own_lo;
            rc = oracle_encode_planes(ax, ay, W, prev + ob * ax * ay, codec, q,
                                      N_prev + (own_lo + R) * pb);
            if (rc == ORACLE_OK)
                rc = oracle_encode_planes(ax, ay, W, curr + ob * ax * ay, codec, q,
                                          N_curr + (own_lo + R) * pb);
        }
        memcpy(S_prev, N_prev, store_bytes);
        memcpy(S_curr, N_curr, store_bytes);
    }
    free(v);
    free(pa);
    free(pbuf);
    free(N_prev);
    free(N_curr);
    free(plan);
    return rc;
}

int oracle_pipeline(int64_t ax, int64_t ay, int64_t nz, int64_t n, int64_t k, float dt,
                    int64_t steps, int codec, int q, const uint8_t *S_vel, uint8_t *S_prev,
                    uint8_t *S_curr) {
    return oracle_pipeline_s(0, ax, ay, nz, n, k, dt, steps, codec, q, S_vel, S_prev, S_curr);
}

/* ------------------------------------------------------------------ */
/* ZFP fixed-rate codec (NEXT-1): the algorithm of zfp 0.5.5 as used by  */
/* cuZFP, 3-D float blocks, written out step by step:  */
/*   1. block-floating-point: common exponent emax of the 64 values,     */
/*      values scaled to 30-bit signed integers (truncation);            */
/*   2. decorrelating transform: integer lifting along x, then y, then z;*/
/*   3. reorder by total sequency, map to negabinary;                    */
/*   4. embedded coding of bit planes, MSB first, with group testing,    */
/*      truncated at maxbits = 64 * rate bits (fixed rate).              */
/* Record = maxbits bits, written LSB-first into 64-bit words.           */
/* Bitstream compatibility with the zfp library itself is parity         */
/* unpinned (no zfp in this environment); the pins are the transform's   */
/* documented matrices, the embedded-prefix property, exact cases and   */
/* error behaviour (tests/test_oracle_zfp.py).                          */
/* ------------------------------------------------------------------ */

#define ZFP_EBITS 8
#define ZFP_EBIAS 127
#define ZFP_NBMASK 0xaaaaaaaau

typedef struct {
    uint64_t *w; /* words */
    int64_t pos; /* bit position */
} oracle_bits;

static void zb_put(oracle_bits *s, uint64_t bit) {
    if (bit & 1u) s->w[s->pos >> 6] |= (uint64_t)1 << (s->pos & 63);
    s->pos++;
}
static uint64_t zb_get(oracle_bits *s) {
    uint64_t b = (s->w[s->pos >> 6] >> (s->pos & 63)) & 1u;
    s->pos++;
    return b;
}

/* sequency order of the 64 coefficients of a 4x4x4 block: coefficient (i, j, k) of the
 * transform sits at i + 4j + 16k; listed by non-decreasing total sequency i + j + k, in zfp's
 * order (perm_3) */
#define ZI(i, j, k) ((i) + 4 * (j) + 16 * (k))
const unsigned char zfp_perm3[64] = {
    ZI(0,0,0), ZI(1,0,0), ZI(0,1,0), ZI(0,0,1), ZI(0,1,1), ZI(1,0,1),
    ZI(1,1,0), ZI(2,0,0), ZI(0,2,0), ZI(0,0,2), ZI(1,1,1), ZI(2,1,0),
    ZI(2,0,1), ZI(0,2,1), ZI(1,2,0), ZI(1,0,2), ZI(0,1,2), ZI(3,0,0),
    ZI(0,3,0), ZI(0,0,3), ZI(2,1,1), ZI(1,2,1), ZI(1,1,2), ZI(0,2,2),
    ZI(2,0,2), ZI(2,2,0), ZI(3,1,0), ZI(3,0,1), ZI(0,3,1), ZI(1,3,0),
    ZI(1,0,3), ZI(0,1,3), ZI(1,2,2), ZI(2,1,2), ZI(2,2,1), ZI(3,1,1),
    ZI(1,3,1), ZI(1,1,3), ZI(3,2,0), ZI(3,0,2), ZI(0,3,2), ZI(2,3,0),
    ZI(2,0,3), ZI(0,2,3), ZI(2,2,2), ZI(3,2,1), ZI(3,1,2), ZI(1,3,2),
    ZI(2,3,1), ZI(2,1,3), ZI(1,2,3), ZI(0,3,3), ZI(3,0,3), ZI(3,3,0),
    ZI(3,2,2), ZI(2,3,2), ZI(2,2,3), ZI(1,3,3), ZI(3,1,3), ZI(3,3,1),
    ZI(2,3,3), ZI(3,2,3), ZI(3,3,2), ZI(3,3,3),
};
#undef ZI

/* forward lifting of 4 values p[0], p[s], p[2s], p[3s] (zfp fwd_lift):
 *          ( 4  4  4  4)
 *   1/16 * ( 5  1 -1 -5)
 *          (-4  4  4 -4)
 *          (-2  6 -6  2)   (exact when no shift drops bits) */
void oracle_zfp_fwd_lift(int32_t *p, int s) {
    int32_t x = p[0], y = p[s], z = p[2 * s], w = p[3 * s];
    x += w; x >>= 1; w -= x;
    z += y; z >>= 1; y -= z;
    x += z; x >>= 1; z -= x;
    w += y; w >>= 1; y -= w;
    w += y >> 1; y -= w >> 1;
    p[0] = x; p[s] = y; p[2 * s] = z; p[3 * s] = w;
}

/* inverse lifting (zfp inv_lift):
 *         ( 4  6 -4 -1)
 *   1/4 * ( 4  2  4  5)
 *         ( 4 -2  4 -5)
 *         ( 4 -6 -4  1) */
void oracle_zfp_inv_lift(int32_t *p, int s) {
    int32_t x = p[0], y = p[s], z = p[2 * s], w = p[3 * s];
    y += w >> 1; w -= y >> 1;
    y += w; w <<= 1; w -= y;
    z += x; x <<= 1; x -= z;
    y += z; z <<= 1; z -= y;
    w += x; x <<= 1; x -= w;
    p[0] = x; p[s] = y; p[2 * s] = z; p[3 * s] = w;
}

void oracle_zfp_fwd_xform(int32_t *b) {
    for (int z = 0; z < 4; z++)
        for (int y = 0; y < 4; y++) oracle_zfp_fwd_lift(b + 4 * y + 16 * z, 1);
    for (int x = 0; x < 4; x++)
        for (int z = 0; z < 4; z++) oracle_zfp_fwd_lift(b + 16 * z + x, 4);
    for (int y = 0; y < 4; y++)
        for (int x = 0; x < 4; x++) oracle_zfp_fwd_lift(b + x + 4 * y, 16);
}

void oracle_zfp_inv_xform(int32_t *b) {
    for (int y = 0; y < 4; y++)
        for (int x = 0; x < 4; x++) oracle_zfp_inv_lift(b + x + 4 * y, 16);
    for (int x = 0; x < 4; x++)
        for (int z = 0; z < 4; z++) oracle_zfp_inv_lift(b + 16 * z + x, 4);
    for (int z = 0; z < 4; z++)
        for (int y = 0; y < 4; y++) oracle_zfp_inv_lift(b + 4 * y + 16 * z, 1);
}

uint32_t oracle_zfp_int2uint(int32_t x) { return ((uint32_t)x + ZFP_NBMASK) ^ ZFP_NBMASK; }
int32_t oracle_zfp_uint2int(uint32_t x) { return (int32_t)((x ^ ZFP_NBMASK) - ZFP_NBMASK); }

/* exponent of x >= 0 as frexp gives it, clamped for denormals; -EBIAS for 0 */
static int zfp_exponent(float x) {
    if (x > 0) {
        int e;
        frexpf(x, &e);
        return e > 1 - ZFP_EBIAS ? e : 1 - ZFP_EBIAS;
    }
    return -ZFP_EBIAS;
}

/* encode one block of 64 floats (j = xi + 4 yi + 16 zi) into maxbits = 64*rate bits
 * (the record must be zeroed by the caller).  Returns ORACLE_ERR_DATA on NaN/Inf. */
int oracle_zfp_encode_block(const float *x, int rate, uint64_t *rec) {
    const int maxbits = 64 * rate;
    float amax = 0;
    for (int j = 0; j < 64; ++j) {
        if (!isfinite(x[j])) return ORACLE_ERR_DATA;
        if (fabsf(x[j]) > amax) amax = fabsf(x[j]);
    }
    oracle_bits s = {rec, 0};
    const int emax = zfp_exponent(amax);
    const unsigned e = (unsigned)(emax + ZFP_EBIAS); /* fixed-rate: precision is never 0 for floats */
    if (!e) { /* all zeros: a single 0 bit, rest padding */
        zb_put(&s, 0);
        return ORACLE_OK;
    }
    /* 1. header: 2e+1 in 1 + EBITS bits (LSB = "nonzero block") */
    const uint64_t head = 2 * (uint64_t)e + 1;
    for (int i = 0; i < 1 + ZFP_EBITS; ++i) zb_put(&s, head >> i);
    /* block-floating-point: integer = (int)(x * 2^(30 - emax)), truncation toward zero */
    /* (zfp forms 2^(30-emax) in float, which overflows for emax < -97; in double the product is
     * exact and identical wherever zfp's is defined) */
    int32_t ib[64];
    const double scale = ldexp(1.0, 30 - emax);
    for (int j = 0; j < 64; ++j) ib[j] = (int32_t)(scale * (double)x[j]);
    /* 2. decorrelating transform */
    oracle_zfp_fwd_xform(ib);
    /* 3. sequency order + negabinary */
    uint32_t ub[64];
    for (int i = 0; i < 64; ++i) ub[i] = oracle_zfp_int2uint(ib[zfp_perm3[i]]);
    /* 4. embedded bit-plane coding with group tests (zfp encode_ints, kmin = 0) */
    unsigned bits = (unsigned)(maxbits - 1 - ZFP_EBITS);
    unsigned n = 0;
    for (int k = 32; bits && k-- > 0;) {
        uint64_t plane = 0;
        for (int i = 0; i < 64; ++i) plane += (uint64_t)((ub[i] >> k) & 1u) << i;
        /* the first n coefficients are already significant: their bits verbatim */
        unsigned m = n < bits ? n : bits;
        bits -= m;
        for (unsigned i = 0; i < m; ++i) zb_put(&s, plane >> i);
        plane = m == 64 ? 0 : plane >> m;
        /* unary run-length code of the remainder: group test, then the next 1 */
        for (; n < 64 && bits; plane >>= 1, n++) {
            bits--;
            zb_put(&s, plane != 0);
            if (!plane) break;
            for (; n < 63 && bits; plane >>= 1, n++) {
                bits--;
                zb_put(&s, plane & 1u);
                if (plane & 1u) break;
            }
        }
    }
    return ORACLE_OK;
}

void oracle_zfp_decode_block(const uint64_t *rec, int rate, float *x) {
    const int maxbits = 64 * rate;
    oracle_bits s = {(uint64_t *)rec, 0};
    if (!zb_get(&s)) {
        for (int j = 0; j < 64; ++j) x[j] = 0.0f;
        return;
    }
    unsigned e = 0;
    for (int i = 0; i < ZFP_EBITS; ++i) e |= (unsigned)zb_get(&s) << i;
    const int emax = (int)e - ZFP_EBIAS;
    uint32_t ub[64] = {0};
    unsigned bits = (unsigned)(maxbits - 1 - ZFP_EBITS);
    unsigned n = 0;
    for (int k = 32; bits && k-- > 0;) {
        unsigned m = n < bits ? n : bits;
        bits -= m;
        uint64_t plane = 0;
        for (unsigned i = 0; i < m; ++i) plane |= zb_get(&s) << i;
        for (; n < 64 && bits; ) {
            bits--;
            if (!zb_get(&s)) break;
            for (; n < 63 && bits; n++) {
                bits--;
                if (zb_get(&s)) break;
            }
            plane += (uint64_t)1 << n;
            n++;
        }
        for (int i = 0; i < 64; ++i) ub[i] += (uint32_t)((plane >> i) & 1u) << k;
    }
    int32_t ib[64];
    for (int i = 0; i < 64; ++i) ib[zfp_perm3[i]] = oracle_zfp_uint2int(ub[i]);
    oracle_zfp_inv_xform(ib);
    /* inverse block-floating-point: (float)int * 2^(emax-30) (zfp inv_cast; in double, exact) */
    const double scale = ldexp(1.0, emax - 30);
    for (int j = 0; j < 64; ++j) x[j] = (float)((double)(float)ib[j] * scale);
}

/* Array-level ZFP over whole 4-plane slabs, same slab-major block order as BlockQuant; each block
 * record is 64*rate bits = 8*rate bytes. */
int oracle_zfp_encode_planes(int64_t ax, int64_t ay, int64_t planes, const float *src, int rate, uint8_t *dst) {
    if (ax % 4 || ay % 4 || planes % 4 || rate < 1 || rate > 32) return ORACLE_ERR_CONFIG;
    const int64_t nbx = ax / 4, nby = ay / 4, nbz = planes / 4;
    const int64_t rec_bytes = 8 * rate;
    int err = ORACLE_OK;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (int64_t bz = 0; bz < nbz; ++bz) {
        float blk[64];
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                for (int zi = 0; zi < 4; ++zi)
                    for (int yi = 0; yi < 4; ++yi)
                        for (int xi = 0; xi < 4; ++xi)
                            blk[xi + 4 * yi + 16 * zi] = src[((4 * bz + zi) * ay + 4 * by + yi) * ax + 4 * bx + xi];
                uint64_t *rec = (uint64_t *)(dst + ((bz * nby + by) * nbx + bx) * rec_bytes);
                memset(rec, 0, (size_t)rec_bytes);
                err |= oracle_zfp_encode_block(blk, rate, rec);
            }
    }
    return err ? ORACLE_ERR_DATA : ORACLE_OK;
}

void oracle_zfp_decode_planes(int64_t ax, int64_t ay, int64_t planes, const uint8_t *src, int rate, float *dst) {
    const int64_t nbx = ax / 4, nby = ay / 4, nbz = planes / 4;
    const int64_t rec_bytes = 8 * rate;
#pragma omp parallel for schedule(static)
    for (int64_t bz = 0; bz < nbz; ++bz) {
        float blk[64];
        for (int64_t by = 0; by < nby; ++by)
            for (int64_t bx = 0; bx < nbx; ++bx) {
                oracle_zfp_decode_block((const uint64_t *)(src + ((bz * nby + by) * nbx + bx) * rec_bytes), rate, blk);
                for (int zi = 0; zi < 4; ++zi)
                    for (int yi = 0; yi < 4; ++yi)
                        for (int xi = 0; xi < 4; ++xi)
                            dst[((4 * bz + zi) * ay + 4 * by + yi) * ax + 4 * bx + xi] = blk[xi + 4 * yi + 16 * zi];
            }
    }
}
