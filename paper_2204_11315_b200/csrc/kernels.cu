// Hot-path kernels for sm_100a: fixed-rate BlockQuant decode/encode (P:L116,
// P:L153) and the 25-point acoustic-wave leapfrog step (P:L163,
// P:L212).  All three are HBM-bound streaming kernels (no dense contraction:
// tensor cores do not apply); see DESIGN.md §6 for their rooflines.
//
// Working-buffer layout (shared with runtime.cu): planes x ay rows x pitch
// floats, element x of a row at column x + XOFF (XOFF = 28) so interior x = R
// starts on a 128-byte line; pitch is a multiple of 32 floats.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cmath>

#include "oocs_internal.h"

namespace oocs {

// ---------------------------------------------------------------------------
// Warp-level 32x32 bit-matrix transpose: lane l holds row l (32 bits); on
// return lane m holds column m (bit l = bit m of row l).  Five butterfly
// stages, each one SHFL plus: for the 16- and 8-bit stages one byte permute
// (PRMT) with a lane-dependent selector, for the others a funnel rotate (SHF.W)
// by a lane-dependent amount and one LOP3 select -- the per-lane selectors,
// rotate amounts and masks are computed once per kernel.  This is the codec's "warp-level bit-plane
// packing": a block's 64 codes of <= 16 bits become its bit planes in one pass.
// ---------------------------------------------------------------------------
struct Xpose {
    uint32_t rot[5], keep[5];  // stages 2..4 (4-, 2-, 1-bit moves)
    uint32_t sel[2];           // stages 0, 1 (16- and 8-bit moves): one byte permute each
    __device__ __forceinline__ explicit Xpose(int lane) {
        // upper lanes keep their low half and take the partner's low half above it; lower lanes the
        // mirror image: [x0 x1 y0 y1] / [y2 y3 x2 x3] for 16 bits, [x0 y0 x2 y2] / [y1 x1 y3 x3] for 8
        sel[0] = (lane & 16) == 0 ? 0x5410u : 0x3276u;
        sel[1] = (lane & 8) == 0 ? 0x6240u : 0x3715u;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int j = 16 >> s;
            const uint32_t m = s == 0 ? 0x0000FFFFu : s == 1 ? 0x00FF00FFu : s == 2 ? 0x0F0F0F0Fu
                             : s == 3 ? 0x33333333u : 0x55555555u;
            const bool upper = (lane & j) == 0;
            rot[s] = upper ? (uint32_t)j : (uint32_t)(32 - j);  // rotl by j == <<j, by 32-j == >>j (masked)
            keep[s] = upper ? m : ~m;
        }
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16 >> s);
            if (s < 2) {
                x = __byte_perm(x, y, sel[s]);
                continue;
            }
            const uint32_t t = __funnelshift_l(y, y, rot[s]);
            // bitwise mux (keep ? x : t) in one LOP3: lut = (c & a) | (~c & b) = 0xE4
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x) : "r"(x), "r"(t), "r"(keep[s]));
        }
        return x;
    }
};

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// (float)code + 0.5f without the quarter-rate I2F: 2^23 + code is the bit pattern 0x4B000000 | code
// (code < 2^23), and subtracting 2^23 - 0.5 (representable) is exact (Sterbenz) -- bq_decode_kernel
// paired fp32 add rounded toward -inf (FADD2.RM)
__device__ __forceinline__ float2 fadd2_rd(float2 a, float2 b) {
    unsigned long long ua, ub, ur;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(ur) : "l"(ua), "l"(ub));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(ur));
    return r;
}

// three-input min / max that propagate NaN (FMNMX3.NAN, sm_100): a block's min and max are NaN iff one
// of its values is, so the encoder's NaN check rides on the statistics it needs anyway
__device__ __forceinline__ float min3n(float a, float b, float c) {
    float r;
    asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max3n(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float min2n(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float max2n(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// bin-centre patterns of the low / high 16-bit code of a packed word: bytes [c0 c1 00 4B] = 2^23 + code
__device__ __forceinline__ uint32_t pat_lo(uint32_t w) { return __byte_perm(w, 0x4B000000u, 0x7410); }
__device__ __forceinline__ uint32_t pat_hi(uint32_t w) { return __byte_perm(w, 0x4B000000u, 0x7432); }

// Warp task = one 128-byte line segment of 16 rows (4 y x 4 z) of a
// 4-plane slab: the blocks bx in [max(0,8L-7), min(nbx-1,8L)] whose columns
// lie in line L (column of x is x + 28, block bx covers x in [4bx, 4bx+4)).
// Grid: x = line L, y = group of 8 block rows (one per warp), z = slab.
struct LineTask {
    int bz, by, b0, nb;
};
// ring_nl > 0 (decode only): a compact grid over the x/y ring of the allocated grid -- x in [0, 2 nl):
// the first / last group of 8 block rows of every line, x in [2 nl, 2 nl + 2 ng): the first / last line of
// every group (corners twice, same values)
__device__ __forceinline__ LineTask line_task(int nbx, int bz, int grp, int ring_nl = 0, int ring_ng = 0) {
    LineTask t;
    int L = blockIdx.x;
    if (ring_nl) {
        int i = blockIdx.x;
        if (i < 2 * ring_nl) {
            grp = i < ring_nl ? 0 : ring_ng - 1;
            L = i < ring_nl ? i : i - ring_nl;
        } else {
            i -= 2 * ring_nl;
            L = i < ring_ng ? 0 : ring_nl - 1;
            grp = i < ring_ng ? i : i - ring_ng;
        }
    }
    t.by = grp * 8 + (threadIdx.x >> 5);
    t.bz = bz;
    t.b0 = L == 0 ? 0 : 8 * L - 7;
    const int b1 = min(nbx - 1, 8 * L);
    t.nb = b1 - t.b0 + 1;
    return t;
}

constexpr int CODEC_WARPS = 8;

// up to 3 arrays of one chunk in one launch (grid y = array * gy + row group, z = slab): one ramp and one tail
// per chunk instead of one per array
struct CodecArrays {
    const void *src[N_ARRAYS];
    void *dst[N_ARRAYS];
    int gy;                // grid y per array (groups of 8 block rows; 1 for the ring grid): y = array * gy + group
    int ring_nl, ring_ng;  // decode: > 0 = the x/y ring only (line_task)
    // array and row group of this CTA from blockIdx.y (<= 3 arrays: two compares, no integer division)
    __device__ __forceinline__ int array() const { return (blockIdx.y >= (unsigned)gy) + (blockIdx.y >= 2u * gy); }
    // selects, not a dynamic index: an indexed kernel-parameter array would be copied to local memory
    __device__ __forceinline__ const void *in(int a) const { return a == 0 ? src[0] : a == 1 ? src[1] : src[2]; }
    __device__ __forceinline__ void *out(int a) const { return a == 0 ? dst[0] : a == 1 ? dst[1] : dst[2]; }
};
constexpr int CODE_LD = 68;  // padded per-block code row (u32)

// ---------------------------------------------------------------------------
// BlockQuant decode: compressed slab-major records -> working buffer.
// x^_j = fma((float)code_j + 0.5f, step, mn), step = fl(fl(mx-mn) * 2^-q)
// Every load of the warp's (up to 8) records is issued before any use.
// ---------------------------------------------------------------------------
template <bool TWO, int QT>
__global__ void __launch_bounds__(CODEC_WARPS * 32)
bq_decode_kernel(const CodecArrays A, int nbx, int nby, int64_t pitch, int64_t pstride, int q_rt) {
    const int q = QT ? QT : q_rt;
    __shared__ __align__(16) uint32_t codes[CODEC_WARPS][8][CODE_LD];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int arr = A.array();
    const uint8_t *__restrict__ src = static_cast<const uint8_t *>(A.in(arr));
    float *__restrict__ dst = static_cast<float *>(A.out(arr));
    const LineTask t = line_task(nbx, blockIdx.z, blockIdx.y - arr * A.gy, A.ring_nl, A.ring_ng);
    if (t.by >= nby) return;
    const int recw = 2 * (q + 1);  // record size in 32-bit words
    const uint32_t *rec0 = reinterpret_cast<const uint32_t *>(src) +
                           ((int64_t)(t.bz * nby + t.by) * nbx + t.b0) * recw;
    const int b = lane & 15, half = lane >> 4;
    const int w0i = b < q ? 2 + 2 * (q - 1 - b) + half : -1;
    const int w1i = (TWO && 16 + b < q) ? 2 + 2 * (q - 17 - b) + half : -1;
    uint32_t w0[8], w1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        w0[i] = (i < t.nb && w0i >= 0) ? __ldg(rec0 + i * recw + w0i) : 0u;
        if (TWO) w1[i] = (i < t.nb && w1i >= 0) ? __ldg(rec0 + i * recw + w1i) : 0u;
    }
    // header words: lane i < 8 -> mn of block i, lane 8+i -> mx of block i
    const uint32_t hdr = (lane < 16 && (lane & 7) < t.nb) ? __ldg(rec0 + (lane & 7) * recw + (lane >> 3)) : 0u;
    const float mx_l = __uint_as_float(__shfl_down_sync(0xffffffffu, hdr, 8));
    const float mn_l = __uint_as_float(hdr);
    const float step_l = __fmul_rn(__fsub_rn(mx_l, mn_l), pow2f(-q));  // valid on lanes 0..7
    const Xpose X(lane);
    uint32_t(*cw)[CODE_LD] = codes[warp];
    // blocks i >= nb (line ends) decode zeros that are never written out; keeping the loop
    // unconditional keeps every shuffle warp-convergent
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t y0 = X(w0[i]);
        if (TWO) {
            const uint32_t y1 = X(w1[i]);
            cw[i][lane] = (y0 & 0xFFFFu) | ((y1 & 0xFFFFu) << 16);
            cw[i][lane + 32] = (y0 >> 16) | ((y1 >> 16) << 16);
        } else {
            cw[i][lane] = y0;  // packed: low half = code lane, high half = code lane + 32
        }
    }
    __syncwarp();
    // reconstruct in the store layout: lane -> block ib, rows r0, r0+4, r0+8, r0+12 (code j = xi + 4r),
    // each row one aligned float4: per instruction 4 rows x 128 contiguous bytes
    const int ib = lane & 7, r0 = lane >> 3;
    const float mn = __shfl_sync(0xffffffffu, mn_l, ib), step = __shfl_sync(0xffffffffu, step_l, ib);
    float *dbase = dst + (int64_t)(4 * t.bz) * pstride + (int64_t)(4 * t.by) * pitch + XOFF + 4 * t.b0 + 4 * ib;
    const float2 s2 = make_float2(step, step), m2 = make_float2(mn, mn);
    auto put = [&](int r, uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3) {
        // two values per paired-fp32 op (same IEEE operations as the scalar fma(code + 0.5, step, mn))
        const float2 h = make_float2(-8388607.5f, -8388607.5f);
        const float2 lo = __ffma2_rn(__fadd2_rn(make_float2(__uint_as_float(p0), __uint_as_float(p1)), h), s2, m2);
        const float2 hi = __ffma2_rn(__fadd2_rn(make_float2(__uint_as_float(p2), __uint_as_float(p3)), h), s2, m2);
        __stcs(reinterpret_cast<float4 *>(dbase + (int64_t)(r >> 2) * pstride + (int64_t)(r & 3) * pitch),
               make_float4(lo.x, lo.y, hi.x, hi.y));
    };
    if (ib < t.nb) {
        if (TWO) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = r0 + 4 * u;
                const uint4 c = *reinterpret_cast<const uint4 *>(&cw[ib][4 * r]);
                put(r, 0x4B000000u | c.x, 0x4B000000u | c.y, 0x4B000000u | c.z, 0x4B000000u | c.w);
            }
        } else {
            // codes j = xi + 4r of rows r = r0 + 4u (u < 2) are the low halves of words 4r + xi, those of
            // rows r + 8 the high halves of the same words
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int r = r0 + 4 * u;
                const uint4 c = *reinterpret_cast<const uint4 *>(&cw[ib][4 * r]);
                put(r, pat_lo(c.x), pat_lo(c.y), pat_lo(c.z), pat_lo(c.w));
                put(r + 8, pat_hi(c.x), pat_hi(c.y), pat_hi(c.z), pat_hi(c.w));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// BlockQuant encode: working buffer -> compressed records, bit-exact with
// oracle_bq_encode_block (same IEEE binary32 operations in the same order;
// -0 is canonicalised on mn/mx only, which yields the same codes).
// Statistics and quantisation are vectorised over the warp's 8 blocks
// (lane l: block l & 7, 4 rows); the bit planes are then packed per block.
// ---------------------------------------------------------------------------
// The per-warp encode core: the lane holds 4 rows (r0 + 4u, r = yi + 4 zi) of block ib (v), `live` says whether that block is
// written, bit i of live_mask whether block i is.  rec0 = the first block's record (32-bit words),
// cw = this warp's 8 x CODE_LD code scratch.  Returns true if a live value was rejected.
template <bool TWO, int QT>
__device__ __forceinline__ bool bq_encode_core(const float4 (&v)[4], bool live, uint32_t live_mask, uint32_t *rec0,
                                               int q_rt, uint32_t (*cw)[CODE_LD], int lane) {
    const int q = QT ? QT : q_rt;
    const int ib = lane & 7, r0 = lane >> 3;
    // block min / max with NaN propagation (FMNMX3.NAN): 16 values in 8 + 8 ops, and a NaN anywhere in the
    // block makes both NaN, which the range check below rejects together with +-Inf and |x| >= 2^126
    const float e[16] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w,
                         v[2].x, v[2].y, v[2].z, v[2].w, v[3].x, v[3].y, v[3].z, v[3].w};
    // a depth-3 tree (5 + 2 + 1 ops), not an 8-deep chain: the statistics sit on the encoder's critical path
    float mn, mx;
    {
        const float a0 = min3n(e[0], e[1], e[2]), a1 = min3n(e[3], e[4], e[5]), a2 = min3n(e[6], e[7], e[8]),
                    a3 = min3n(e[9], e[10], e[11]), a4 = min3n(e[12], e[13], e[14]);
        const float b0 = max3n(e[0], e[1], e[2]), b1 = max3n(e[3], e[4], e[5]), b2 = max3n(e[6], e[7], e[8]),
                    b3 = max3n(e[9], e[10], e[11]), b4 = max3n(e[12], e[13], e[14]);
        mn = min2n(min3n(a0, a1, a2), min3n(a3, a4, e[15]));
        mx = max2n(max3n(b0, b1, b2), max3n(b3, b4, e[15]));
    }
    mn = min2n(mn, __shfl_xor_sync(0xffffffffu, mn, 8));
    mx = max2n(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mn = min2n(mn, __shfl_xor_sync(0xffffffffu, mn, 16));
    mx = max2n(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    mn = __fadd_rn(mn, 0.0f);  // -0 -> +0
    mx = __fadd_rn(mx, 0.0f);
    const bool bad = live && (!(fabsf(mn) < 0x1p126f) || !(fabsf(mx) < 0x1p126f));
    const float range = __fsub_rn(mx, mn);
    const float step = __fmul_rn(range, pow2f(-q));
    const bool small = !(step >= 0x1p-126f);
    const float scale = small ? 0.f : __fdiv_rn(pow2f(q), range);
    const uint32_t cmax = (1u << q) - 1u;
    // code = min(cmax, floor(y)), y = (x - mn) * scale >= 0, without the quarter-rate F2I: y + 2^23
    // rounded down is the pattern of 2^23 + floor(y) while y < 2^23, and beyond it is >= 2^23 + 2^23 >
    // every clamp, so the min gives the same code.  When q <= 16 the pattern itself (2^23 + code) is
    // kept: the transpose below only uses its low 16 bits, which are the code's.  scale = 0 (a
    // (near-)constant block) makes every code 0
    // two values per paired-fp32 op: the same IEEE operations as fadd_rd(fmul(fsub(x, mn), scale), 2^23)
    const float2 nmn = make_float2(-mn, -mn), sc2 = make_float2(scale, scale), big = make_float2(0x1p23f, 0x1p23f);
    auto code2 = [&](float a, float b) -> uint2 {
        const float2 t = fadd2_rd(__fmul2_rn(__fadd2_rn(make_float2(a, b), nmn), sc2), big);
        const uint32_t ba = __float_as_uint(t.x), bb = __float_as_uint(t.y);
        return TWO ? make_uint2(min(cmax, ba - 0x4B000000u), min(cmax, bb - 0x4B000000u))
                   : make_uint2(min(cmax + 0x4B000000u, ba), min(cmax + 0x4B000000u, bb));
    };
    if (TWO) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = r0 + 4 * u;  // r = yi + 4 zi, so j = xi + 4 r
            const uint2 c01 = code2(v[u].x, v[u].y), c23 = code2(v[u].z, v[u].w);
            *reinterpret_cast<uint4 *>(&cw[ib][4 * r]) = make_uint4(c01.x, c01.y, c23.x, c23.y);
        }
    } else {
        // q <= 16: word m = (code m) | (code m+32) << 16 is the transpose's input row m.  Codes m and
        // m + 32 are rows r and r + 8 of this lane (u and u + 2), so the packing is in registers
        uint2 c[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            c[u][0] = code2(v[u].x, v[u].y);
            c[u][1] = code2(v[u].z, v[u].w);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
            *reinterpret_cast<uint4 *>(&cw[ib][4 * (r0 + 4 * u)]) =
                make_uint4(__byte_perm(c[u][0].x, c[u + 2][0].x, 0x5410), __byte_perm(c[u][0].y, c[u + 2][0].y, 0x5410),
                           __byte_perm(c[u][1].x, c[u + 2][1].x, 0x5410), __byte_perm(c[u][1].y, c[u + 2][1].y, 0x5410));
    }
    __syncwarp();
    // ---- bit planes: lane m of the transpose owns plane (m & 15), half (m >> 4)
    const int recw = 2 * (q + 1);
    const Xpose X(lane);
    const int b = lane & 15, half = lane >> 4;
    const int wi0 = b < q ? 2 + 2 * (q - 1 - b) + half : -1;
    const int wi1 = (TWO && 16 + b < q) ? 2 + 2 * (q - 17 - b) + half : -1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // unconditional (convergent shuffles); stores only for live blocks
        uint32_t *rec = rec0 + i * recw;
        const bool st = (live_mask >> i) & 1u;
        if (!TWO) {
            const uint32_t T0 = X(cw[i][lane]);
            if (st && wi0 >= 0) rec[wi0] = T0;
        } else {
            const uint32_t c_lo = cw[i][lane], c_hi = cw[i][lane + 32];
            const uint32_t T0 = X((c_lo & 0xFFFFu) | (c_hi << 16));
            if (st && wi0 >= 0) rec[wi0] = T0;
            const uint32_t T1 = X((c_lo >> 16) | ((c_hi >> 16) << 16));
            if (st && wi1 >= 0) rec[wi1] = T1;
        }
    }
    // block headers straight from the statistics lanes (lane l < 8 holds block l's mn/mx)
    if (lane < 8 && live) *reinterpret_cast<uint2 *>(rec0 + lane * recw) = make_uint2(__float_as_uint(mn), __float_as_uint(mx));
    __syncwarp();
    return bad;
}

template <bool TWO, int QT>
__global__ void __launch_bounds__(CODEC_WARPS * 32)
bq_encode_kernel(const CodecArrays A, int nbx, int nby, int64_t pitch, int64_t pstride, int q_rt, int *err) {
    const int q = QT ? QT : q_rt;
    __shared__ __align__(16) uint32_t codes[CODEC_WARPS][8][CODE_LD];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int arr = A.array();
    const float *__restrict__ src = static_cast<const float *>(A.in(arr));
    uint8_t *__restrict__ dst = static_cast<uint8_t *>(A.out(arr));
    const LineTask t = line_task(nbx, blockIdx.z, blockIdx.y - arr * A.gy);
    if (t.by >= nby) return;
    // ---- load straight into the statistics layout: lane -> block ib, rows r0, r0+4, r0+8, r0+12
    //      (per instruction 4 rows x 128 contiguous bytes: coalesced, no shared-memory staging).  Row
    //      r = yi + 4 zi = r0 + 4u is plane u, row r0 of the slab.  Lanes of blocks past the line's end
    //      (ib >= nb, first and last line only) read the rest of their 128-byte line -- inside the row's
    //      pitch -- and are never stored, so every load is unconditional
    const int ib = lane & 7, r0 = lane >> 3;
    const bool live = ib < t.nb;
    const float4 *sbase = reinterpret_cast<const float4 *>(src + (int64_t)(4 * t.bz) * pstride +
                                                           (int64_t)(4 * t.by + r0) * pitch + XOFF + 4 * t.b0 + 4 * ib);
    const int64_t ps4 = pstride / 4;  // pitch (hence pstride) is a multiple of 32 floats
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(sbase + u * ps4);
    const int recw = 2 * (q + 1);
    uint32_t *rec0 = reinterpret_cast<uint32_t *>(dst) + ((int64_t)(t.bz * nby + t.by) * nbx + t.b0) * recw;
    const bool bad = bq_encode_core<TWO, QT>(v, live, (1u << t.nb) - 1u, rec0, q, codes[warp], lane);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1);
}

// ---------------------------------------------------------------------------
// Identity codec: raw fp32 planes (row length ax) <-> working buffer.
// ---------------------------------------------------------------------------
__global__ void id_decode_kernel(const float4 *__restrict__ src, float *__restrict__ dst, int64_t n4,
                                 int ax4, int64_t pitch) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / ax4;
        const int c = (int)(i - row * ax4);
        *reinterpret_cast<float4 *>(dst + row * pitch + XOFF + 4 * c) = __ldcs(src + i);
    }
}

__global__ void id_encode_kernel(const float *__restrict__ src, float4 *__restrict__ dst, int64_t n4,
                                 int ax4, int64_t pitch) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / ax4;
        const int c = (int)(i - row * ax4);
        dst[i] = *reinterpret_cast<const float4 *>(src + row * pitch + XOFF + 4 * c);
    }
}

// ---------------------------------------------------------------------------
// Truncate-16 codec: fp32 -> bfloat16 with round-to-nearest-even (the hardware
// cvt.rn.bf16.f32), NaN -> 0x7FC0; raw bf16 planes, row length ax.  A thread moves 4 words of 8
// values per iteration, all loads issued before any store (enough bytes in flight per SM to cover
// HBM latency); blockIdx.y = plane, 32-bit in-plane indices.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t tr16_bits(float x) {
    return x != x ? 0x7FC0u : (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// the bf16 side is a flat array: one 16-byte word = 8 values = two 4-groups (ax % 4 == 0, so a
// 4-group never straddles a row; the two may sit in different rows)
__device__ __forceinline__ int64_t tr16_ws_off(int q, int ax4, int64_t pitch) {
    const int row = q / ax4;
    return row * pitch + 4 * (q - row * ax4);
}

// The ws side is addressed by global row: rows of all planes are contiguous at `pitch` floats
// (pstride = ay * pitch), so a flat 4-group index q maps to row q / ax4, column 4 (q mod ax4).
__global__ void tr16_encode_kernel(const float *__restrict__ src, uint4 *__restrict__ dst, uint32_t n8, int ax4,
                                   int64_t pitch) {
    const float *s = src + XOFF;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n8; i0 += 4 * stride) {
        float4 v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + j * stride;
            if (i < n8) {
                v[j][0] = __ldcs(reinterpret_cast<const float4 *>(s + tr16_ws_off(2 * i, ax4, pitch)));
                v[j][1] = __ldcs(reinterpret_cast<const float4 *>(s + tr16_ws_off(2 * i + 1, ax4, pitch)));
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + j * stride;
            if (i < n8)
                __stcs(dst + i, make_uint4(tr16_bits(v[j][0].x) | tr16_bits(v[j][0].y) << 16,
                                           tr16_bits(v[j][0].z) | tr16_bits(v[j][0].w) << 16,
                                           tr16_bits(v[j][1].x) | tr16_bits(v[j][1].y) << 16,
                                           tr16_bits(v[j][1].z) | tr16_bits(v[j][1].w) << 16));
        }
    }
}

__device__ __forceinline__ float4 tr16_expand(uint32_t lo, uint32_t hi) {
    return make_float4(__uint_as_float(lo << 16), __uint_as_float(lo & 0xFFFF0000u), __uint_as_float(hi << 16),
                       __uint_as_float(hi & 0xFFFF0000u));
}

__global__ void tr16_decode_kernel(const uint2 *__restrict__ src, float *__restrict__ dst, uint32_t rows, int ax4,
                                   int64_t pitch) {
    // one 4-group (8 B in, 16 B out) per thread and step, consecutive lanes on consecutive bytes; every
    // row is widened by one zero group on each side (pad columns XOFF-4.. and ax.., never read), so a
    // row's stores span whole 32-byte sectors (XOFF-4 = 24 floats = 96 B); 4 steps in flight per thread
    const int w = ax4 + 2;
    const uint32_t n = rows * (uint32_t)w;
    float *d = dst + XOFF - 4;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
        uint2 u[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + j * stride;
            const uint32_t row = i / w;
            const int c = (int)(i - row * w) - 1;
            u[j] = make_uint2(0u, 0u);
            if (i < n && c >= 0 && c < ax4) u[j] = __ldcs(src + (uint64_t)row * ax4 + c);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = i0 + j * stride;
            const uint32_t row = i / w;
            if (i < n)
                __stcs(reinterpret_cast<float4 *>(d + row * pitch + 4 * (i - row * w)), tr16_expand(u[j].x, u[j].y));
        }
    }
}

// one wave of resident CTAs over the whole range (a 2-D per-plane grid left 1.33 waves: ncu)
template <typename K>
static unsigned tr16_grid(K kernel, uint64_t n8) {
    static int blocks = 0;
    if (!blocks) {
        int dev = 0, sms = 148, per = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, 256, 0);
        blocks = sms * std::max(per, 1);
    }
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)blocks, (n8 + 1023) / 1024));
}

// ---------------------------------------------------------------------------
// 25-point leapfrog step:
//   p_prev <- 2 p_curr - p_prev + (v dt)^2 * sum_axes sum_m c_m ((f(+m) + f(-m)) - 2 f0)
//
// 2.5-D blocking with a TMA pipeline.  A CTA owns a 64 x 16 xy tile and
// marches a z range.  One thread issues cp.async.bulk.tensor loads, two
// planes ahead, of (a) the p_curr plane with its 4-cell star halo (72 x 24
// box) into a 9-slot shared-memory ring and (b) the p_prev and v tiles into
// 3-slot rings, completing on per-stage mbarriers.  Each thread computes a
// 2 x 2 cell patch (float2 along x); the z column lives in a 9-deep register
// queue indexed at compile time (the plane loop is unrolled by 9), x/y
// neighbours come from the ring with 64-bit shared loads.
// ---------------------------------------------------------------------------
// TY = tile rows (16: 256 threads, 2 CTAs per SM).  The p_curr ring has 9 slots, one per unrolled plane
// (so every slot index is a compile-time constant): at plane z it holds the x/y-neighbour plane z, the
// queue-feed plane z+4 and the two planes in flight (z+5, z+6).
template <int TY>
struct S2T {
    static constexpr int TX = 64, THREADS = 16 * TY, CTAS = TY == 16 ? 2 : 1;
    static constexpr int PW = TX + 2 * R, PH = TY + 2 * R;  // p_curr box with the star halo
    static constexpr int NB = 3, D = 2;                     // p_prev/v stages, prefetch distance
    static constexpr uint32_t PBYTES = PW * PH * 4, TBYTES = TX * TY * 4;
};
constexpr int S2_NS = 9;

template <int TY>
struct S2Smem {
    float p[S2_NS][TY + 2 * R][64 + 2 * R];
    float pp[3][TY][64];
    float v[3][TY][64];
    unsigned long long bar[4];
};
constexpr int S2_TX = 64, S2_NB = 3, S2_D = 2;

// Decode -> first step (NEXT-2, OOCS_FLAG_FUSE_DECODE): the first of a chunk's k steps reads p_{t-1} straight
// from its compressed BlockQuant records instead of a decoded working-buffer copy -- p_{t-1} is read once,
// by this step, and then overwritten by p_{t+1}, so decoding it to HBM and reading it back is 8 B per value
// of pure traffic.  Per 4-plane slab the CTA's 16 x 4 records (one bulk copy per block row, one slab ahead,
// on their own mbarriers) are decoded by the 8 warps with the decode kernel's warp transpose into a 16-bit
// code tile, and each thread reconstructs its own cells with the decode kernel's arithmetic (bitwise the
// same values).  q odd and <= 15: 16-byte records.  NF = number of arrays read this way (1; the velocity
// as a second one was measured slower -- it must still be written decoded for the later steps, so it
// saves 4 B per value for the same decode work: DESIGN.md §6).
constexpr int FS_ROWP = 68;              // u16 per code row (64 + 4): 34 words, rows 2 banks apart
constexpr int FS_PLANEP = 16 * 68 + 16;  // u16 per code plane: 552 words, planes 8 banks apart -> the
                                         // transpose's scatter (8 rows x 2 words per block) is conflict-free
constexpr int FS_RECW = 32;              // max record words (q <= 15)
template <int TY, int NF>
struct S2SmemF {
    float p[S2_NS][TY + 2 * R][64 + 2 * R];
    float v[3][TY][64];
    uint32_t stage[NF][2][TY / 4][16 * FS_RECW];  // records of a slab: 16 per block row (double-buffered)
    uint16_t cs[NF][4 * FS_PLANEP];               // codes of the slab: [plane][row][x]
    float2 hdr[NF][TY / 4][16];                   // (mn, step) per block
    unsigned long long bar[4];
    unsigned long long sbar[2];
};

// coefficients of d2/dx2, order 8 (Q1): 8/5, -1/5, 8/315, -1/560
#define C1 1.6f
#define C2 (-0.2f)
#define C3 0.025396825396825397f
#define C4 (-0.0017857142857142857f)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

struct StepArgs {
    float *pprev;
    const float *pcurr;
    int nx, ny, z_lo, z_hi, zchunk, gx;
    int64_t pitch, pstride;
    float dt;
    // fused decode (S2SmemF): records of the chunk extent's first slab of p_{t-1}, blocks per row / column
    // of the allocated grid, code bits, record words
    const uint32_t *rec[1];
    int nbx, nby, q, recw;
};

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// one thread: bulk-copy slab bz's records of the tile (block rows y0/4+1.., columns x0/4+1..+15) of each
// fused array into stage buf
template <int TY, int NF>
__device__ __forceinline__ void fuse_stage(S2SmemF<TY, NF> &S, const StepArgs &a, int bz, int buf, int x0, int y0) {
    const int bx0 = x0 / 4 + 1, nblk = min(16, a.nbx - bx0);
    const uint32_t row_bytes = (uint32_t)(nblk * a.recw * 4);
    int rows = 0;
#pragma unroll
    for (int r = 0; r < TY / 4; ++r) rows += (y0 / 4 + 1 + r < a.nby) ? 1 : 0;
    mbar_expect_tx(&S.sbar[buf], NF * rows * row_bytes);
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int r = 0; r < TY / 4; ++r) {
            const int by = y0 / 4 + 1 + r;
            if (by < a.nby)
                bulk_load(&S.stage[f][buf][r][0],
                          a.rec[f] + ((int64_t)bz * a.nby + by) * a.nbx * a.recw + (int64_t)bx0 * a.recw, row_bytes,
                          &S.sbar[buf]);
        }
}

// every warp, per fused array: decode its 8 records (block row warp/2, columns 8 (warp&1) ..) of stage buf
// into the code tile (same transpose and (mn, step) arithmetic as bq_decode_kernel)
template <int TY, int NF>
__device__ __forceinline__ void fuse_decode(S2SmemF<TY, NF> &S, const StepArgs &a, int buf, int x0, int y0, int lane,
                                            int warp) {
    const int r = warp >> 1, bl0 = 8 * (warp & 1), q = a.q, recw = a.recw;
    const int nbv = (y0 / 4 + 1 + r < a.nby) ? min(8, max(0, a.nbx - (x0 / 4 + 1 + bl0))) : 0;
    const int b = lane & 15, half = lane >> 4;
    const int w0i = b < q ? 2 + 2 * (q - 1 - b) + half : -1;
    const Xpose X(lane);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const uint32_t *st = &S.stage[f][buf][r][bl0 * recw];
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (i < nbv && w0i >= 0) ? st[i * recw + w0i] : 0u;
        const uint32_t hdr = (lane < 16 && (lane & 7) < nbv) ? st[(lane & 7) * recw + (lane >> 3)] : 0u;
        const float mx_l = __uint_as_float(__shfl_down_sync(0xffffffffu, hdr, 8));
        const float mn_l = __uint_as_float(hdr);
        if (lane < 8) S.hdr[f][r][bl0 + lane] = make_float2(mn_l, __fmul_rn(__fsub_rn(mx_l, mn_l), pow2f(-q)));
        // lane m holds codes m (low half) and m + 32 (high half): j = xi + 4 yi + 16 zi
        uint16_t *c = S.cs[f] + (lane >> 4) * FS_PLANEP + (4 * r + ((lane >> 2) & 3)) * FS_ROWP + 4 * bl0 + (lane & 3);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t y = X(w[i]);
            c[4 * i] = (uint16_t)y;
            c[4 * i + 2 * FS_PLANEP] = (uint16_t)(y >> 16);
        }
    }
}

// the two cells (x, x+1) of row y of plane zi of fused array f: x = fma((float)code + 0.5, step, mn), as
// bq_decode_kernel's put()
template <typename SM>
__device__ __forceinline__ float2 fuse_value(const SM &S, int f, int zi, int y, int x, float2 hm) {
    const uint32_t c = *reinterpret_cast<const uint32_t *>(S.cs[f] + zi * FS_PLANEP + y * FS_ROWP + x);
    const float2 h = make_float2(-8388607.5f, -8388607.5f);
    return __ffma2_rn(__fadd2_rn(make_float2(__uint_as_float(pat_lo(c)), __uint_as_float(pat_hi(c))), h),
                      make_float2(hm.y, hm.y), make_float2(hm.x, hm.x));
}

// one plane of the march; OFF = (z - zs) mod 9 is a compile-time register-queue rotation
template <int OFF, int TY, int NF, typename SM>
__device__ __forceinline__ bool s2_plane(SM &S, const CUtensorMap *mP, const CUtensorMap *mPP,
                                         const CUtensorMap *mV, const StepArgs &a, int z, int zs, int ze,
                                         int x0, int y0, float2 (&q)[9][2], uint32_t &ph, bool okr0,
                                         bool okr1, int64_t g0, float2 (&hm)[1]) {
    if (z >= ze) return false;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncthreads();  // every thread is done with plane z-1: its ring slots may be refilled
    // ring slot of plane P is (P - zs + 4) mod 9 (OFF + 4 mod 9, known at compile time)
    constexpr int NS = S2_NS;
    if (tid == 0 && z + S2_D < ze) {
        constexpr int ps = (OFF + 4 + S2_D + R) % NS;  // slot of plane z+D+4 (previously plane z+D+4-NS)
        constexpr int st = (OFF + S2_D) % S2_NB;     // stage of plane z+D
        unsigned long long *bar = &S.bar[st];
        mbar_expect_tx(bar, S2T<TY>::PBYTES + (2 - NF) * S2T<TY>::TBYTES);
        tma_load_3d(&S.p[ps][0][0], mP, XOFF + x0, y0, z + S2_D + R, bar);
        if constexpr (NF == 0) tma_load_3d(&S.pp[st][0][0], mPP, XOFF + R + x0, R + y0, z + S2_D, bar);
        tma_load_3d(&S.v[st][0][0], mV, XOFF + R + x0, R + y0, z + S2_D, bar);
    }
    if constexpr (NF > 0) {
        if (((z - zs) & 3) == 0) {  // a new slab: decode it (its records arrived one slab ago)
            const int j = (z - zs) >> 2;
            if (tid == 0 && z + 4 < ze) fuse_stage<TY, NF>(S, a, (z >> 2) + 1, (j + 1) & 1, x0, y0);
            mbar_wait(&S.sbar[j & 1], (uint32_t)(j >> 1) & 1u);
            fuse_decode<TY, NF>(S, a, j & 1, x0, y0, lane, warp);
            __syncthreads();
#pragma unroll
            for (int f = 0; f < NF; ++f) hm[f] = S.hdr[f][warp >> 1][lane >> 1];
        }
    }
    constexpr int st = OFF % S2_NB;
    mbar_wait(&S.bar[st], (ph >> st) & 1u);
    ph ^= 1u << st;
    constexpr int sz = (OFF + 4) % NS, sz4 = (OFF + 4 + R) % NS;
    const int cx = 2 * lane, cy = 2 * warp;
    // feed the queue with plane z+4 (own cells)
    q[(OFF + 8) % 9][0] = *reinterpret_cast<const float2 *>(&S.p[sz4][R + cy][R + cx]);
    q[(OFF + 8) % 9][1] = *reinterpret_cast<const float2 *>(&S.p[sz4][R + cy + 1][R + cx]);
    const float(*P)[S2T<TY>::PW] = S.p[sz];
    // y neighbours: rows cy..cy+3 and cy+6..cy+9 of the box at columns cx+4, cx+5
    float2 yr[10];
#pragma unroll
    for (int m = 0; m < 10; ++m)
        if (m != 4 && m != 5) yr[m] = *reinterpret_cast<const float2 *>(&P[cy + m][R + cx]);
    yr[4] = q[(OFF + 4) % 9][0];
    yr[5] = q[(OFF + 4) % 9][1];
    float2 pp0, pp1, v0, v1;
    if constexpr (NF > 0) {
        const int zi = (z - zs) & 3;
        pp0 = fuse_value(S, 0, zi, cy, cx, hm[0]);
        pp1 = fuse_value(S, 0, zi, cy + 1, cx, hm[0]);
    } else {
        pp0 = *reinterpret_cast<const float2 *>(&S.pp[st][cy][cx]);
        pp1 = *reinterpret_cast<const float2 *>(&S.pp[st][cy + 1][cx]);
    }
    v0 = *reinterpret_cast<const float2 *>(&S.v[st][cy][cx]);
    v1 = *reinterpret_cast<const float2 *>(&S.v[st][cy + 1][cx]);
    // The two x-adjacent cells of a row go through Blackwell's paired fp32 pipe (FADD2 / FMUL2 /
    // FFMA2): every operation is the same IEEE-rounded scalar operation as before, on both cells at
    // once, so results are bitwise those of the scalar form below (difference form, x-y-z FMA chain):
    //   lap = C1((f(x-1)+f(x+1)) - 2f0) + ... ;  p_next = (v dt)^2 lap + (2 f0 - p_prev)
    const float2 k1 = make_float2(C1, C1), k2 = make_float2(C2, C2), k3 = make_float2(C3, C3),
                 k4 = make_float2(C4, C4);
    float2 out[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int row = R + cy + r;
        // x neighbours: columns cx..cx+3 and cx+6..cx+9 (centres cx+4, cx+5 come from the queue)
        const float2 xa = *reinterpret_cast<const float2 *>(&P[row][cx]);
        const float2 xb = *reinterpret_cast<const float2 *>(&P[row][cx + 2]);
        const float2 xc = *reinterpret_cast<const float2 *>(&P[row][cx + 6]);
        const float2 xd = *reinterpret_cast<const float2 *>(&P[row][cx + 8]);
        const float2 f0 = q[(OFF + 4) % 9][r];
        const float2 f2 = __fadd2_rn(f0, f0);
        const float2 nf2 = make_float2(-f2.x, -f2.y);
        // (f(-m) + f(+m)) - 2 f0 for both cells
        auto d = [&](float2 lo, float2 hi) { return __fadd2_rn(__fadd2_rn(lo, hi), nf2); };
        float2 lap = __fmul2_rn(k1, d(make_float2(xb.y, f0.x), make_float2(f0.y, xc.x)));
        lap = __ffma2_rn(k2, d(xb, xc), lap);
        lap = __ffma2_rn(k3, d(make_float2(xa.y, xb.x), make_float2(xc.y, xd.x)), lap);
        lap = __ffma2_rn(k4, d(xa, xd), lap);
        lap = __ffma2_rn(k1, d(yr[3 + r], yr[5 + r]), lap);
        lap = __ffma2_rn(k2, d(yr[2 + r], yr[6 + r]), lap);
        lap = __ffma2_rn(k3, d(yr[1 + r], yr[7 + r]), lap);
        lap = __ffma2_rn(k4, d(yr[0 + r], yr[8 + r]), lap);
        lap = __ffma2_rn(k1, d(q[(OFF + 3) % 9][r], q[(OFF + 5) % 9][r]), lap);
        lap = __ffma2_rn(k2, d(q[(OFF + 2) % 9][r], q[(OFF + 6) % 9][r]), lap);
        lap = __ffma2_rn(k3, d(q[(OFF + 1) % 9][r], q[(OFF + 7) % 9][r]), lap);
        lap = __ffma2_rn(k4, d(q[(OFF + 0) % 9][r], q[(OFF + 8) % 9][r]), lap);
        const float2 vv = r ? v1 : v0, pv = r ? pp1 : pp0;
        const float2 vd = __fmul2_rn(vv, make_float2(a.dt, a.dt));
        out[r] = __ffma2_rn(__fmul2_rn(vd, vd), lap, __fadd2_rn(f2, make_float2(-pv.x, -pv.y)));
    }
    float *dst = a.pprev + (int64_t)z * a.pstride + g0;
    if (okr0) __stcs(reinterpret_cast<float2 *>(dst), out[0]);
    if (okr1) __stcs(reinterpret_cast<float2 *>(dst + a.pitch), out[1]);
    return true;
}

template <int TY, int NF>
__global__ void __launch_bounds__(S2T<TY>::THREADS, S2T<TY>::CTAS)
stencil_step_tma_kernel(const __grid_constant__ CUtensorMap mP, const __grid_constant__ CUtensorMap mPP,
                        const __grid_constant__ CUtensorMap mV, const StepArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using SM = std::conditional_t<NF == 0, S2Smem<TY>, S2SmemF<TY, NF>>;
    SM &S = *reinterpret_cast<SM *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int x0 = blockIdx.x * S2_TX, y0 = blockIdx.y * TY;
    const int zs = a.z_lo + blockIdx.z * a.zchunk;
    const int ze = min(a.z_hi, zs + a.zchunk);
    if (zs >= ze) return;
    const int x = x0 + 2 * lane, y = y0 + 2 * warp;
    const bool okx = x < a.nx;
    const bool okr0 = okx && y < a.ny, okr1 = okx && y + 1 < a.ny;
    // element (x, y, z) of the working buffer: z*pstride + (y+R)*pitch + x + R + XOFF
    const int64_t g0 = (int64_t)(y + R) * a.pitch + x + R + XOFF;
    if (tid == 0) {
        for (int i = 0; i <= S2_NB; ++i) mbar_init(&S.bar[i], 1);
        if constexpr (NF > 0) {
            mbar_init(&S.sbar[0], 1);
            mbar_init(&S.sbar[1], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        // prologue: p_curr planes zs..zs+3 (x/y neighbours of the first 4 planes), then the
        // first D stages (plane z+4 of p_curr, plane z of p_prev and v)
        unsigned long long *pro = &S.bar[S2_NB];
        mbar_expect_tx(pro, 4 * S2T<TY>::PBYTES);
        constexpr int NS = S2_NS;
        for (int i = 0; i < 4; ++i) tma_load_3d(&S.p[(4 + i) % NS][0][0], &mP, XOFF + x0, y0, zs + i, pro);
        if constexpr (NF > 0) fuse_stage<TY, NF>(S, a, zs >> 2, 0, x0, y0);  // records of the first slab
        for (int j = 0; j < S2_D; ++j) {
            const int z = zs + j;
            if (z >= ze) break;
            unsigned long long *bar = &S.bar[j % S2_NB];
            mbar_expect_tx(bar, S2T<TY>::PBYTES + (2 - NF) * S2T<TY>::TBYTES);
            tma_load_3d(&S.p[(j + 4 + R) % NS][0][0], &mP, XOFF + x0, y0, z + R, bar);
            if constexpr (NF == 0) tma_load_3d(&S.pp[j % S2_NB][0][0], &mPP, XOFF + R + x0, R + y0, z, bar);
            tma_load_3d(&S.v[j % S2_NB][0][0], &mV, XOFF + R + x0, R + y0, z, bar);
        }
    }
    // register queue: planes zs-4 .. zs+3 of the own 2x2 cells (index m <-> plane zs-4+m)
    float2 q[9][2];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const float *src = a.pcurr + (int64_t)(zs - R + m) * a.pstride + g0;
        float2 r0 = make_float2(0.f, 0.f), r1 = r0;
        if (okr0) r0 = __ldg(reinterpret_cast<const float2 *>(src));
        if (okr1) r1 = __ldg(reinterpret_cast<const float2 *>(src + a.pitch));
        q[m][0] = r0;
        q[m][1] = r1;
    }
    q[8][0] = q[8][1] = make_float2(0.f, 0.f);
    mbar_wait(&S.bar[S2_NB], 0);
    uint32_t ph = 0;
    float2 hm[1] = {make_float2(0.f, 0.f)};
    for (int zb = zs; zb < ze; zb += 9) {
        if (!s2_plane<0, TY, NF>(S, &mP, &mPP, &mV, a, zb + 0, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<1, TY, NF>(S, &mP, &mPP, &mV, a, zb + 1, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<2, TY, NF>(S, &mP, &mPP, &mV, a, zb + 2, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<3, TY, NF>(S, &mP, &mPP, &mV, a, zb + 3, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<4, TY, NF>(S, &mP, &mPP, &mV, a, zb + 4, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<5, TY, NF>(S, &mP, &mPP, &mV, a, zb + 5, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<6, TY, NF>(S, &mP, &mPP, &mV, a, zb + 6, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<7, TY, NF>(S, &mP, &mPP, &mV, a, zb + 7, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
        if (!s2_plane<8, TY, NF>(S, &mP, &mPP, &mV, a, zb + 8, zs, ze, x0, y0, q, ph, okr0, okr1, g0, hm)) break;
    }
}

// ---------------------------------------------------------------------------
// ZFP fixed-rate codec (NEXT-1; the algorithm of cuZFP), one thread per 4x4x4 block,
// everything in registers: block-floating-point -> integer lifting along x, y, z -> sequency order
// + negabinary -> a 2 x (32x32) in-register bit transpose turns the 64 coefficients into 32 bit
// planes -> embedded coding with group tests, truncated at maxbits = 64 * rate.  Bit-exact with
// oracle_zfp_encode_block / oracle_zfp_decode_block.
// ---------------------------------------------------------------------------
// compile-time copy (register renaming needs constant indices)
struct ZfpPerm {
    unsigned char p[64];
};
__host__ __device__ constexpr ZfpPerm zfp_perm() {
    return ZfpPerm{{0,  1,  4,  16, 20, 17, 5,  2,  8,  32, 21, 6,  18, 24, 9,  33, 36, 3,  12, 48, 22, 25,
                    37, 40, 34, 10, 7,  19, 28, 13, 49, 52, 41, 38, 26, 23, 29, 53, 11, 35, 44, 14, 50, 56,
                    42, 27, 39, 45, 30, 54, 57, 60, 51, 15, 43, 46, 58, 61, 55, 31, 62, 59, 47, 63}};
}

__device__ __forceinline__ void zfp_fwd_lift(int32_t &x, int32_t &y, int32_t &z, int32_t &w) {
    x += w; x >>= 1; w -= x;
    z += y; z >>= 1; y -= z;
    x += z; x >>= 1; z -= x;
    w += y; w >>= 1; y -= w;
    w += y >> 1; y -= w >> 1;
}
__device__ __forceinline__ void zfp_inv_lift(int32_t &x, int32_t &y, int32_t &z, int32_t &w) {
    y += w >> 1; w -= y >> 1;
    y += w; w <<= 1; w -= y;
    z += x; x <<= 1; x -= z;
    y += z; z <<= 1; z -= y;
    w += x; x <<= 1; x -= w;
}
__device__ __forceinline__ void zfp_fwd_xform(int32_t (&b)[64]) {
#pragma unroll
    for (int z = 0; z < 4; z++)
#pragma unroll
        for (int y = 0; y < 4; y++) {
            const int o = 4 * y + 16 * z;
            zfp_fwd_lift(b[o], b[o + 1], b[o + 2], b[o + 3]);
        }
#pragma unroll
    for (int x = 0; x < 4; x++)
#pragma unroll
        for (int z = 0; z < 4; z++) {
            const int o = 16 * z + x;
            zfp_fwd_lift(b[o], b[o + 4], b[o + 8], b[o + 12]);
        }
#pragma unroll
    for (int y = 0; y < 4; y++)
#pragma unroll
        for (int x = 0; x < 4; x++) {
            const int o = x + 4 * y;
            zfp_fwd_lift(b[o], b[o + 16], b[o + 32], b[o + 48]);
        }
}
__device__ __forceinline__ void zfp_inv_xform(int32_t (&b)[64]) {
#pragma unroll
    for (int y = 0; y < 4; y++)
#pragma unroll
        for (int x = 0; x < 4; x++) {
            const int o = x + 4 * y;
            zfp_inv_lift(b[o], b[o + 16], b[o + 32], b[o + 48]);
        }
#pragma unroll
    for (int x = 0; x < 4; x++)
#pragma unroll
        for (int z = 0; z < 4; z++) {
            const int o = 16 * z + x;
            zfp_inv_lift(b[o], b[o + 4], b[o + 8], b[o + 12]);
        }
#pragma unroll
    for (int z = 0; z < 4; z++)
#pragma unroll
        for (int y = 0; y < 4; y++) {
            const int o = 4 * y + 16 * z;
            zfp_inv_lift(b[o], b[o + 1], b[o + 2], b[o + 3]);
        }
}

// in-register 32x32 bit transpose (LSB convention): afterwards bit j of a[k] = old bit k of a[j]
__device__ __forceinline__ void transpose32_regs(uint32_t *a) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = s == 0 ? 0x0000FFFFu : s == 1 ? 0x00FF00FFu : s == 2 ? 0x0F0F0F0Fu
                         : s == 3 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            if (r & j) continue;
            if (j >= 8) {  // whole bytes move: two byte permutes instead of the shift/xor swap
                const uint32_t x = a[r], y = a[r | j];
                a[r] = __byte_perm(x, y, j == 16 ? 0x5410 : 0x6240);
                a[r | j] = __byte_perm(x, y, j == 16 ? 0x7632 : 0x7351);
                continue;
            }
            const uint32_t t = ((a[r] >> j) ^ a[r | j]) & m;
            a[r] ^= t << j;
            a[r | j] ^= t;
        }
    }
}

// LSB-first writer over 32-bit words: fewer than 32 bits pending in a 64-bit accumulator, so a put of
// m <= 32 bits is a shift, an OR and a rarely divergent word store
struct BitOut {
    uint32_t *out;
    uint64_t cur;
    int nb;  // bits pending in cur (0..31)
    __device__ __forceinline__ void put(uint32_t v, int m) {  // 0 <= m <= 32, v < 2^m
        cur |= (uint64_t)v << nb;
        nb += m;
        if (nb >= 32) {
            *out++ = (uint32_t)cur;
            cur >>= 32;
            nb -= 32;
        }
    }
    __device__ __forceinline__ void put64(uint64_t v, int m) {  // low m bits of v, 0 <= m <= 64
        if (m <= 32) {
            put(m == 32 ? (uint32_t)v : (uint32_t)v & ((1u << m) - 1u), m);
        } else {
            put((uint32_t)v, 32);
            const uint32_t hi = (uint32_t)(v >> 32);
            put(m == 64 ? hi : hi & ((1u << (m - 32)) - 1u), m - 32);
        }
    }
};

// LSB-first reader over 32-bit words: a right-aligned 64-bit buffer that always holds >= 32 valid
// bits, so the next 32 bits are one register read and consuming m <= 32 bits is a 64-bit shift plus a
// rarely taken refill (bits past the record read as zeros)
struct BitBuf {
    const uint32_t *in, *end;  // next word to load, end of the record
    uint64_t buf;
    int cnt;       // valid bits in buf (32..64)
    uint32_t nxt;  // the word after buf, loaded one refill ahead (its latency hides behind ~32 bits)
    __device__ __forceinline__ void init(const uint32_t *p, int words) {
        end = p + words;
        buf = (uint64_t)__ldg(p) | (words > 1 ? (uint64_t)__ldg(p + 1) << 32 : 0);
        nxt = words > 2 ? __ldg(p + 2) : 0u;
        in = p + 3;
        cnt = 64;
    }
    __device__ __forceinline__ uint32_t peek32() const { return (uint32_t)buf; }
    __device__ __forceinline__ void consume(int m) {  // 0 <= m <= 32
        buf >>= m;
        cnt -= m;
        if (cnt < 32) {
            buf |= (uint64_t)nxt << cnt;
            cnt += 32;
            nxt = in < end ? __ldg(in) : 0u;
            ++in;
        }
    }
    __device__ __forceinline__ uint64_t read(int m) {  // 0 <= m <= 64
        if (m <= 32) {
            const uint32_t v = m == 32 ? peek32() : peek32() & ((1u << m) - 1u);
            consume(m);
            return v;
        }
        const uint32_t lo = peek32();
        consume(32);
        const uint32_t hi = m == 64 ? peek32() : peek32() & ((1u << (m - 32)) - 1u);
        consume(m - 32);
        return (uint64_t)lo | ((uint64_t)hi << 32);
    }
};

__device__ __forceinline__ uint32_t zfp_int2uint(int32_t x) { return ((uint32_t)x + 0xaaaaaaaau) ^ 0xaaaaaaaau; }
__device__ __forceinline__ int32_t zfp_uint2int(uint32_t x) { return (int32_t)((x ^ 0xaaaaaaaau) - 0xaaaaaaaau); }

// grid: x over the (by, bx) blocks of a slab (one thread each), y = slab
__global__ void __launch_bounds__(128)
zfp_encode_kernel(const float *__restrict__ src, uint64_t *__restrict__ dst, int nbx, int nby, int64_t pitch,
                  int64_t pstride, int rate, int *err) {
    __shared__ uint64_t zs_planes[32][128];
    // one thread per block, flattened over the slab's (by, bx) so no lanes idle at row ends
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nbx * nby) return;
    const int bx = (int)(t % nbx), by = (int)(t / nbx), bz = blockIdx.y;
    const int words = 2 * rate;  // 64 * rate bits in 32-bit words
    uint32_t *rec = reinterpret_cast<uint32_t *>(dst + ((int64_t)(bz * nby + by) * nbx + bx) * rate);
    float x[64];
    const float *s0 = src + (int64_t)(4 * bz) * pstride + (int64_t)(4 * by) * pitch + XOFF + 4 * bx;
#pragma unroll
    for (int zi = 0; zi < 4; ++zi)
#pragma unroll
        for (int yi = 0; yi < 4; ++yi) {
            const float4 v = __ldcs(reinterpret_cast<const float4 *>(s0 + (int64_t)zi * pstride + (int64_t)yi * pitch));
            x[16 * zi + 4 * yi + 0] = v.x;
            x[16 * zi + 4 * yi + 1] = v.y;
            x[16 * zi + 4 * yi + 2] = v.z;
            x[16 * zi + 4 * yi + 3] = v.w;
        }
    float amax = 0.f;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        bad |= !(fabsf(x[j]) <= 3.402823466e38f);  // NaN or Inf
        amax = fmaxf(amax, fabsf(x[j]));
    }
    if (bad) {
        atomicOr(err, 1);
        return;
    }
    BitOut bw{rec, 0, 0};
    if (amax > 0.f) {
        const int be = (int)(__float_as_uint(amax) >> 23);
        const int emax = max(be - 126, -126);  // frexp exponent, clamped for denormals
        const uint32_t e = (uint32_t)(emax + 127);
        bw.put(2 * e + 1, 9);
        int32_t ib[64];
        if (emax >= -97) {  // 2^(30-emax) is a normal float: the float product is exact
            const float sc = __int_as_float((127 + 30 - emax) << 23);
#pragma unroll
            for (int j = 0; j < 64; ++j) ib[j] = (int32_t)(sc * x[j]);
        } else {
            const double sc = ldexp(1.0, 30 - emax);
#pragma unroll
            for (int j = 0; j < 64; ++j) ib[j] = (int32_t)(sc * (double)x[j]);
        }
        zfp_fwd_xform(ib);
        constexpr ZfpPerm P = zfp_perm();
        uint32_t pl[64];  // coefficients in sequency order, negabinary; transposed into bit planes
#pragma unroll
        for (int i = 0; i < 64; ++i) pl[i] = zfp_int2uint(ib[P.p[i]]);
        transpose32_regs(pl);       // pl[k]      bit j = bit k of coefficient j       (j < 32)
        transpose32_regs(pl + 32);  // pl[32 + k] bit j = bit k of coefficient 32 + j
        // bit planes to shared memory ([plane][thread]: conflict-free), so the data-dependent coding
        // loop below stays rolled (a 32x unrolled loop overflows the instruction cache)
#pragma unroll
        for (int k = 0; k < 32; ++k) zs_planes[k][threadIdx.x] = (uint64_t)pl[k] | ((uint64_t)pl[32 + k] << 32);
        int bits = 64 * rate - 9;
        int n = 0;
#pragma unroll 1
        for (int k = 31; k >= 0; --k) {
            if (bits <= 0) break;
            uint64_t plane = zs_planes[k][threadIdx.x];
            const int m = min(n, bits);
            bits -= m;
            bw.put64(plane, m);
            plane = m == 64 ? 0 : plane >> m;
            // unary run-length code of the remainder, one step per newly significant coefficient:
            // group test bit, then the zeros up to the next 1 and that 1 (implied at position 63)
            while (n < 64 && bits > 0) {
                bits--;
                if (!plane) {  // group test 0
                    bw.put(0, 1);
                    break;
                }
                const int z = __ffsll((long long)plane) - 1, zmax = 63 - n;
                const int len = z < zmax ? z + 1 : zmax;  // bits the zfp loop would write
                if (len <= bits) {  // group bit 1, z zeros and a 1 (implied when n reaches 63): one put
                    if (len < 32)
                        bw.put(1u | (z < zmax ? 2u << z : 0u), len + 1);
                    else
                        bw.put64(1u | (z < zmax ? (uint64_t)2 << z : 0), len + 1);
                    bits -= len;
                    const int adv = z < zmax ? z + 1 : zmax + 1;
                    n += adv;
                    plane = adv >= 64 ? 0 : plane >> adv;
                } else {  // budget ends inside the zero run
                    bw.put64(1u, bits + 1);
                    n += bits + 1;
                    plane = 0;
                    bits = 0;
                }
            }
        }
    } else {
        bw.put(0, 1);
    }
    // pad the record with zeros up to maxbits
    if (bw.nb) *bw.out++ = (uint32_t)bw.cur;
    while (bw.out < rec + words) *bw.out++ = 0;
}

__global__ void __launch_bounds__(128)
zfp_decode_kernel(const uint64_t *__restrict__ src, float *__restrict__ dst, int nbx, int nby, int64_t pitch,
                  int64_t pstride, int rate) {
    __shared__ uint64_t zs_planes[32][128];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nbx * nby) return;
    const int bx = (int)(t % nbx), by = (int)(t / nbx), bz = blockIdx.y;
    const uint64_t *rec = src + ((int64_t)(bz * nby + by) * nbx + bx) * rate;
    BitBuf br;
    br.init(reinterpret_cast<const uint32_t *>(rec), 2 * rate);
    float x[64];
    const uint32_t head = br.peek32();
    if (!(head & 1u)) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = 0.f;
    } else {
        const int emax = (int)((head >> 1) & 0xFFu) - 127;
        br.consume(9);
#pragma unroll
        for (int k = 0; k < 32; ++k) zs_planes[k][threadIdx.x] = 0;
        int bits = 64 * rate - 9;
        int n = 0;
#pragma unroll 1
        for (int k = 31; k >= 0; --k) {
            if (bits <= 0) break;
            // the first n coefficients (already significant) are sent verbatim
            const int m = min(n, bits);
            bits -= m;
            uint64_t plane = br.read(m);
            // then per newly significant coefficient: group-test bit 1, zeros, a 1 (implied at 63); the
            // inner zfp loop reads at most lim = min(63 - n, bits) run bits and leaves n at the 1 it
            // found, or lim further on (budget or position 63 reached), where the bit is set either way
            while (n < 64 && bits > 0) {
                bits--;
                const uint32_t w = br.peek32();
                if (!(w & 1u)) {  // group test 0: nothing more in this plane
                    br.consume(1);
                    break;
                }
                const int lim = min(63 - n, bits);
                const uint32_t t = w >> 1;  // the next 31 stream bits
                if (t || lim <= 31) {
                    const int z = min(t ? __ffs(t) - 1 : 31, lim);
                    const int used = z < lim ? z + 1 : z;  // run of zeros (+ its terminating 1)
                    br.consume(1 + used);
                    bits -= used;
                    n += z;
                } else {  // >= 31 zeros and room for more: count the run word by word
                    br.consume(1);
                    int rem = lim;
                    while (true) {
                        const uint32_t w2 = br.peek32();
                        const int zz = w2 ? __ffs(w2) - 1 : 32;
                        if (zz < 32 && zz < rem) {  // the terminating 1
                            br.consume(zz + 1);
                            bits -= zz + 1;
                            n += zz;
                            break;
                        }
                        if (rem <= 32) {  // limit reached inside the run
                            br.consume(rem);
                            bits -= rem;
                            n += rem;
                            break;
                        }
                        br.consume(32);
                        bits -= 32;
                        n += 32;
                        rem -= 32;
                    }
                }
                plane |= (uint64_t)1 << n;
                n++;
            }
            zs_planes[k][threadIdx.x] = plane;
        }
        uint32_t pl[64];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint64_t plane = zs_planes[k][threadIdx.x];
            pl[k] = (uint32_t)plane;
            pl[32 + k] = (uint32_t)(plane >> 32);
        }
        transpose32_regs(pl);       // back to coefficients: pl[j] bit k = plane k bit j
        transpose32_regs(pl + 32);
        constexpr ZfpPerm P = zfp_perm();
        int32_t ib[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) ib[P.p[i]] = zfp_uint2int(pl[i]);
        zfp_inv_xform(ib);
        if (emax >= -96) {  // 2^(emax-30) is a normal float: one fp32 product = the exact product rounded once
            const float sc = __int_as_float((127 + emax - 30) << 23);
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = __fmul_rn(__int2float_rn(ib[j]), sc);
        } else {
            const double sc = ldexp(1.0, emax - 30);
#pragma unroll
            for (int j = 0; j < 64; ++j) x[j] = (float)((double)__int2float_rn(ib[j]) * sc);
        }
    }
    float *d0 = dst + (int64_t)(4 * bz) * pstride + (int64_t)(4 * by) * pitch + XOFF + 4 * bx;
#pragma unroll
    for (int zi = 0; zi < 4; ++zi)
#pragma unroll
        for (int yi = 0; yi < 4; ++yi)
            __stcs(reinterpret_cast<float4 *>(d0 + (int64_t)zi * pstride + (int64_t)yi * pitch),
                   make_float4(x[16 * zi + 4 * yi], x[16 * zi + 4 * yi + 1], x[16 * zi + 4 * yi + 2],
                               x[16 * zi + 4 * yi + 3]));
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline int64_t nlines_of(int64_t ax) { return (XOFF + ax + 31) / 32; }

cudaError_t launch_decode(const void *const *src, float *const *dst, int n_arr, int64_t ax, int64_t ay,
                          int64_t planes, int64_t pitch, int codec, int q, cudaStream_t st) {
    if (planes <= 0 || n_arr <= 0) return cudaSuccess;
    if (n_arr > N_ARRAYS) return cudaErrorInvalidValue;
    const int64_t pstride = ay * pitch;
    if (codec == 1) {  // BlockQuant: all arrays in one launch
        const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
        const int nl = (int)nlines_of(ax);
        CodecArrays A{};
        for (int a = 0; a < n_arr; ++a) {
            A.src[a] = src[a];
            A.dst[a] = dst[a];
        }
        A.gy = (nby + 7) / 8;
        const dim3 blocks((unsigned)nl, (unsigned)(A.gy * n_arr), (unsigned)(planes / 4));
#define DEC(TWO, QT) bq_decode_kernel<TWO, QT><<<blocks, CODEC_WARPS * 32, 0, st>>>(A, nbx, nby, pitch, pstride, q)
        switch (q) {  // the BASELINE.json rate sweep 8/12/16/24 bits/value gets constant-folded kernels
        case 7: DEC(false, 7); break;
        case 11: DEC(false, 11); break;
        case 15: DEC(false, 15); break;
        case 23: DEC(true, 23); break;
        default:
            if (q > 16) DEC(true, 0);
            else DEC(false, 0);
        }
#undef DEC
        return cudaGetLastError();
    }
    for (int a = 0; a < n_arr; ++a) {
        if (codec == 2) {  // ZFP: q carries the rate
            const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
            const dim3 grid((unsigned)(((int64_t)nbx * nby + 127) / 128), (unsigned)(planes / 4));
            zfp_decode_kernel<<<grid, 128, 0, st>>>(static_cast<const uint64_t *>(src[a]), dst[a], nbx, nby, pitch,
                                                    pstride, q);
        } else if (codec == 3) {
            // flat over all planes in launches of < 2^31 words (32-bit indices); ax, ay multiples of 4
            const int64_t plane8 = ay * ax / 8, per = std::max<int64_t>(1, ((int64_t)1 << 30) / plane8);
            for (int64_t z = 0; z < planes; z += per) {
                const uint64_t n8 = (uint64_t)std::min(per, planes - z) * plane8;
                tr16_decode_kernel<<<tr16_grid(tr16_decode_kernel, n8), 256, 0, st>>>(
                    static_cast<const uint2 *>(src[a]) + 2 * z * plane8, dst[a] + z * pstride,
                    (uint32_t)(std::min(per, planes - z) * ay), (int)(ax / 4), pitch);
            }
        } else {
            const int64_t n4 = planes * ay * (ax / 4);
            const int threads = 256;
            const int64_t blocks = std::min<int64_t>((n4 + threads - 1) / threads, 148 * 16);
            id_decode_kernel<<<(unsigned)blocks, threads, 0, st>>>(static_cast<const float4 *>(src[a]), dst[a], n4,
                                                                  (int)(ax / 4), pitch);
        }
    }
    return cudaGetLastError();
}

// BlockQuant, one array: decode only the blocks of the x/y ring (bx = 0, nbx-1; by = 0, nby-1) of every slab,
// with their lines / row groups (the fused first step overwrites the interior)
cudaError_t launch_decode_ring(const void *src, float *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch, int q,
                               cudaStream_t st) {
    if (planes <= 0) return cudaSuccess;
    const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
    CodecArrays A{};
    A.src[0] = src;
    A.dst[0] = dst;
    A.gy = 1;
    A.ring_nl = (int)nlines_of(ax);
    A.ring_ng = (nby + 7) / 8;
    const dim3 blocks((unsigned)(2 * A.ring_nl + 2 * A.ring_ng), 1u, (unsigned)(planes / 4));
    const int64_t pstride = ay * pitch;
#define DEC(TWO, QT) bq_decode_kernel<TWO, QT><<<blocks, CODEC_WARPS * 32, 0, st>>>(A, nbx, nby, pitch, pstride, q)
    switch (q) {
    case 7: DEC(false, 7); break;
    case 11: DEC(false, 11); break;
    case 15: DEC(false, 15); break;
    default:
        if (q > 16) DEC(true, 0);
        else DEC(false, 0);
    }
#undef DEC
    return cudaGetLastError();
}

cudaError_t launch_encode(const float *const *src, void *const *dst, int n_arr, int64_t ax, int64_t ay,
                          int64_t planes, int64_t pitch, int codec, int q, int *err, cudaStream_t st) {
    if (planes <= 0 || n_arr <= 0) return cudaSuccess;
    if (n_arr > N_ARRAYS) return cudaErrorInvalidValue;
    const int64_t pstride = ay * pitch;
    if (codec == 1) {  // BlockQuant: all arrays in one launch
        const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
        const int nl = (int)nlines_of(ax);
        CodecArrays A{};
        for (int a = 0; a < n_arr; ++a) {
            A.src[a] = src[a];
            A.dst[a] = dst[a];
        }
        A.gy = (nby + 7) / 8;
        const dim3 blocks((unsigned)nl, (unsigned)(A.gy * n_arr), (unsigned)(planes / 4));
#define ENC(TWO, QT) bq_encode_kernel<TWO, QT><<<blocks, CODEC_WARPS * 32, 0, st>>>(A, nbx, nby, pitch, pstride, q, err)
        switch (q) {
        case 7: ENC(false, 7); break;
        case 11: ENC(false, 11); break;
        case 15: ENC(false, 15); break;
        case 23: ENC(true, 23); break;
        default:
            if (q > 16) ENC(true, 0);
            else ENC(false, 0);
        }
#undef ENC
        return cudaGetLastError();
    }
    for (int a = 0; a < n_arr; ++a) {
        if (codec == 2) {  // ZFP: q carries the rate
            const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
            const dim3 grid((unsigned)(((int64_t)nbx * nby + 127) / 128), (unsigned)(planes / 4));
            zfp_encode_kernel<<<grid, 128, 0, st>>>(src[a], static_cast<uint64_t *>(dst[a]), nbx, nby, pitch,
                                                    pstride, q, err);
        } else if (codec == 3) {
            const int64_t plane8 = ay * ax / 8, per = std::max<int64_t>(1, ((int64_t)1 << 30) / plane8);
            for (int64_t z = 0; z < planes; z += per) {
                const uint64_t n8 = (uint64_t)std::min(per, planes - z) * plane8;
                tr16_encode_kernel<<<tr16_grid(tr16_encode_kernel, n8), 256, 0, st>>>(
                    src[a] + z * pstride, static_cast<uint4 *>(dst[a]) + z * plane8, (uint32_t)n8, (int)(ax / 4),
                    pitch);
            }
        } else {
            const int64_t n4 = planes * ay * (ax / 4);
            const int threads = 256;
            const int64_t blocks = std::min<int64_t>((n4 + threads - 1) / threads, 148 * 16);
            id_encode_kernel<<<(unsigned)blocks, threads, 0, st>>>(src[a], static_cast<float4 *>(dst[a]), n4,
                                                                  (int)(ax / 4), pitch);
        }
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Multi-GPU halo send: two (src, dst) byte ranges of the same length, dst in a neighbour's HBM mapped
// through CUDA IPC (NVLink peer stores) -- SM-driven so the copy engines stay free for the PCIe
// pipeline.  16-byte vectors when every pointer and the length allow it, else 8-byte.
// ---------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) peer_copy_kernel(const V *__restrict__ s0, V *__restrict__ d0,
                                                        const V *__restrict__ s1, V *__restrict__ d1, uint64_t n) {
    const V *s = blockIdx.y ? s1 : s0;
    V *d = blockIdx.y ? d1 : d0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
        V v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * stride < n) v[j] = __ldcs(s + i + j * stride);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * stride < n) d[i + j * stride] = v[j];
    }
}

cudaError_t launch_peer_copy(const void *src0, void *dst0, const void *src1, void *dst1, uint64_t bytes,
                             cudaStream_t st, int ranges) {
    if (!bytes) return cudaSuccess;
    const uintptr_t all = reinterpret_cast<uintptr_t>(src0) | reinterpret_cast<uintptr_t>(dst0) |
                          reinterpret_cast<uintptr_t>(src1) | reinterpret_cast<uintptr_t>(dst1) | (uintptr_t)bytes;
    if (all & 7) return cudaErrorInvalidValue;
    const bool v16 = (all & 15) == 0;
    const uint64_t n = bytes / (v16 ? 16 : 8);
    const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(148, (n + 1023) / 1024));
    const dim3 grid(gx, ranges == 1 ? 1 : 2);
    if (v16)
        peer_copy_kernel<uint4><<<grid, 256, 0, st>>>(static_cast<const uint4 *>(src0), static_cast<uint4 *>(dst0),
                                                       static_cast<const uint4 *>(src1), static_cast<uint4 *>(dst1), n);
    else
        peer_copy_kernel<uint2><<<grid, 256, 0, st>>>(static_cast<const uint2 *>(src0), static_cast<uint2 *>(dst0),
                                                       static_cast<const uint2 *>(src1), static_cast<uint2 *>(dst1), n);
    return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency,
// so the library still loads on a CPU-only box)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    // resolved once, thread-safe (plans may be driven from several host threads)
    static const EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return (EncodeTiledFn) nullptr;
    }();
    return fn;
}

static bool make_map(CUtensorMap *m, const float *base, int64_t pitch, int64_t ay, int64_t planes, int bx, int by) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)ay, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)(pitch * ay) * 4};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, box, es,
              // L2 promotion 256 B: same-box A/B on the HBM-resident c3 pipeline, stencil 5683-5689 GB/s vs
              // 5611-5637 with 128 B, 5505 with 64 B, 5616-5634 with none (profiles/r02_tma_promotion.json)
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TY, int NF>
static cudaError_t launch_stencil(const float *vel, float *pprev, const float *pcurr, int64_t ax, int64_t ay,
                                  int64_t pitch, int64_t planes, int64_t z_lo, int64_t z_hi, float dt, StepArgs a,
                                  cudaStream_t st) {
    if (z_hi <= z_lo) return cudaSuccess;
    using SM = std::conditional_t<NF == 0, S2Smem<TY>, S2SmemF<TY, NF>>;
    const size_t smem = sizeof(SM);
    // per device (the attribute is per function and device); idempotent, so racing threads are harmless
    cudaError_t e = cudaFuncSetAttribute(stencil_step_tma_kernel<TY, NF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    CUtensorMap mP, mPP, mV;
    if (!make_map(&mP, pcurr, pitch, ay, planes, S2T<TY>::PW, S2T<TY>::PH) ||
        !make_map(&mPP, pprev, pitch, ay, planes, S2_TX, TY) || !make_map(&mV, vel, pitch, ay, planes, S2_TX, TY))
        return cudaErrorInvalidValue;
    a.pprev = pprev;
    a.pcurr = pcurr;
    a.nx = (int)(ax - 2 * R);
    a.ny = (int)(ay - 2 * R);
    a.z_lo = (int)z_lo;
    a.z_hi = (int)z_hi;
    a.pitch = pitch;
    a.pstride = ay * pitch;
    a.dt = dt;
    const int gx = (a.nx + S2_TX - 1) / S2_TX, gy = (a.ny + TY - 1) / TY;
    a.gx = gx;
    // split z so the grid is close to a whole number of waves (the fused decode: whole 4-plane slabs)
    const int Z = (int)(z_hi - z_lo), tiles = gx * gy, res = 148 * S2T<TY>::CTAS;
    auto chunk_of = [&](int nzc) {
        const int c = (Z + nzc - 1) / nzc;
        return NF ? (c + 3) & ~3 : c;
    };
    int best = 1;
    double best_eff = 0;
    for (int nzc = 1; nzc <= 16; ++nzc) {
        const int chunk = chunk_of(nzc);
        if (nzc > 1 && chunk < 24) break;
        const int items = tiles * ((Z + chunk - 1) / chunk);
        const double waves = (double)items / res;
        const double eff = waves / std::ceil(waves) * (double)chunk / (chunk + 4.0);  // tail x warm-up
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = nzc;
        }
    }
    a.zchunk = chunk_of(best);
    const int nzc = (Z + a.zchunk - 1) / a.zchunk;
    dim3 grid(gx, gy, nzc);
    stencil_step_tma_kernel<TY, NF><<<grid, S2T<TY>::THREADS, smem, st>>>(mP, mPP, mV, a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// STAR7 (oocs_stencil 1): the 2nd-order 7-point Laplacian, radius 1, for small exact tests.
// Not a hot path: one thread per (x, y) column of a 32 x 8 tile marching over its z range with the
// z-neighbours in registers, x/y neighbours through L1.  Difference form as the 25-point kernel:
//   L = ((f(x-1)+f(x+1)) - 2 f0) + ((f(y-1)+f(y+1)) - 2 f0) + ((f(z-1)+f(z+1)) - 2 f0)  (left to right)
//   p_next = (v dt)^2 L + (2 f0 - p_prev)  (one FMA)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) star7_step_kernel(const float *__restrict__ vel, float *pprev,
                                                         const float *__restrict__ pcurr, int nx, int ny, int z_lo,
                                                         int z_hi, int zchunk, int64_t pitch, int64_t pstride,
                                                         float dt) {
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    if (x >= nx || y >= ny) return;
    const int zs = z_lo + blockIdx.z * zchunk, ze = min(z_hi, zs + zchunk);
    const int64_t g = (int64_t)(y + R) * pitch + x + R + XOFF;
    float fm = __ldg(pcurr + (int64_t)(zs - 1) * pstride + g);
    float f0 = zs < ze ? __ldg(pcurr + (int64_t)zs * pstride + g) : 0.f;
    for (int z = zs; z < ze; ++z) {
        const int64_t i = (int64_t)z * pstride + g;
        const float fp = __ldg(pcurr + i + pstride);
        const float f2 = __fadd_rn(f0, f0);
        const float dx = __fsub_rn(__fadd_rn(__ldg(pcurr + i - 1), __ldg(pcurr + i + 1)), f2);
        const float dy = __fsub_rn(__fadd_rn(__ldg(pcurr + i - pitch), __ldg(pcurr + i + pitch)), f2);
        const float dz = __fsub_rn(__fadd_rn(fm, fp), f2);
        const float lap = __fadd_rn(__fadd_rn(dx, dy), dz);
        const float vd = __fmul_rn(__ldg(vel + i), dt);
        pprev[i] = __fmaf_rn(__fmul_rn(vd, vd), lap, __fsub_rn(f2, pprev[i]));
        fm = f0;
        f0 = fp;
    }
}

cudaError_t launch_step(const float *vel, float *pprev, const float *pcurr, int64_t ax, int64_t ay, int64_t pitch,
                        int64_t planes, int64_t z_lo, int64_t z_hi, float dt, int stencil, cudaStream_t st) {
    if (stencil == OOCS_STENCIL_STAR7) {
        if (z_hi <= z_lo) return cudaSuccess;
        const int nx = (int)(ax - 2 * R), ny = (int)(ay - 2 * R), Z = (int)(z_hi - z_lo);
        const int tiles = ((nx + 31) / 32) * ((ny + 7) / 8);
        const int nzc = std::max(1, std::min(Z, (148 * 8 + tiles - 1) / tiles));
        const int zchunk = (Z + nzc - 1) / nzc;
        const dim3 grid((nx + 31) / 32, (ny + 7) / 8, (Z + zchunk - 1) / zchunk);
        star7_step_kernel<<<grid, dim3(32, 8), 0, st>>>(vel, pprev, pcurr, nx, ny, (int)z_lo, (int)z_hi, zchunk, pitch,
                                                         ay * pitch, dt);
        return cudaGetLastError();
    }
    StepArgs a{};
    return launch_stencil<16, 0>(vel, pprev, pcurr, ax, ay, pitch, planes, z_lo, z_hi, dt, a, st);
}

bool step_fused_ok(int q) { return q <= 15 && (q & 1); }

cudaError_t launch_step_fused(const float *vel, float *pprev, const float *pcurr, const void *rec_pprev, int64_t ax,
                              int64_t ay, int64_t pitch, int64_t planes, int64_t z_lo, int64_t z_hi, float dt, int q,
                              cudaStream_t st) {
    // whole slabs of 16-byte aligned records
    if (!step_fused_ok(q) || (z_lo & 3) || (reinterpret_cast<uintptr_t>(rec_pprev) & 15)) return cudaErrorInvalidValue;
    StepArgs a{};
    a.rec[0] = static_cast<const uint32_t *>(rec_pprev);
    a.nbx = (int)(ax / 4);
    a.nby = (int)(ay / 4);
    a.q = q;
    a.recw = 2 * (q + 1);
    return launch_stencil<16, 1>(vel, pprev, pcurr, ax, ay, pitch, planes, z_lo, z_hi, dt, a, st);
}

// max |x| over rows of n floats (CFL check of a loaded velocity); float bits of non-negative values order
// like unsigned integers, and NaN's bits exceed +Inf's
__global__ void __launch_bounds__(256) absmax_kernel(const float *__restrict__ src, int64_t rows, int64_t n,
                                                     int64_t pitch, uint32_t *out) {
    uint32_t m = 0;
    const int64_t total = rows * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / n, c = i - r * n;
        m = max(m, __float_as_uint(src[r * pitch + c]) & 0x7fffffffu);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

cudaError_t launch_absmax(const float *src, int64_t rows, int64_t n, int64_t pitch, uint32_t *out, cudaStream_t st) {
    if (rows <= 0 || n <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>(148 * 8, (rows * n + 255) / 256);
    absmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, rows, n, pitch, out);
    return cudaGetLastError();
}


}  // namespace oocs
