// Hot-path kernels for sm_100a: fixed-rate BlockQuant decode/encode (P:L116,
// P:L153) and the 25-point acoustic-wave leapfrog step (P:L163,
// P:L212).  All three are HBM-bound streaming kernels (no dense contraction:
// tensor cores do not apply); see DESIGN.md §6 for their rooflines.
//
// Working-buffer layout (shared with runtime.cu): planes x ay rows x pitch
// floats, element x of a row at column x + XOFF (XOFF = 28) so interior x = R
// starts on a 128-byte line; pitch is a multiple of 32 floats.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "oocs_internal.h"

namespace oocs {

// ---------------------------------------------------------------------------
// Warp-level 32x32 bit-matrix transpose: lane l holds row l (32 bits); on
// return lane m holds column m (bit l = bit m of row l).  5 butterfly stages
// of shfl.xor + funnel/select + LOP3; this is the bit-plane (de)interleave of
// the codec ("warp-level bit-plane packing", north star).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t m = (j == 16) ? 0x0000FFFFu
                         : (j == 8)  ? 0x00FF00FFu
                         : (j == 4)  ? 0x0F0F0F0Fu
                         : (j == 2)  ? 0x33333333u
                                     : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool upper = (lane & j) == 0;
        const uint32_t s = upper ? (y << j) : (y >> j);
        const uint32_t keep = upper ? m : ~m;
        x = (x & keep) | (s & ~keep);
    }
    return x;
}

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// Warp task = one 128-byte line segment of 16 rows (4 y x 4 z) of a
// 4-plane slab: the blocks bx in [max(0,8L-7), min(nbx-1,8L)] whose columns
// lie in line L (column of x is x + 28, block bx covers x in [4bx, 4bx+4)).
struct LineTask {
    int bz, by, b0, nb;
};
__device__ __forceinline__ LineTask line_task(int64_t task, int nbx, int nby, int nlines) {
    LineTask t;
    const int L = (int)(task % nlines);
    const int64_t rest = task / nlines;
    t.by = (int)(rest % nby);
    t.bz = (int)(rest / nby);
    t.b0 = L == 0 ? 0 : 8 * L - 7;
    const int b1 = min(nbx - 1, 8 * L);
    t.nb = b1 - t.b0 + 1;
    return t;
}

constexpr int CODEC_WARPS = 8;
constexpr int TILE_LD = 36;  // padded row (floats): conflict-free scatter of 4x4 block rows

// ---------------------------------------------------------------------------
// BlockQuant decode: compressed slab-major records -> working buffer.
// x^_j = fma((float)code_j + 0.5f, step, mn), step = fl(fl(mx-mn) * 2^-q)
// ---------------------------------------------------------------------------
template <bool TWO>
__global__ void __launch_bounds__(CODEC_WARPS * 32)
bq_decode_kernel(const uint8_t *__restrict__ src, float *__restrict__ dst, int nbx, int nby,
                 int64_t ntasks, int nlines, int64_t pitch, int64_t pstride, int q) {
    __shared__ __align__(16) float tile[CODEC_WARPS][16][TILE_LD];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t task = (int64_t)blockIdx.x * CODEC_WARPS + warp;
    if (task >= ntasks) return;
    const LineTask t = line_task(task, nbx, nby, nlines);
    const int recw = 2 * (q + 1);  // record size in 32-bit words
    const uint32_t *rec0 = reinterpret_cast<const uint32_t *>(src) +
                           ((int64_t)(t.bz * nby + t.by) * nbx + t.b0) * recw;
    const float twomq = pow2f(-q);
    const int b = lane & 15, half = lane >> 4;
    const int xi = lane & 3, yi = (lane >> 2) & 3, zi = lane >> 4;
    float(*tl)[TILE_LD] = tile[warp];
    for (int i = 0; i < t.nb; ++i) {
        const uint32_t *rec = rec0 + (int64_t)i * recw;
        const float mn = __uint_as_float(__ldg(rec)), mx = __uint_as_float(__ldg(rec + 1));
        const uint32_t w0 = (b < q) ? __ldg(rec + 2 + 2 * (q - 1 - b) + half) : 0u;
        uint32_t c_lo, c_hi;
        {
            const uint32_t y0 = warp_transpose32(w0, lane);
            c_lo = y0 & 0xFFFFu;
            c_hi = y0 >> 16;
        }
        if (TWO) {
            const int b2 = 16 + b;
            const uint32_t w1 = (b2 < q) ? __ldg(rec + 2 + 2 * (q - 1 - b2) + half) : 0u;
            const uint32_t y1 = warp_transpose32(w1, lane);
            c_lo |= (y1 & 0xFFFFu) << 16;
            c_hi |= (y1 >> 16) << 16;
        }
        const float step = __fmul_rn(__fsub_rn(mx, mn), twomq);
        const float v_lo = __fmaf_rn(__fadd_rn(__uint2float_rn(c_lo), 0.5f), step, mn);
        const float v_hi = __fmaf_rn(__fadd_rn(__uint2float_rn(c_hi), 0.5f), step, mn);
        tl[yi + 4 * zi][4 * i + xi] = v_lo;
        tl[yi + 4 * (zi + 2)][4 * i + xi] = v_hi;
    }
    __syncwarp();
    const int col0 = XOFF + 4 * t.b0;
    for (int f = lane; f < 16 * t.nb; f += 32) {
        const int r = f / t.nb, c = f - r * t.nb;
        const float4 v = *reinterpret_cast<const float4 *>(&tl[r][4 * c]);
        float *d = dst + (int64_t)(4 * t.bz + (r >> 2)) * pstride + (int64_t)(4 * t.by + (r & 3)) * pitch +
                   col0 + 4 * c;
        *reinterpret_cast<float4 *>(d) = v;
    }
}

// ---------------------------------------------------------------------------
// BlockQuant encode: working buffer -> compressed records (bit-exact with
// oracle_bq_encode_block: same IEEE binary32 operations in the same order).
// ---------------------------------------------------------------------------
template <bool TWO>
__global__ void __launch_bounds__(CODEC_WARPS * 32)
bq_encode_kernel(const float *__restrict__ src, uint8_t *__restrict__ dst, int nbx, int nby,
                 int64_t ntasks, int nlines, int64_t pitch, int64_t pstride, int q, int *err) {
    __shared__ __align__(16) float tile[CODEC_WARPS][16][TILE_LD];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t task = (int64_t)blockIdx.x * CODEC_WARPS + warp;
    if (task >= ntasks) return;
    const LineTask t = line_task(task, nbx, nby, nlines);
    float(*tl)[TILE_LD] = tile[warp];
    const int col0 = XOFF + 4 * t.b0;
    for (int f = lane; f < 16 * t.nb; f += 32) {
        const int r = f / t.nb, c = f - r * t.nb;
        const float *s = src + (int64_t)(4 * t.bz + (r >> 2)) * pstride +
                         (int64_t)(4 * t.by + (r & 3)) * pitch + col0 + 4 * c;
        *reinterpret_cast<float4 *>(&tl[r][4 * c]) = __ldcs(reinterpret_cast<const float4 *>(s));
    }
    __syncwarp();
    const int recw = 2 * (q + 1);
    uint32_t *rec0 = reinterpret_cast<uint32_t *>(dst) + ((int64_t)(t.bz * nby + t.by) * nbx + t.b0) * recw;
    const float twomq = pow2f(-q), twoq = pow2f(q);
    const uint32_t cmax = (1u << q) - 1u;
    const int xi = lane & 3, yi = (lane >> 2) & 3, zi = lane >> 4;
    const int b = lane & 15, half = lane >> 4;
    bool bad = false;
    for (int i = 0; i < t.nb; ++i) {
        float x_lo = __fadd_rn(tl[yi + 4 * zi][4 * i + xi], 0.0f);  // -0 -> +0
        float x_hi = __fadd_rn(tl[yi + 4 * (zi + 2)][4 * i + xi], 0.0f);
        bad |= !(fabsf(x_lo) < 0x1p126f) || !(fabsf(x_hi) < 0x1p126f);
        float mn = fminf(x_lo, x_hi), mx = fmaxf(x_lo, x_hi);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        const float range = __fsub_rn(mx, mn);
        const float step = __fmul_rn(range, twomq);
        uint32_t c_lo = 0, c_hi = 0;
        if (step >= 0x1p-126f) {
            const float scale = __fdiv_rn(twoq, range);
            c_lo = min(cmax, __float2uint_rd(__fmul_rn(__fsub_rn(x_lo, mn), scale)));
            c_hi = min(cmax, __float2uint_rd(__fmul_rn(__fsub_rn(x_hi, mn), scale)));
        }
        uint32_t *rec = rec0 + (int64_t)i * recw;
        const uint32_t T0 = warp_transpose32((c_lo & 0xFFFFu) | (c_hi << 16), lane);
        if (b < q) rec[2 + 2 * (q - 1 - b) + half] = T0;
        if (TWO) {
            const uint32_t T1 = warp_transpose32((c_lo >> 16) | ((c_hi >> 16) << 16), lane);
            const int b2 = 16 + b;
            if (b2 < q) rec[2 + 2 * (q - 1 - b2) + half] = T1;
        }
        // lanes 15 and 31 always carry an unused plane slot (q <= 15, or b2 = 31 >= q)
        if (lane == 15) rec[0] = __float_as_uint(mn);
        if (lane == 31) rec[1] = __float_as_uint(mx);
    }
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
// 25-point leapfrog step:
//   p_prev <- 2 p_curr - p_prev + (v dt)^2 * sum_axes sum_m c_m ((f(+m) + f(-m)) - 2 f0)
// 2.5-D blocking: a CTA owns a 32x32 xy tile and marches a z range; the
// current xy plane (+4-cell star halo) is staged in double-buffered shared
// memory, the z column lives in a 9-deep register queue, pprev/v/halo are
// prefetched one plane ahead.  Each thread computes 2 y-adjacent cells.
// ---------------------------------------------------------------------------
constexpr int ST_TX = 32, ST_TY = 16, ST_SY = 32;  // threads x, threads y, tile rows
constexpr int ST_THREADS = ST_TX * ST_TY;
constexpr int ST_W = ST_TX + 2 * R;                // 40 smem columns
constexpr int ST_H = ST_SY + 2 * R;                // 40 smem rows

// coefficients of d2/dx2, order 8 (Q1): 8/5, -1/5, 8/315, -1/560
#define C1 1.6f
#define C2 (-0.2f)
#define C3 0.025396825396825397f
#define C4 (-0.0017857142857142857f)

__global__ void __launch_bounds__(ST_THREADS, 2)
stencil_step_kernel(const float *__restrict__ vel, float *__restrict__ pprev, const float *__restrict__ pcurr,
                    int nx, int ny, int64_t pitch, int64_t pstride, int z_lo, int z_hi, int zchunk, float dt) {
    __shared__ float sm[2][ST_H][ST_W];
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * ST_TX, y0 = blockIdx.y * ST_SY;
    const int zs = z_lo + blockIdx.z * zchunk;
    const int ze = min(z_hi, zs + zchunk);
    if (zs >= ze) return;
    const int x = x0 + tx;
    const int ya = y0 + 2 * ty, yb = ya + 1;
    // compute flags (interior cells) and load flags (cells inside the allocated grid)
    const bool oka = x < nx && ya < ny, okb = x < nx && yb < ny;
    const bool lda = x < nx + R && ya < ny + R, ldb = x < nx + R && yb < ny + R;
    // element (interior x, y, plane z) at z*pstride + (y+R)*pitch + x + R + XOFF = ... + x + 32
    const int64_t ia = (int64_t)(ya + R) * pitch + x + 32;
    const int64_t ib = ia + pitch;
    // halo cell owned by this thread (star stencil: no corners)
    int hr, hc;  // smem row/col
    if (tid < 256) {
        const int r = tid >> 5;
        hr = r < 4 ? r : r + ST_SY;
        hc = R + (tid & 31);
    } else {
        const int u = tid - 256;
        hr = R + (u >> 3);
        const int c = u & 7;
        hc = c < 4 ? c : c + ST_TX;
    }
    const int hx = x0 - R + hc, hy = y0 - R + hr;  // interior coords of the halo cell
    const bool okh = hx < nx + R && hy < ny + R;   // >= -R always
    const int64_t ih = (int64_t)(hy + R) * pitch + hx + 32;

    float qa[9], qb[9];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t zo = (int64_t)(zs - R + i) * pstride;
        qa[i] = lda ? __ldg(pcurr + zo + ia) : 0.f;
        qb[i] = ldb ? __ldg(pcurr + zo + ib) : 0.f;
    }
    int64_t zo = (int64_t)zs * pstride;
    qa[8] = lda ? __ldg(pcurr + zo + (int64_t)R * pstride + ia) : 0.f;
    qb[8] = ldb ? __ldg(pcurr + zo + (int64_t)R * pstride + ib) : 0.f;
    float ppa = oka ? __ldcs(pprev + zo + ia) : 0.f, ppb = okb ? __ldcs(pprev + zo + ib) : 0.f;
    float va = oka ? __ldcs(vel + zo + ia) : 0.f, vb = okb ? __ldcs(vel + zo + ib) : 0.f;
    float hv = okh ? __ldg(pcurr + zo + ih) : 0.f;

    const int sy = R + 2 * ty, sx = R + tx;
    for (int z = zs; z < ze; ++z) {
        float(*s)[ST_W] = sm[z & 1];
        s[sy][sx] = qa[4];
        s[sy + 1][sx] = qb[4];
        s[hr][hc] = hv;
        // prefetch plane z+1 (and z+5 for the queue)
        float na = 0.f, nb = 0.f, npa = 0.f, npb = 0.f, nva = 0.f, nvb = 0.f, nh = 0.f;
        if (z + 1 < ze) {
            const int64_t zn = (int64_t)(z + 1) * pstride;
            const int64_t zq = zn + (int64_t)R * pstride;
            if (lda) na = __ldg(pcurr + zq + ia);
            if (ldb) nb = __ldg(pcurr + zq + ib);
            if (oka) { npa = __ldcs(pprev + zn + ia); nva = __ldcs(vel + zn + ia); }
            if (okb) { npb = __ldcs(pprev + zn + ib); nvb = __ldcs(vel + zn + ib); }
            if (okh) nh = __ldg(pcurr + zn + ih);
        }
        __syncthreads();
        // y-neighbour rows sy-4 .. sy+5 shared by the two cells
        float col[10];
#pragma unroll
        for (int m = 0; m < 10; ++m) col[m] = s[sy - R + m][sx];
        {
            const float f0 = qa[4], f2 = __fadd_rn(f0, f0);
            float lap = __fmul_rn(C1, __fsub_rn(__fadd_rn(s[sy][sx - 1], s[sy][sx + 1]), f2));
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(s[sy][sx - 2], s[sy][sx + 2]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(s[sy][sx - 3], s[sy][sx + 3]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(s[sy][sx - 4], s[sy][sx + 4]), f2), lap);
            lap = __fmaf_rn(C1, __fsub_rn(__fadd_rn(col[3], col[5]), f2), lap);
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(col[2], col[6]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(col[1], col[7]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(col[0], col[8]), f2), lap);
            lap = __fmaf_rn(C1, __fsub_rn(__fadd_rn(qa[3], qa[5]), f2), lap);
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(qa[2], qa[6]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(qa[1], qa[7]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(qa[0], qa[8]), f2), lap);
            const float vd = __fmul_rn(va, dt);
            const float c = __fmul_rn(vd, vd);
            if (oka) pprev[(int64_t)z * pstride + ia] = __fmaf_rn(c, lap, __fsub_rn(f2, ppa));
        }
        {
            const float f0 = qb[4], f2 = __fadd_rn(f0, f0);
            float lap = __fmul_rn(C1, __fsub_rn(__fadd_rn(s[sy + 1][sx - 1], s[sy + 1][sx + 1]), f2));
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(s[sy + 1][sx - 2], s[sy + 1][sx + 2]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(s[sy + 1][sx - 3], s[sy + 1][sx + 3]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(s[sy + 1][sx - 4], s[sy + 1][sx + 4]), f2), lap);
            lap = __fmaf_rn(C1, __fsub_rn(__fadd_rn(col[4], col[6]), f2), lap);
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(col[3], col[7]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(col[2], col[8]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(col[1], col[9]), f2), lap);
            lap = __fmaf_rn(C1, __fsub_rn(__fadd_rn(qb[3], qb[5]), f2), lap);
            lap = __fmaf_rn(C2, __fsub_rn(__fadd_rn(qb[2], qb[6]), f2), lap);
            lap = __fmaf_rn(C3, __fsub_rn(__fadd_rn(qb[1], qb[7]), f2), lap);
            lap = __fmaf_rn(C4, __fsub_rn(__fadd_rn(qb[0], qb[8]), f2), lap);
            const float vd = __fmul_rn(vb, dt);
            const float c = __fmul_rn(vd, vd);
            if (okb) pprev[(int64_t)z * pstride + ib] = __fmaf_rn(c, lap, __fsub_rn(f2, ppb));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            qa[i] = qa[i + 1];
            qb[i] = qb[i + 1];
        }
        qa[8] = na;
        qb[8] = nb;
        ppa = npa; ppb = npb; va = nva; vb = nvb; hv = nh;
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline int64_t nlines_of(int64_t ax) { return (XOFF + ax + 31) / 32; }

cudaError_t launch_decode(const void *src, float *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch,
                          int codec, int q, cudaStream_t st) {
    if (planes <= 0) return cudaSuccess;
    const int64_t pstride = ay * pitch;
    if (codec == 0) {
        const int64_t n4 = planes * ay * (ax / 4);
        const int threads = 256;
        const int64_t blocks = std::min<int64_t>((n4 + threads - 1) / threads, 148 * 16);
        id_decode_kernel<<<(unsigned)blocks, threads, 0, st>>>(static_cast<const float4 *>(src), dst, n4,
                                                              (int)(ax / 4), pitch);
        return cudaGetLastError();
    }
    const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
    const int nl = (int)nlines_of(ax);
    const int64_t ntasks = (planes / 4) * nby * (int64_t)nl;
    const int64_t blocks = (ntasks + CODEC_WARPS - 1) / CODEC_WARPS;
    if (q > 16)
        bq_decode_kernel<true><<<(unsigned)blocks, CODEC_WARPS * 32, 0, st>>>(
            static_cast<const uint8_t *>(src), dst, nbx, nby, ntasks, nl, pitch, pstride, q);
    else
        bq_decode_kernel<false><<<(unsigned)blocks, CODEC_WARPS * 32, 0, st>>>(
            static_cast<const uint8_t *>(src), dst, nbx, nby, ntasks, nl, pitch, pstride, q);
    return cudaGetLastError();
}

cudaError_t launch_encode(const float *src, void *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch,
                          int codec, int q, int *err, cudaStream_t st) {
    if (planes <= 0) return cudaSuccess;
    const int64_t pstride = ay * pitch;
    if (codec == 0) {
        const int64_t n4 = planes * ay * (ax / 4);
        const int threads = 256;
        const int64_t blocks = std::min<int64_t>((n4 + threads - 1) / threads, 148 * 16);
        id_encode_kernel<<<(unsigned)blocks, threads, 0, st>>>(src, static_cast<float4 *>(dst), n4,
                                                              (int)(ax / 4), pitch);
        return cudaGetLastError();
    }
    const int nbx = (int)(ax / 4), nby = (int)(ay / 4);
    const int nl = (int)nlines_of(ax);
    const int64_t ntasks = (planes / 4) * nby * (int64_t)nl;
    const int64_t blocks = (ntasks + CODEC_WARPS - 1) / CODEC_WARPS;
    if (q > 16)
        bq_encode_kernel<true><<<(unsigned)blocks, CODEC_WARPS * 32, 0, st>>>(
            src, static_cast<uint8_t *>(dst), nbx, nby, ntasks, nl, pitch, pstride, q, err);
    else
        bq_encode_kernel<false><<<(unsigned)blocks, CODEC_WARPS * 32, 0, st>>>(
            src, static_cast<uint8_t *>(dst), nbx, nby, ntasks, nl, pitch, pstride, q, err);
    return cudaGetLastError();
}

cudaError_t launch_step(const float *vel, float *pprev, const float *pcurr, int64_t ax, int64_t ay, int64_t pitch,
                        int64_t z_lo, int64_t z_hi, float dt, cudaStream_t st) {
    if (z_hi <= z_lo) return cudaSuccess;
    const int nx = (int)(ax - 2 * R), ny = (int)(ay - 2 * R);
    const int gx = (nx + ST_TX - 1) / ST_TX, gy = (ny + ST_SY - 1) / ST_SY;
    const int Z = (int)(z_hi - z_lo);
    const int resident = 148 * 2;
    int nzc = (3 * resident + gx * gy - 1) / (gx * gy);
    nzc = std::max(1, std::min(nzc, Z / 32));
    const int zchunk = (Z + nzc - 1) / nzc;
    nzc = (Z + zchunk - 1) / zchunk;
    dim3 grid(gx, gy, nzc);
    stencil_step_kernel<<<grid, ST_THREADS, 0, st>>>(vel, pprev, pcurr, nx, ny, pitch, ay * pitch, (int)z_lo,
                                                     (int)z_hi, zchunk, dt);
    return cudaGetLastError();
}

}  // namespace oocs
