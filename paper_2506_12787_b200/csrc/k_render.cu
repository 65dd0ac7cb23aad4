// Per-(position, Gaussian) setup, tile binning (count -> scan -> emit ->
// stable one-digit radix sort keyed on (position, tile), primitive order kept),
// tile rasterisation and the AoA / pooled-magnitude / RSSI heads.
//
// Reference: splat::rasterize and its prepare() (/root/reference/proj/src/splat.cpp:159-482),
// tasks::pooled_magnitude / aoa_extract (tasks.cpp:32-39, 154-169).
//
// Bit-exactness: every float operation whose rounding reaches the bins, the
// render state or a cutoff mask is written as an explicit _rn intrinsic (no FMA
// contraction), mirroring the reference's expression order. Bins additionally
// depend only on FP64 ops whose float inputs multiply exactly.
#include "swr_internal.h"

#include <type_traits>

#include <cfloat>

namespace swr
{

namespace
{
__device__ __forceinline__ float fmaxr(float a, float b) { return (a < b) ? b : a; } // std::max
__device__ __forceinline__ float fminr(float a, float b) { return (b < a) ? b : a; } // std::min

// splat.cpp:72-82
__device__ __forceinline__ float wrap_pm_pi(float x)
{
    if (x < (float)(-8 * kPi) || x > (float)(8 * kPi))
        x = fmodf(x, (float)(2 * kPi));
    while (x >= (float)kPi)
        x = __fsub_rn(x, (float)(2 * kPi));
    while (x < (float)(-kPi))
        x = __fadd_rn(x, (float)(2 * kPi));
    return x;
}

// Tiles of one primitive, splat.cpp:255-282 (count only)
__device__ __forceinline__ int tile_count(const Grid &g, int r0, int r1, int j0, int len)
{
    if (r1 < r0)
        return 0;
    const int ntr = r1 / g.tile - r0 / g.tile + 1;
    int ntc;
    if (len >= g.W)
        ntc = g.tw;
    else
    {
        const int jend = j0 + len - 1;
        ntc = min(jend, g.W - 1) / g.tile - j0 / g.tile + 1;
        if (jend >= g.W)
        {
            const int e1 = min((jend - g.W) / g.tile, j0 / g.tile - 1);
            ntc += e1 >= 0 ? e1 + 1 : 0;
        }
    }
    return ntr * ntc;
}

struct PrimOut
{
    float el, az, delta, re, im;
};

// splat.cpp:94-118 with host-precomputed el0/az0/delta0 (bit-identical to the
// reference's glibc tanhf/expf results)
__device__ __forceinline__ PrimOut deform_prim(const SceneDev &s, const float *res, int64_t plane, int g, bool with_res)
{
    PrimOut p;
    p.el = s.el0[g];
    p.az = s.az0[g];
    p.delta = s.delta0[g];
    p.re = s.re0[g];
    p.im = s.im0[g];
    if (with_res)
    {
        p.el = __fadd_rn(p.el, res[0 * plane + g]);
        p.az = __fadd_rn(p.az, res[1 * plane + g]);
        p.re = __fadd_rn(p.re, res[2 * plane + g]);
        p.im = __fadd_rn(p.im, res[3 * plane + g]);
        p.delta = fminr(fmaxr(__fadd_rn(p.delta, res[4 * plane + g]), 0.0f), 1.0f);
    }
    return p;
}

// bbox rows/cols (splat.cpp:197-248); returns (r0, r1, j0, len), rows empty = (0, -1)
__device__ __forceinline__ int4 bbox_of(const Grid &g, float el, float az, float delta, double2 h)
{
    if (delta <= 0.0f)
        return make_int4(0, -1, 0, 0);
    if (!g.cut)
        return make_int4(0, g.H - 1, 0, g.W);
    int r0 = (int)floor(__dsub_rn(__ddiv_rn(__dsub_rn((double)el, h.x), g.cell_el), 0.5));
    int r1 = (int)ceil(__dsub_rn(__ddiv_rn(__dadd_rn((double)el, h.x), g.cell_el), 0.5));
    r0 = max(r0, 0);
    r1 = min(r1, g.H - 1);
    if (r0 > r1)
        return make_int4(0, -1, 0, 0);
    if (__dmul_rn(2.0, h.y) >= __dmul_rn((double)g.W, g.cell_az))
        return make_int4(r0, r1, 0, g.W);
    int j0 = (int)floor(__dsub_rn(__ddiv_rn(__dsub_rn((double)az, h.y), g.cell_az), 0.5));
    const int j1 = (int)ceil(__dsub_rn(__ddiv_rn(__dadd_rn((double)az, h.y), g.cell_az), 0.5));
    const int len = min(j1 - j0 + 1, g.W);
    j0 = ((j0 % g.W) + g.W) % g.W;
    return make_int4(r0, r1, j0, len);
}
} // namespace

// ------------------------------------------------------------------------ setup

// One thread per (position, 4 consecutive Gaussians): float4 loads of the
// planar residuals and static SoA; writes dyn (el, az, k_re, k_im), the
// row/column ranges and the tile count.
__global__ void __launch_bounds__(256) setup_kernel(Grid g, SceneDev sd, const float *__restrict__ res, int64_t plane,
                                                    float4 *__restrict__ dyn, int4 *__restrict__ rng, int *__restrict__ cnt,
                                                    int with_res, int64_t *__restrict__ nonfinite,
                                                    const int64_t *__restrict__ gate)
{
    if (gate && *gate == 0)
        return;
    const int s = blockIdx.y;
    const int g4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (g4 >= g.np)
        return;
    const int64_t base = (int64_t)s * g.np;
    float r_el[4], r_az[4], r_re[4], r_im[4], r_dl[4];
    const float4 e0 = *reinterpret_cast<const float4 *>(sd.el0 + g4);
    const float4 a0 = *reinterpret_cast<const float4 *>(sd.az0 + g4);
    const float4 d0 = *reinterpret_cast<const float4 *>(sd.delta0 + g4);
    const float4 re = *reinterpret_cast<const float4 *>(sd.re0 + g4);
    const float4 im = *reinterpret_cast<const float4 *>(sd.im0 + g4);
    r_el[0] = e0.x; r_el[1] = e0.y; r_el[2] = e0.z; r_el[3] = e0.w;
    r_az[0] = a0.x; r_az[1] = a0.y; r_az[2] = a0.z; r_az[3] = a0.w;
    r_dl[0] = d0.x; r_dl[1] = d0.y; r_dl[2] = d0.z; r_dl[3] = d0.w;
    r_re[0] = re.x; r_re[1] = re.y; r_re[2] = re.z; r_re[3] = re.w;
    r_im[0] = im.x; r_im[1] = im.y; r_im[2] = im.z; r_im[3] = im.w;
    if (with_res)
    {
        const float *rb = res + base;
        const float4 x0 = *reinterpret_cast<const float4 *>(rb + 0 * plane + g4);
        const float4 x1 = *reinterpret_cast<const float4 *>(rb + 1 * plane + g4);
        const float4 x2 = *reinterpret_cast<const float4 *>(rb + 2 * plane + g4);
        const float4 x3 = *reinterpret_cast<const float4 *>(rb + 3 * plane + g4);
        const float4 x4 = *reinterpret_cast<const float4 *>(rb + 4 * plane + g4);
        const float v0[4] = {x0.x, x0.y, x0.z, x0.w}, v1[4] = {x1.x, x1.y, x1.z, x1.w};
        const float v2[4] = {x2.x, x2.y, x2.z, x2.w}, v3[4] = {x3.x, x3.y, x3.z, x3.w};
        const float v4[4] = {x4.x, x4.y, x4.z, x4.w};
        if (nonfinite)
        {
            // an fp16 overflow in the tensor-core MLP surfaces here as NaN (k_mlp_tc2.cu)
            bool bad = false;
#pragma unroll
            for (int k = 0; k < 4; k++)
                bad |= !isfinite(v0[k]) || !isfinite(v1[k]) || !isfinite(v2[k]) || !isfinite(v3[k]) || !isfinite(v4[k]);
            if (bad && g4 < g.n)
                *nonfinite = 1;
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
        {
            r_el[k] = __fadd_rn(r_el[k], v0[k]);
            r_az[k] = __fadd_rn(r_az[k], v1[k]);
            r_re[k] = __fadd_rn(r_re[k], v2[k]);
            r_im[k] = __fadd_rn(r_im[k], v3[k]);
            r_dl[k] = fminr(fmaxr(__fadd_rn(r_dl[k], v4[k]), 0.0f), 1.0f);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; k++)
    {
        const int gi = g4 + k;
        int4 b = make_int4(0, -1, 0, 0);
        if (gi < g.n)
            b = bbox_of(g, r_el[k], r_az[k], r_dl[k], sd.half[gi]);
        dyn[base + gi] = make_float4(r_el[k], r_az[k], __fmul_rn(r_re[k], r_dl[k]), __fmul_rn(r_im[k], r_dl[k]));
        rng[base + gi] = b;
        cnt[base + gi] = gi < g.n ? tile_count(g, b.x, b.y, b.z, b.w) : 0;
    }
}

void launch_setup(Ctx &c, int nb, bool with_res, cudaStream_t st)
{
    dim3 grid((c.g.np / 4 + 255) / 256, nb);
    if (grid.x == 0) // empty Gaussian set: nothing to set up (the counts are never read)
        return;
    setup_kernel<<<grid, 256, 0, st>>>(c.g, c.s, c.w.res, c.w.cap_b * c.g.np, c.w.dyn, c.w.rng, c.w.cnt, with_res,
                                       with_res ? c.w.stats + 2 : nullptr, c.gate);
    c.launches++;
}

// The reference's 11-float render state (splat.cpp:133-147, 200-211); all
// zero when delta <= 0 (splat.cpp:197-198). Parity hook only.
__global__ void state_out_kernel(Grid g, SceneDev sd, const float *__restrict__ res, int64_t plane, int with_res,
                                 float *__restrict__ state, int nb)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nb * g.n)
        return;
    const int s = (int)(idx / g.n), gi = (int)(idx % g.n);
    const PrimOut p = deform_prim(sd, res + (int64_t)s * g.np, plane, gi, with_res);
    float *st = state + idx * kStateStride;
    if (p.delta <= 0.0f)
    {
        for (int k = 0; k < kStateStride; k++)
            st[k] = 0.0f;
        return;
    }
    const float4 sh = sd.shape[gi];
    st[0] = p.el;
    st[1] = p.az;
    st[2] = sh.x;
    st[3] = sh.y;
    st[4] = sh.z;
    st[5] = p.delta;
    st[6] = p.re;
    st[7] = p.im;
    st[8] = sh.w;
    st[9] = sd.inv_l3[gi];
    st[10] = sd.l2[gi];
}

void launch_state_out(Ctx &c, int nb, bool with_res, float *d_state, cudaStream_t st)
{
    const int64_t total = (int64_t)nb * c.g.n;
    state_out_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(c.g, c.s, c.w.res, c.w.cap_b * c.g.np,
                                                                      with_res ? 1 : 0,
                                                                      d_state, nb);
    c.launches++;
}

// ---------------------------------------------------------------- bin: counts

// Block-wide exclusive scan helper (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ int block_excl_scan(int v, int *warp_sums, int &total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
    {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0)
    {
        int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
        {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o)
                w += y;
        }
        if (lane < nw)
            warp_sums[lane] = w;
    }
    __syncthreads();
    const int before = (wid > 0 ? warp_sums[wid - 1] : 0) + x - v;
    total = warp_sums[nw - 1];
    __syncthreads();
    return before;
}

// One CTA per position: exclusive scan of per-primitive tile counts (the pair
// offsets of each primitive inside its position's segment).
__global__ void __launch_bounds__(1024) seg_scan_kernel(const int *__restrict__ cnt, int *__restrict__ poff,
                                                        int64_t *__restrict__ seg_len, int np, int n,
                                                        const int64_t *__restrict__ gate)
{
    __shared__ int ws[32];
    if (gate && *gate == 0)
        return;
    const int s = blockIdx.x;
    const int *c = cnt + (int64_t)s * np;
    int *o = poff + (int64_t)s * np;
    int carry = 0;
    for (int base = 0; base < n; base += 4 * blockDim.x)
    {
        const int i0 = base + 4 * threadIdx.x;
        int v[4], sum = 0;
#pragma unroll
        for (int k = 0; k < 4; k++)
        {
            v[k] = (i0 + k < n) ? c[i0 + k] : 0;
            sum += v[k];
        }
        int total;
        int run = block_excl_scan(sum, ws, total) + carry;
#pragma unroll
        for (int k = 0; k < 4; k++)
        {
            if (i0 + k < n)
                o[i0 + k] = run;
            run += v[k];
        }
        carry += total;
    }
    if (threadIdx.x == 0)
        seg_len[s] = carry;
}

// Exclusive scan over the position segments (one CTA): seg[s] = first pair of
// position s, seg[nb] = total; out[0] = total, out[1] = longest segment.
__global__ void __launch_bounds__(1024) seg_base_kernel(int64_t *__restrict__ seg, int nb, int64_t *__restrict__ out,
                                                        const int64_t *__restrict__ gate)
{
    __shared__ int64_t part[1024];
    __shared__ int64_t mx[1024];
    if (gate && *gate == 0)
        return;
    const int t = threadIdx.x;
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    int64_t sum = 0, m = 0;
    for (int k = 0; k < per; k++)
    {
        const int i = t * per + k;
        if (i < nb)
        {
            sum += seg[i];
            m = max(m, seg[i]);
        }
    }
    part[t] = sum;
    mx[t] = m;
    __syncthreads();
    if (t == 0)
    {
        int64_t run = 0, mm = 0;
        const int used = min((int)blockDim.x, (nb + per - 1) / max(per, 1)); // threads that hold positions
        for (int i = 0; i < used; i++)
        {
            const int64_t v = part[i];
            part[i] = run;
            run += v;
            mm = max(mm, mx[i]);
        }
        out[0] = run;
        out[1] = mm;
        seg[nb] = run; // total (seg[i < nb] are only rewritten below)
    }
    __syncthreads();
    int64_t run = part[t];
    for (int k = 0; k < per; k++)
    {
        const int i = t * per + k;
        if (i < nb)
        {
            const int64_t v = seg[i];
            seg[i] = run;
            run += v;
        }
    }
}

void launch_bin_count(Ctx &c, int nb, cudaStream_t st)
{
    // seg[] first receives the per-position lengths, then their exclusive scan
    seg_scan_kernel<<<nb, 1024, 0, st>>>(c.w.cnt, c.w.poff, c.w.seg, c.g.np, c.g.n, c.gate);
    seg_base_kernel<<<1, 1024, 0, st>>>(c.w.seg, nb, c.w.stats, c.gate);
    c.launches += 2;
}

// ------------------------------------------------------------ bin: emit + sort

// Emit (tile key, primitive) pairs in (position, primitive) order; the tiles of
// one primitive follow the reference's visit order (splat.cpp:255-282).
__global__ void __launch_bounds__(256) emit_kernel(Grid g, const int4 *__restrict__ rng, const int *__restrict__ poff,
                                                   const int64_t *__restrict__ seg, uint16_t *__restrict__ keys,
                                                   int *__restrict__ vals, int64_t cap)
{
    (void)cap;
    const int s = blockIdx.y;
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= g.n)
        return;
    const int4 b = rng[(int64_t)s * g.np + gi];
    if (b.y < b.x)
        return;
    int64_t o = seg[s] + poff[(int64_t)s * g.np + gi];
    const int tr0 = b.x / g.tile, tr1 = b.y / g.tile;
    auto col = [&](int tc) {
        for (int tr = tr0; tr <= tr1; tr++)
        {
            SWR_DCHECK(o >= seg[s] && o < seg[s + 1] && o < cap, "emit: pair outside its position's segment / buffer");
            SWR_DCHECK(tc >= 0 && tc < g.tw && tr >= 0 && tr < g.th, "emit: tile outside the grid");
            keys[o] = (uint16_t)(tr * g.tw + tc);
            vals[o] = gi;
            o++;
        }
    };
    if (b.w >= g.W)
    {
        for (int tc = 0; tc < g.tw; tc++)
            col(tc);
        return;
    }
    const int jend = b.z + b.w - 1;
    for (int tc = b.z / g.tile; tc <= min(jend, g.W - 1) / g.tile; tc++)
        col(tc);
    if (jend >= g.W)
        for (int tc = 0; tc <= min((jend - g.W) / g.tile, b.z / g.tile - 1); tc++)
            col(tc);
}

constexpr int kSortThreads = 256; // 8 warps, kSort / 8 pairs per warp per sort chunk

// Per (position, chunk of kSort pairs): histogram of tile keys.
__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const uint16_t *__restrict__ keys,
                                                                 const int64_t *__restrict__ seg, int *__restrict__ hist,
                                                                 int max_chunks, int tiles)
{
    extern __shared__ int h[];
    const int s = blockIdx.y;
    // chunks c = blockIdx.x, + gridDim.x, ... of this position's segment (the grid may
    // be sized below the segment's chunk count: the async path launches without it)
    for (int c = blockIdx.x;; c += gridDim.x)
    {
        const int64_t b = seg[s] + (int64_t)c * kSort, e = min(seg[s + 1], b + kSort);
        if (b >= e && c > 0)
            break;
        for (int t = threadIdx.x; t < tiles; t += blockDim.x)
            h[t] = 0;
        __syncthreads();
        // all of this thread's keys in flight first, then the shared-memory counts
        constexpr int kPer = kSort / kSortThreads;
        uint32_t kv[kPer];
#pragma unroll
        for (int r = 0; r < kPer; r++)
        {
            const int64_t i = b + threadIdx.x + (int64_t)r * kSortThreads;
            kv[r] = i < e ? (uint32_t)keys[i] : 0xffffffffu;
        }
#pragma unroll
        for (int r = 0; r < kPer; r++)
            if (kv[r] != 0xffffffffu)
            {
                SWR_DCHECK((int)kv[r] < tiles, "sort_hist: tile key out of range");
                atomicAdd(&h[kv[r]], 1);
            }
        __syncthreads();
        SWR_DCHECK(c < max_chunks, "sort_hist: chunk histogram overflow");
        int *out = hist + ((int64_t)s * max_chunks + c) * tiles;
        for (int t = threadIdx.x; t < tiles; t += blockDim.x)
            out[t] = h[t];
        __syncthreads();
    }
}

// Per position: CSR tile offsets (exclusive scan over tiles) and, in place,
// each chunk's starting offset per tile (tile-major, chunk-minor).
__global__ void __launch_bounds__(1024) sort_scan_kernel(const int64_t *__restrict__ seg, int *__restrict__ hist,
                                                         int *__restrict__ tile_off, int max_chunks, int tiles)
{
    __shared__ int ws[32];
    const int s = blockIdx.x, t = threadIdx.x;
    const int64_t len = seg[s + 1] - seg[s];
    const int nch = (int)((len + kSort - 1) / kSort);
    SWR_DCHECK(nch <= max_chunks, "sort_scan: more chunks than the histogram holds");
    int *hs = hist + (int64_t)s * max_chunks * tiles;
    int total_t = 0;
    if (t < tiles)
        for (int c = 0; c < nch; c++)
            total_t += hs[c * tiles + t];
    int all;
    const int off = block_excl_scan(total_t, ws, all);
    if (t < tiles)
    {
        tile_off[(int64_t)s * (tiles + 1) + t] = off;
        int run = off;
        for (int c = 0; c < nch; c++)
        {
            const int v = hs[c * tiles + t];
            hs[c * tiles + t] = run;
            run += v;
        }
    }
    if (t == 0)
        tile_off[(int64_t)s * (tiles + 1) + tiles] = (int)len;
}

// Stable scatter of one chunk: warp-level ranking with __match_any_sync keeps
// primitive order among equal tiles (a one-digit LSD radix pass).
__global__ void __launch_bounds__(kSortThreads) sort_scatter_kernel(const uint16_t *__restrict__ keys,
                                                                    const int *__restrict__ vals,
                                                                    const int64_t *__restrict__ seg,
                                                                    const int *__restrict__ hist, int *__restrict__ out,
                                                                    int *__restrict__ perm, int max_chunks, int tiles,
                                                                    int64_t cap)
{
    (void)cap;
    extern __shared__ int whist[]; // [8][tiles]
    constexpr int kWarps = kSortThreads / 32, kRounds = kSort / kSortThreads;
    const int s = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = blockIdx.x;; c += gridDim.x)
    {
    const int64_t b = seg[s] + (int64_t)c * kSort, e = min(seg[s + 1], b + kSort);
    if (b >= e)
        return;
    __syncthreads(); // the previous chunk's ranks are consumed
    for (int i = threadIdx.x; i < kWarps * tiles; i += blockDim.x)
        whist[i] = 0;
    __syncthreads();
    int *wh = whist + w * tiles;
    int rk[kRounds];
    uint16_t ky[kRounds];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kRounds; k++)
    {
        const int64_t i = b + (int64_t)w * (kSort / kWarps) + k * 32 + lane;
        const bool valid = i < e;
        const unsigned key = valid ? keys[i] : 0xffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (valid)
            base = wh[key];
        __syncwarp();
        if (valid && lane == leader)
            wh[key] = base + __popc(peers);
        __syncwarp();
        rk[k] = base + __popc(peers & lt);
        ky[k] = (uint16_t)key;
    }
    __syncthreads();
    const int *hc = hist + ((int64_t)s * max_chunks + c) * tiles;
    for (int t = threadIdx.x; t < tiles; t += blockDim.x)
    {
        int run = hc[t];
        for (int ww = 0; ww < kWarps; ww++)
        {
            const int v = whist[ww * tiles + t];
            whist[ww * tiles + t] = run;
            run += v;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRounds; k++)
    {
        const int64_t i = b + (int64_t)w * (kSort / kWarps) + k * 32 + lane;
        if (i < e)
        {
            const int64_t dst = seg[s] + wh[ky[k]] + rk[k];
            SWR_DCHECK(dst >= seg[s] && dst < seg[s + 1] && dst < cap, "sort_scatter: slot outside the segment");
            out[dst] = vals[i];
            if (perm) // CSR slot of each emitted pair (the backward merges per primitive)
                perm[i] = (int)dst;
        }
    }
    }
}

void launch_bin_sort(Ctx &c, int nb, int64_t pairs, int max_seg, cudaStream_t st)
{
    const int tiles = c.g.tiles;
    dim3 ge((c.g.n + 255) / 256, nb);
    if (ge.x > 0) // an empty set emits no pairs (the sort still writes empty tile lists)
        emit_kernel<<<ge, 256, 0, st>>>(c.g, c.w.rng, c.w.poff, c.w.seg, c.w.keys, c.w.vals, c.w.cap_pairs);
    // sort CTAs per position: the chunk count of max_seg -- the longest segment when the
    // host knows it, else an estimate (the CTAs loop over chunks, so a longer segment
    // is still covered, only with fewer CTAs)
    const int nch = std::max(1, (max_seg + kSort - 1) / kSort);
    (void)pairs;
    dim3 gs(nch, nb);
    sort_hist_kernel<<<gs, kSortThreads, tiles * sizeof(int), st>>>(c.w.keys, c.w.seg, c.w.chunk_hist, c.w.max_chunks,
                                                                    tiles);
    sort_scan_kernel<<<nb, 1024, 0, st>>>(c.w.seg, c.w.chunk_hist, c.w.tile_off, c.w.max_chunks, tiles);
    sort_scatter_kernel<<<gs, kSortThreads, 8 * tiles * sizeof(int), st>>>(c.w.keys, c.w.vals, c.w.seg,
                                                                           c.w.chunk_hist, c.w.sorted,
                                                                           c.w.want_perm ? c.w.perm : nullptr,
                                                                           c.w.max_chunks, tiles, c.w.cap_pairs);
    c.launches += 4;
}

// ------------------------------------------------------------------ raster

// Block reduction of (max |A|, first argmax cell, sum |A|) for the heads.
__device__ __forceinline__ void heads_reduce(float mag, int cell, double msum, float4 *tile_part, double *tile_sum)
{
    __shared__ float smax[32];
    __shared__ int sidx[32];
    __shared__ double ssum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
    {
        const float om = __shfl_xor_sync(0xffffffffu, mag, o);
        const int oi = __shfl_xor_sync(0xffffffffu, cell, o);
        if (om > mag || (om == mag && oi < cell))
        {
            mag = om;
            cell = oi;
        }
        msum += __shfl_xor_sync(0xffffffffu, msum, o);
    }
    if (lane == 0)
    {
        smax[wid] = mag;
        sidx[wid] = cell;
        ssum[wid] = msum;
    }
    __syncthreads();
    if (threadIdx.x == 0)
    {
        float m = smax[0];
        int ci = sidx[0];
        double sm = ssum[0];
        for (int k = 1; k < nw; k++)
        {
            if (smax[k] > m || (smax[k] == m && sidx[k] < ci))
            {
                m = smax[k];
                ci = sidx[k];
            }
            sm += ssum[k];
        }
        *tile_part = make_float4(m, __int_as_float(ci), 0.f, 0.f);
        *tile_sum = sm;
    }
}

// magnitude (spectrum.cpp:141): float(hypot(double re, double im))
__device__ __forceinline__ float cell_mag(float re, float im)
{
    const double x = re, y = im;
    return (float)__dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
}

// splat.cpp:72-82 for |x| < 3 pi (one conditional step, same result as the
// reference's loops); larger displacements take the loop.
__device__ __forceinline__ float wrap_fast(float x)
{
    if (fabsf(x) >= (float)(3 * kPi))
        return wrap_pm_pi(x);
    x = x >= (float)kPi ? __fsub_rn(x, (float)(2 * kPi)) : x;
    x = x < (float)(-kPi) ? __fadd_rn(x, (float)(2 * kPi)) : x;
    return x;
}


// floor(x / d) == (x * m[d]) >> 12 for 0 <= x < 128, 1 <= d <= 32, m[d] = ceil(4096 / d)
__host__ __device__ constexpr uint32_t magic12(int d) { return (4096u + d - 1) / d; }

// the two-step wrap of wrap_fast without its |x| >= 3 pi escape (caller guarantees |x| < 3 pi)
__device__ __forceinline__ float wrap_near(float x)
{
    x = x >= (float)kPi ? __fsub_rn(x, (float)(2 * kPi)) : x;
    x = x < (float)(-kPi) ? __fadd_rn(x, (float)(2 * kPi)) : x;
    return x;
}

__device__ __forceinline__ float2 shfl_f2(float2 v, int src)
{
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

#ifndef SWR_RASTER_MINB
#define SWR_RASTER_MINB 4 // x 8 warps: resident warps per SM / 8
#endif
#ifndef SWR_SWEEP_UNROLL
#define SWR_SWEEP_UNROLL 1 // sweeps unrolled per record; measured (swizzled copies): 1 / 2 / 4 = 18.1 / 18.7 / 18.8 ms per 1024 spectra at 50k
#endif
constexpr int kSweepUnroll = SWR_SWEEP_UNROLL;

// ---------------------------------------------------------------- raster
//
// One CTA of 4 warps per (tile, position), 9 CTAs resident per SM. The tile's pair
// list (ascending primitive index, splat.cpp:251-292) is cut into chunks of 32;
// warp w takes chunks w, w+4, ... For a chunk, each lane first turns one pair into a
// record (gathers the pair's dynamic state, shape and box, clips it to the tile:
// rows [max(r0, tile), min(r1, tile)] x the one or two wrapped column spans,
// splat.cpp:450-470, rows per sweep = 16 / columns), the warp sorts the 32 records
// by sweep count (bitonic, shuffles) and stores them in that order, so similar
// records pair up. Each half-warp then evaluates one record at a time: its 16 lanes
// write the record's row table (d_el, q_c = i00 d_el^2, or +inf where the reference
// skips the row, splat.cpp:405-408, and the row's swizzled accumulator address;
// single-buffered with SWR_RASTER_SLIM, a __syncwarp before and after the write),
// map themselves onto the clipped box (magic division: lane -> (row, column)),
// compute their column's w1 / w2 and sweep rows lr, lr + rpi, ... with a
// pointer-bounded loop (each lane its own trip count). Each half-warp accumulates
// into its own shared-memory copy of the tile with a predicated read-modify-write
// (no atomics); the copies are summed in fixed order, so results are
// bit-deterministic. The cutoff mask uses the reference's float q in its operation
// order (no FMA); exp(-q/2) is ex2.approx of a prescaled argument. Chunks whose
// azimuths could need the reference's multi-turn wrap take a separate instantiation.
//
// Measured against the round-1 kernel (same decomposition, packed records, two
// __syncwarps and a shuffled common trip count per record pair): ncu source view
// ~96 -> ~60 warp-instructions per record pair outside the sweep loop and 19 -> 15
// inside it (4.49 -> 3.44 G warp-instructions per 256-position launch at 50k), but
// only 6-9% less time: the kernel is now bound by the shared-memory data pipe (81%
// of peak wavefronts: a row-table read and a 64-bit accumulator RMW per cell), issue
// 69% active. Tried and not kept: padded accumulator rows
// against bank conflicts (occupancy loss > conflict gain), register-tile
// accumulation (lane = tile column, rows unrolled in registers: no shared traffic
// per cell, but ~53% column utilisation and per-row guards: 22.0 vs 19.4 ms per
// 1024 spectra at 50k), a software-pipelined sweep loop (more instructions).
#ifndef SWR_RASTER_SLIM
#define SWR_RASTER_SLIM 1 // 40-byte records (separate int2 array), single-buffered row tables: 9 CTAs per SM
                          // (measured 1-3% faster than 48-byte records + double buffers at 8 CTAs)
#endif
#if SWR_RASTER_SLIM
struct Rec2
{
    float4 dyn;   // el, az, amplitude re, im
    float4 shape; // i00, 2*i01 (exact), i11, 1/l1
};
// + a parallel int2 array (6-bit fields: tiles up to 32): magic(ncol) | ncol << 13 |
// rows per sweep << 19 | columns of the first span << 25; first column of the first
// span | first row << 6 | (last row + 1) << 12
constexpr int kRecExtra = 8;
#ifndef SWR_RASTER_CTAS
#define SWR_RASTER_CTAS 9 // 10 / 12 (48 / 40 registers, small spills) measured 4% / 12% slower
#endif
constexpr int kRasterCtas = SWR_RASTER_CTAS;
#else
struct Rec2
{
    float4 dyn;   // el, az, amplitude re, im
    float4 shape; // i00, 2*i01 (exact), i11, 1/l1
    int4 a;       // magic(ncol); ncol | rows per sweep (0: empty) << 8 | columns of the first span << 16;
                  // first column of the first span (tile-relative) | first row << 8 | last row << 16; sweeps
};
constexpr int kRecExtra = 0;
constexpr int kRasterCtas = 8;
#endif

// Accumulator copies are [T rows][TS slots] float2 (TS = 16 for tiles <= 16, else
// 32) with cell (r, c) in slot c ^ brev(r): a half-warp's 64-bit read-modify-write
// covers rpi rows x ncol columns of a record's box, and in a plain row-major copy
// (16 float2 = all 32 banks per row) rows of the same column collide. XOR-ing the
// column with the bit-reversed row sends consecutive rows to disjoint slot sets
// (bank-conflict model over the measured (ncol, nrow) histogram of a 10k scene: 1.14
// wavefronts per half-warp access instead of 1.77; padding the rows instead costs
// the occupancy the accumulator copies already bound: pad 0/1/3/7/9 measured
// 19.6/20.3/19.7/20.7/20.9 ms per 1024 spectra at 50k). The row table carries each
// row's swizzled base address, so a cell's address is one XOR per sweep.
template <int kRasterWarps, int G>
__global__ void __launch_bounds__(32 * kRasterWarps, kRasterCtas * 4 / kRasterWarps)
    raster2_kernel(Grid g, SceneDev sd, const float4 *__restrict__ dyn, const int4 *__restrict__ rng,
                   const int64_t *__restrict__ seg, const int *__restrict__ tile_off, const int *__restrict__ prims,
                   float *__restrict__ spec, float4 *__restrict__ tile_part, double *__restrict__ tile_sum,
                   int want_heads, int s_base)
{
    extern __shared__ __align__(256) float2 acc[]; // [G * warps][T][TS], then Rec2 [warps][32]
    __shared__ float elc[32], azc[32];
    __shared__ uint32_t magic[33];
    constexpr int LPR = 32 / G; // lanes per record slot
    // double-buffered (d_el, q_c | +inf, swizzled row address) per tile row
    constexpr int kTabBufs = SWR_RASTER_SLIM ? 1 : 2;
    __shared__ __align__(16) float4 rowtab_all[kRasterWarps * G][kTabBufs][LPR];
    const int T = g.tile, TT = T * T, TS = T <= 16 ? 16 : 32, ACOPY = T * TS;
    const int swz_shift = T <= 16 ? 28 : 27; // brev(r) >> shift = r's low 4 (5) bits reversed
    const int t = blockIdx.x, s = s_base + blockIdx.y;
    const int tr0 = (t / g.tw) * T, tc0 = (t % g.tw) * T;
    const int tr1 = min(tr0 + T, g.H) - 1, tc1 = min(tc0 + T, g.W) - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Rec2 *recs = reinterpret_cast<Rec2 *>(acc + G * kRasterWarps * ACOPY) + warp * 32;
    for (int i = threadIdx.x; i < G * kRasterWarps * ACOPY; i += blockDim.x)
        acc[i] = make_float2(0.f, 0.f);
    if (threadIdx.x < 32)
        elc[threadIdx.x] = (int)threadIdx.x < T && tr0 + (int)threadIdx.x <= tr1 ? sd.el_c[tr0 + threadIdx.x] : 0.f;
    if (threadIdx.x < T)
        azc[threadIdx.x] = tc0 + (int)threadIdx.x <= tc1 ? sd.az_c[tc0 + threadIdx.x] : 0.f;
    if (threadIdx.x <= 32)
        magic[threadIdx.x] = threadIdx.x ? magic12(threadIdx.x) : 0u;
    __syncthreads();
    const int *tl = tile_off + (int64_t)s * (g.tiles + 1);
    const int64_t lb = seg[s] + tl[t], le = seg[s] + tl[t + 1];
    SWR_DCHECK(lb >= seg[s] && lb <= le && le <= seg[s + 1], "raster: tile list outside its position's segment");
    const int64_t sbase = (int64_t)s * g.np;
    const int half = G == 2 ? lane >> 4 : 0, hl = lane & (LPR - 1);
    const int slot = G * warp + half;
    const uint32_t acc_base = (uint32_t)__cvta_generic_to_shared(acc + slot * ACOPY); // TS * 8-byte aligned
    const uint32_t tab_base = (uint32_t)__cvta_generic_to_shared(&rowtab_all[slot][0][0]);
    const float cut2 = g.cut2;
    const float kExp = -0.72134752044448170368f; // -0.5 * log2(e)
    const float my_elc = elc[hl < T ? hl : 0];     // this lane's tile row for the row table
    // this lane's row's swizzled base address in its slot's copy (row table entry)
    const uint32_t my_row_addr = acc_base + 8u * (uint32_t)(hl * TS) + 8u * (__brev((uint32_t)hl) >> swz_shift);
    const int *plist = prims + lb;
    const int cnt = (int)(le - lb);
    const float4 *dyn_s = dyn + sbase;
    const int4 *rng_s = rng + sbase;
    const int tcw = tc1 - tc0 + 1;

    // 32-bit shared addresses kept in registers across the record loop (the compiler
    // otherwise rebuilds them from the shared window base per record)
    const uint32_t rec0 = (uint32_t)__cvta_generic_to_shared(recs + half);
    int2 *recx = reinterpret_cast<int2 *>(reinterpret_cast<Rec2 *>(acc + G * kRasterWarps * ACOPY) + kRasterWarps * 32) +
                 warp * 32; // SWR_RASTER_SLIM: the records' packed integer fields
    const uint32_t recx0 = (uint32_t)__cvta_generic_to_shared(recx + half);
    (void)recx0;
    const uint32_t azc_base = (uint32_t)__cvta_generic_to_shared(azc);
    const uint32_t my_tab0 = tab_base + 16u * (uint32_t)hl, my_tab1 = my_tab0 + 16u * LPR * (kTabBufs - 1);

    auto evaluate = [&](auto slow_tag, int j0) {
        constexpr bool SLOW = decltype(slow_tag)::value;
        uint32_t ra_addr = rec0 + (uint32_t)(G * j0) * (uint32_t)sizeof(Rec2);
#pragma unroll 1
        for (int j = j0; j < 32 / G; j++, ra_addr += G * (uint32_t)sizeof(Rec2))
        {
            float4 A, S;
            int4 ra;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(A.x), "=f"(A.y), "=f"(A.z), "=f"(A.w) : "r"(ra_addr));
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+16];"
                         : "=f"(S.x), "=f"(S.y), "=f"(S.z), "=f"(S.w) : "r"(ra_addr));
#if SWR_RASTER_SLIM
            {
                int p0, p1;
                asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(p0), "=r"(p1)
                             : "r"(recx0 + 8u * (uint32_t)(G * j)));
                ra.x = p0 & 0x1fff;
                ra.y = ((p0 >> 13) & 63) | (((p0 >> 19) & 63) << 8) | ((p0 >> 25) << 16);
                ra.z = (p1 & 63) | (((p1 >> 6) & 63) << 8) | ((((p1 >> 12) & 63) - 1) << 16);
                ra.w = 0;
            }
            __syncwarp(); // single-buffered row table: every lane is done with the previous record
#else
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+32];"
                         : "=r"(ra.x), "=r"(ra.y), "=r"(ra.z), "=r"(ra.w) : "r"(ra_addr));
#endif
            const int ncol = ra.y & 255, rpi = (ra.y >> 8) & 255, na = ra.y >> 16;
            const int a0off = ra.z & 255, rfirst = (ra.z >> 8) & 255, rlast = ra.z >> 16;
            SWR_DCHECK(rpi == 0 || (ncol >= 1 && ncol <= T && rpi * ncol <= LPR && rfirst <= rlast && rlast < T &&
                                    na <= ncol && a0off + na <= T),
                       "raster: record box outside the tile");
            // row table of this record: q_c = i00 d_el^2, +inf where the reference skips
            // the row ((d_el / l1)^2 > r^2, splat.cpp:405-408), and the row's swizzled address
            const bool odd = kTabBufs == 2 && (j & 1);
            const uint32_t tb = odd ? tab_base + 16u * LPR : tab_base;
            {
                const float d_el = __fsub_rn(my_elc, A.x);
                const float u0 = __fmul_rn(d_el, S.w);
                const float qc = __fmul_rn(u0, u0) > cut2 ? __int_as_float(0x7f800000)
                                                          : __fmul_rn(__fmul_rn(S.x, d_el), d_el);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(odd ? my_tab1 : my_tab0),
                             "r"(__float_as_uint(d_el)), "r"(__float_as_uint(qc)), "r"(my_row_addr), "r"(0u)
                             : "memory");
            }
            __syncwarp();
            // this lane's cell in the box: rows lr, lr + rpi, ..., column cc of the tile
            const int lr = (int)(((uint32_t)hl * (uint32_t)ra.x) >> 12);
            const int lc = hl - lr * ncol;
            const bool on = lr < rpi;
            const int cc = on ? lc + (lc < na ? a0off : -na) : 0;
            const int row0 = rfirst + lr;
            const uint32_t cc8 = 8u * (uint32_t)cc;
            uint32_t tp = tb + 16u * (uint32_t)row0;
            const uint32_t tp_last = tb + 16u * (uint32_t)rlast, t_step = 16u * (uint32_t)rpi;
            float azc_c;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(azc_c) : "r"(azc_base + 4u * (uint32_t)cc));
            const float xaz = __fsub_rn(azc_c, A.y);
            const float d_az = SLOW ? wrap_fast(xaz) : wrap_near(xaz);
            const float w1 = __fmul_rn(__fmul_rn(S.z, d_az), d_az);
            const float w2 = __fmul_rn(S.y, d_az); // (2 * i01) * d_az
            if (on)
            {
#pragma unroll kSweepUnroll
                for (; tp <= tp_last; tp += t_step)
                {
                    float d_el, qc;
                    uint32_t raddr, pad;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(d_el), "=f"(qc), "=r"(raddr), "=r"(pad)
                                 : "r"(tp));
                    const uint32_t cp = raddr ^ cc8;
#ifdef SWR_CHECKED
                    // own copy of the tile, 8-byte slot, and no two lanes of the warp on the
                    // same cell in this sweep step (the read-modify-write is race-free)
                    SWR_DCHECK(cp >= acc_base && cp < acc_base + 8u * (uint32_t)ACOPY && (cp & 7u) == 0u,
                               "raster: accumulator address outside the slot's copy");
                    SWR_DCHECK(tp >= tb && tp < tb + 16u * (uint32_t)LPR, "raster: row table index");
                    SWR_DCHECK(__popc(__match_any_sync(__activemask(), cp)) == 1, "raster: two lanes on one cell");
#endif
                    const float q = __fadd_rn(__fadd_rn(qc, __fmul_rn(d_el, w2)), w1);
                    float e;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q * kExp));
                    asm volatile("{\n\t.reg .pred p;\n\t.reg .f32 a, b;\n\t"
                                 "setp.le.f32 p, %0, %5;\n\t"
                                 "@p ld.shared.v2.f32 {a, b}, [%1];\n\t"
                                 "@p fma.rn.f32 a, %2, %4, a;\n\t"
                                 "@p fma.rn.f32 b, %3, %4, b;\n\t"
                                 "@p st.shared.v2.f32 [%1], {a, b};\n\t}" ::"f"(q),
                                 "r"(cp), "f"(A.z), "f"(A.w), "f"(e), "f"(cut2)
                                 : "memory");
                }
            }
        }
    };

    int c0 = warp * 32;
    int gi = c0 + lane < cnt ? plist[c0 + lane] : -1;
    SWR_DCHECK(gi < g.n, "raster: primitive index");
    int4 b = gi >= 0 ? rng_s[gi] : make_int4(0, -1, 0, 0);
    float4 d = gi >= 0 ? dyn_s[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 sh = gi >= 0 ? sd.shape[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
    for (; c0 < cnt; c0 += kRasterWarps * 32)
    {
        bool slow;
        int j0;
        {
            int pr0 = max(b.x, tr0), pr1 = min(b.y, tr1);
            // drop the rows the reference skips ((d_el / l1)^2 > r^2, splat.cpp:405-408):
            // u0 is monotonic in the row, so they sit at the two ends of the box
            // (~12% of box cells at the reference grid); same float ops as the row table
            if (gi >= 0)
            {
                const auto skipped = [&](int r) {
                    const float u0 = __fmul_rn(__fsub_rn(elc[r - tr0], d.x), sh.w);
                    return __fmul_rn(u0, u0) > cut2;
                };
                while (pr0 <= pr1 && skipped(pr0))
                    pr0++;
                while (pr1 >= pr0 && skipped(pr1))
                    pr1--;
            }
            int a0 = tc0, na = tcw, nb2 = 0;
            if (b.w < g.W)
            {
                const int jend = b.z + b.w - 1;
                a0 = max(tc0, b.z);
                na = max(0, min(tc1, min(jend, g.W - 1)) - a0 + 1);
                nb2 = jend >= g.W ? max(0, min(tc1, jend - g.W) - tc0 + 1) : 0;
            }
            const int ncol = na + nb2, nrow = pr1 - pr0 + 1;
            int rpi = 0, sweeps = 0;
            uint32_t mn = 0;
            if (gi >= 0 && ncol > 0 && nrow > 0)
            {
                mn = magic[ncol];
                rpi = (int)(((uint32_t)LPR * mn) >> 12);
                sweeps = (int)(((uint32_t)(nrow + rpi - 1) * magic[rpi]) >> 12);
            }
            slow = __any_sync(0xffffffffu, sweeps > 0 && !(d.y > -3.0f && d.y < 9.0f));
            const int nempty = __popc(__ballot_sync(0xffffffffu, sweeps == 0));
            j0 = nempty / G; // records sorted by sweeps: the first j0 slots-groups are empty
            const int a0off = na > 0 ? a0 - tc0 : 0;
            uint32_t key = ((uint32_t)sweeps << 5) | (uint32_t)lane;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                for (int jj = k >> 1; jj > 0; jj >>= 1)
                {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, key, jj);
                    const bool up = (lane & k) == 0, lower = (lane & jj) == 0;
                    key = (lower == up) ? min(key, o) : max(key, o);
                }
            const int src = (int)(key & 31);
            Rec2 r;
            const float2 dxy = shfl_f2(make_float2(d.x, d.y), src), dzw = shfl_f2(make_float2(d.z, d.w), src);
            const float2 sxy = shfl_f2(make_float2(sh.x, __fmul_rn(2.0f, sh.y)), src),
                         szw = shfl_f2(make_float2(sh.z, sh.w), src);
            r.dyn = make_float4(dxy.x, dxy.y, dzw.x, dzw.y);
            r.shape = make_float4(sxy.x, sxy.y, szw.x, szw.y);
#if SWR_RASTER_SLIM
            recx[lane] = make_int2(__shfl_sync(0xffffffffu, (int)mn | (ncol << 13) | (rpi << 19) | (na << 25), src),
                                   __shfl_sync(0xffffffffu,
                                               a0off | ((pr0 - tr0) << 6) | ((max(pr1 - tr0 + 1, 0) & 63) << 12), src));
#else
            r.a = make_int4(__shfl_sync(0xffffffffu, (int)mn, src),
                            __shfl_sync(0xffffffffu, ncol | (rpi << 8) | (na << 16), src),
                            __shfl_sync(0xffffffffu, a0off | ((pr0 - tr0) << 8) | ((pr1 - tr0) << 16), src),
                            __shfl_sync(0xffffffffu, sweeps, src));
#endif
            recs[lane] = r;
        }
        const int cn = c0 + kRasterWarps * 32;
        gi = cn + lane < cnt ? plist[cn + lane] : -1;
        SWR_DCHECK(gi < g.n, "raster: primitive index");
        b = gi >= 0 ? rng_s[gi] : make_int4(0, -1, 0, 0);
        d = gi >= 0 ? dyn_s[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
        sh = gi >= 0 ? sd.shape[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (slow)
            evaluate(std::integral_constant<bool, true>(), j0);
        else
            evaluate(std::integral_constant<bool, false>(), j0);
        __syncwarp(); // records and row tables are rewritten for the next chunk
    }
    __syncthreads();
    float best = -1.0f;
    int bidx = 0x7fffffff;
    double lsum = 0.0;
    for (int cl = threadIdx.x; cl < TT; cl += blockDim.x)
    {
        const int r = tr0 + cl / T, c = tc0 + cl % T;
        if (r > tr1 || c > tc1)
            continue;
        float re = 0.f, im = 0.f;
        const int rr = cl / T, ai = rr * TS + ((cl % T) ^ (int)(__brev((uint32_t)rr) >> swz_shift));
#pragma unroll
        for (int w = 0; w < G * kRasterWarps; w++)
        {
            const float2 v = acc[w * ACOPY + ai];
            re = __fadd_rn(re, v.x);
            im = __fadd_rn(im, v.y);
        }
        if (spec)
            reinterpret_cast<float2 *>(spec)[((int64_t)s * g.H + r) * g.W + c] = make_float2(re, im);
        if (want_heads)
        {
            const float m = cell_mag(re, im);
            const int ci = r * g.W + c;
            if (m > best || (m == best && ci < bidx))
            {
                best = m;
                bidx = ci;
            }
            lsum += (double)m;
        }
    }
    if (want_heads)
        heads_reduce(best, bidx, lsum, tile_part + (int64_t)s * g.tiles + t, tile_sum + (int64_t)s * g.tiles + t);
}

template <int WARPS, int G>
static void launch_raster_w(Ctx &c, int nb, float *d_spec, bool want_heads, cudaStream_t st, int s_base)
{
    const size_t smem =
        (size_t)G * WARPS * c.g.tile * (c.g.tile <= 16 ? 16 : 32) * sizeof(float2) +
        WARPS * 32 * (sizeof(Rec2) + kRecExtra);
    static DeviceOnce once;
    once.get(c.device, [&] {
        check_cuda(cudaFuncSetAttribute(raster2_kernel<WARPS, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(G * WARPS * 32 * 32 * sizeof(float2) +
                                              WARPS * 32 * (sizeof(Rec2) + kRecExtra))),
                   "raster smem attribute");
        // same L1/shared split as the MLP kernel
        check_cuda(cudaFuncSetAttribute(raster2_kernel<WARPS, G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        (int)cudaSharedmemCarveoutMaxShared),
                   "raster carveout");
        return 1;
    });
    raster2_kernel<WARPS, G><<<dim3(c.g.tiles, nb), 32 * WARPS, smem, st>>>(
        c.g, c.s, c.w.dyn, c.w.rng, c.w.seg, c.w.tile_off, c.w.sorted, d_spec, c.w.tile_part, c.w.tile_sum,
        want_heads ? 1 : 0, s_base);
    c.launches++;
}

// warps = 8 (standalone) or 4 (small enough to run beside the persistent MLP kernel);
// two records per warp when a tile row fits in 16 lanes
#ifndef SWR_RASTER_WARPS
#define SWR_RASTER_WARPS 4
#endif
void launch_raster(Ctx &c, int nb, float *d_spec, bool want_heads, cudaStream_t st, int warps, int s_base)
{
    if (warps == 0)
        warps = SWR_RASTER_WARPS;
    const bool narrow = c.g.tile <= 16;
    if (warps == 2)
        narrow ? launch_raster_w<2, 2>(c, nb, d_spec, want_heads, st, s_base)
               : launch_raster_w<2, 1>(c, nb, d_spec, want_heads, st, s_base);
    else if (warps == 4)
        narrow ? launch_raster_w<4, 2>(c, nb, d_spec, want_heads, st, s_base)
               : launch_raster_w<4, 1>(c, nb, d_spec, want_heads, st, s_base);
    else
        narrow ? launch_raster_w<8, 2>(c, nb, d_spec, want_heads, st, s_base)
               : launch_raster_w<8, 1>(c, nb, d_spec, want_heads, st, s_base);
}

// Heads on given spectra: the same per-tile partials as the raster epilogue.
__global__ void tile_heads_kernel(Grid g, const float *__restrict__ spec, float4 *__restrict__ tile_part,
                                  double *__restrict__ tile_sum)
{
    const int t = blockIdx.x, s = blockIdx.y;
    const int tr = t / g.tw, tc = t % g.tw;
    const int ty = threadIdx.x / g.tile, tx = threadIdx.x % g.tile;
    const int r = tr * g.tile + ty, c = tc * g.tile + tx;
    const bool valid = r < g.H && c < g.W && ty < g.tile;
    float mag = -1.0f;
    if (valid)
    {
        const float2 v = reinterpret_cast<const float2 *>(spec)[((int64_t)s * g.H + r) * g.W + c];
        mag = cell_mag(v.x, v.y);
    }
    heads_reduce(mag, valid ? r * g.W + c : 0x7fffffff, valid ? (double)mag : 0.0,
                 tile_part + (int64_t)s * g.tiles + t, tile_sum + (int64_t)s * g.tiles + t);
}

void launch_heads_from_spectra(Ctx &c, int nb, const float *d_spec, cudaStream_t st)
{
    dim3 grid(c.g.tiles, nb);
    const int threads = ((c.g.tile * c.g.tile + 31) / 32) * 32;
    tile_heads_kernel<<<grid, threads, 0, st>>>(c.g, d_spec, c.w.tile_part, c.w.tile_sum);
    c.launches++;
}

// Combine the per-tile partials: AoA = first maximum in row-major order
// (tasks.cpp:158-162), pooled = sum |A| / cells (tasks.cpp:32-39), RSSI affine.
__global__ void heads_kernel(Grid g, const float4 *__restrict__ tile_part, const double *__restrict__ tile_sum,
                             int nb, double slope, double intercept, double *pooled, double *rssi, int32_t *aoa_rc,
                             double *aoa_ang)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nb)
        return;
    float m = -2.0f;
    int ci = 0x7fffffff;
    double sum = 0.0;
    for (int t = 0; t < g.tiles; t++)
    {
        const float4 p = tile_part[(int64_t)s * g.tiles + t];
        const int pi = __float_as_int(p.y);
        if (p.x > m || (p.x == m && pi < ci))
        {
            m = p.x;
            ci = pi;
        }
        sum += tile_sum[(int64_t)s * g.tiles + t];
    }
    const double pm = sum / (double)(g.H * g.W);
    if (pooled)
        pooled[s] = pm;
    if (rssi)
        rssi[s] = slope * pm + intercept;
    const int row = ci / g.W, col = ci % g.W;
    if (aoa_rc)
    {
        aoa_rc[2 * s] = row;
        aoa_rc[2 * s + 1] = col;
    }
    if (aoa_ang)
    {
        aoa_ang[2 * s] = (row + 0.5) * g.cell_el;
        aoa_ang[2 * s + 1] = (col + 0.5) * g.cell_az;
    }
}

void launch_heads(Ctx &c, int nb, uint32_t flags, double *d_pooled, double *d_rssi, int32_t *d_aoa_rc,
                  double *d_aoa_ang, cudaStream_t st)
{
    (void)flags;
    heads_kernel<<<(nb + 127) / 128, 128, 0, st>>>(c.g, c.w.tile_part, c.w.tile_sum, nb, c.rssi_slope,
                                                   c.rssi_intercept, d_pooled, d_rssi, d_aoa_rc, d_aoa_ang);
    c.launches++;
}

} // namespace swr
