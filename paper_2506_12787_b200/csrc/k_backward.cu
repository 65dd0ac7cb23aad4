// Render backward (first part): the gradient of
// a loss wrt the Gaussian parameters and the deformation residuals given the
// upstream gradient dL/dA of every spectrum cell — splat::rasterize_backward
// (splat.cpp:494-669), batched over TX positions.
//
//   raster_bwd_kernel  one CTA per (tile, position), the forward raster's layout:
//                      the tile's (tile, primitive) list cut into chunks of 32,
//                      one record per lane, then the warp evaluates the records
//                      one by one with its lanes over the clipped box, each lane
//                      accumulating the 8 partials (d_el, d_az, dl1, dl2, dl3,
//                      ddelta, dre, dim) of splat.cpp:545-571 for its cells; a
//                      fixed-order warp reduction writes the pair's partials to
//                      its CSR slot (splat.cpp:587-595)
//   bwd_merge_kernel   one thread per (position, primitive): sums the primitive's
//                      slots in ascending tile order (the reference's fixed merge
//                      order, splat.cpp:601-610) and applies the chain rule onto
//                      the raw fields (splat.cpp:612-664)
// Float arithmetic in the reference's operation order; exp is expf. The cell
// partials are summed per lane and then across lanes, so the pair partials
// differ from the reference's sequential sums by rounding only (deterministic).
#include "swr_internal.h"

#include <cstdlib>

namespace swr
{

namespace
{
constexpr int kBwdWarps = 8;
constexpr int kState = 11; // splat.cpp:133-147 state stride

struct BwdRec
{
    float st[12];  // the 11-float render state (+ pad)
    int4 box;      // first row, last row (tile-relative), ncol | na << 6 | a0 << 12 | rpi << 18 | sweeps << 24,
                   // magic(ncol) | magic(rpi) << 13
};

__device__ __forceinline__ uint32_t magic12(int d) { return (4096u + d - 1) / d; }

__device__ __forceinline__ float wrap_pm_pi_f(float x)
{
    // splat.cpp:72-82 for |x| < 3 pi: one conditional step (larger: the loop)
    const float pi = 3.14159265358979323846f, two_pi = 6.28318530717958647692f;
    if (fabsf(x) >= 3.0f * pi)
    {
        while (x >= pi)
            x = __fsub_rn(x, two_pi);
        while (x < -pi)
            x = __fadd_rn(x, two_pi);
        return x;
    }
    x = x >= pi ? __fsub_rn(x, two_pi) : x;
    x = x < -pi ? __fadd_rn(x, two_pi) : x;
    return x;
}

__global__ void __launch_bounds__(32 * kBwdWarps)
    raster_bwd_kernel(Grid g, SceneDev sd, const float *__restrict__ state, const int4 *__restrict__ rng,
                      const int64_t *__restrict__ seg, const int *__restrict__ tile_off, const int *__restrict__ prims,
                      const float *__restrict__ upstream, float *__restrict__ slots, int split)
{
    extern __shared__ float2 up[]; // [T*T] upstream gradient of the tile, then BwdRec [warps][32]
    __shared__ float elc[64], azc[32];
    const int T = g.tile, TT = T * T;
    // blockIdx.y = position * split + part: `split` CTAs share a tile's pairs
    // (every pair owns its slot, so the split changes no arithmetic)
    const int t = blockIdx.x, s = blockIdx.y / split, part = blockIdx.y % split;
    const int tr0 = (t / g.tw) * T, tc0 = (t % g.tw) * T;
    const int tr1 = min(tr0 + T, g.H) - 1, tc1 = min(tc0 + T, g.W) - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BwdRec *recs = reinterpret_cast<BwdRec *>(up + TT) + warp * 32;
    for (int i = threadIdx.x; i < TT; i += blockDim.x)
    {
        const int r = tr0 + i / T, cc = tc0 + i % T;
        up[i] = (r <= tr1 && cc <= tc1)
                    ? reinterpret_cast<const float2 *>(upstream)[((int64_t)s * g.H + r) * g.W + cc]
                    : make_float2(0.f, 0.f);
    }
    if (threadIdx.x < 64)
        elc[threadIdx.x] = (int)threadIdx.x < T && tr0 + (int)threadIdx.x <= tr1 ? sd.el_c[tr0 + threadIdx.x] : 0.f;
    if (threadIdx.x < T)
        azc[threadIdx.x] = tc0 + (int)threadIdx.x <= tc1 ? sd.az_c[tc0 + threadIdx.x] : 0.f;
    __syncthreads();
    const int *tl = tile_off + (int64_t)s * (g.tiles + 1);
    const int64_t lb = seg[s] + tl[t], le = seg[s] + tl[t + 1];
    const int cnt = (int)(le - lb);
    const int tcw = tc1 - tc0 + 1;
    const float cut2 = g.cut2;

    for (int c0 = (part * kBwdWarps + warp) * 32; c0 < cnt; c0 += split * kBwdWarps * 32)
    {
        {
            const int j = c0 + lane;
            const int gi = j < cnt ? prims[lb + j] : -1;
            BwdRec r;
            int sweeps = 0, ncol = 0, na = 0, a0off = 0, rpi = 0, pr0 = 0, pr1 = -1;
            uint32_t mn = 0, mr = 0;
            if (gi >= 0)
            {
                const float *sp = state + ((int64_t)s * g.n + gi) * kState; // [nb][n][11] (state_out_kernel)
                for (int k = 0; k < kState; k++)
                    r.st[k] = sp[k];
                const int4 b = rng[(int64_t)s * g.np + gi];
                pr0 = max(b.x, tr0);
                pr1 = min(b.y, tr1);
                int a0 = tc0, nb2 = 0;
                na = tcw;
                if (b.w < g.W)
                {
                    const int jend = b.z + b.w - 1;
                    a0 = max(tc0, b.z);
                    na = max(0, min(tc1, min(jend, g.W - 1)) - a0 + 1);
                    nb2 = jend >= g.W ? max(0, min(tc1, jend - g.W) - tc0 + 1) : 0;
                }
                ncol = na + nb2;
                a0off = na > 0 ? a0 - tc0 : 0;
                const int nrow = pr1 - pr0 + 1;
                if (ncol > 0 && nrow > 0)
                {
                    mn = magic12(ncol);
                    rpi = (int)((32u * mn) >> 12);
                    mr = magic12(rpi);
                    sweeps = (int)(((uint32_t)(nrow + rpi - 1) * mr) >> 12);
                }
            }
            r.box = make_int4(pr0 - tr0, pr1 - tr0, ncol | (na << 6) | (a0off << 12) | (rpi << 18) | (sweeps << 24),
                              (int)(mn | (mr << 13)));
            recs[lane] = r;
        }
        __syncwarp();
        const int nrec = min(32, cnt - c0);
        for (int j = 0; j < nrec; j++)
        {
            const int4 bx = recs[j].box;
            const int sweeps = bx.z >> 24;
            float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (sweeps > 0)
            {
                const float *st = recs[j].st;
                const float el = st[0], az = st[1], i00 = st[2], i01 = st[3], i11 = st[4], delta = st[5],
                            re = st[6], im = st[7], inv_l1 = st[8], inv_l3 = st[9], l2 = st[10];
                const int ncol = bx.z & 63, na = (bx.z >> 6) & 63, a0off = (bx.z >> 12) & 63,
                          rpi = (bx.z >> 18) & 63;
                const uint32_t mn = (uint32_t)bx.w & 0x1fffu;
                const int lr = (int)(((uint32_t)lane * mn) >> 12), lc = lane - lr * ncol;
                if (lr < rpi)
                {
                    const int cc = lc < na ? a0off + lc : lc - na;
                    const float d_az = wrap_pm_pi_f(__fsub_rn(azc[cc], az));
                    const float w1 = __fmul_rn(__fmul_rn(i11, d_az), d_az);
                    const float w2 = __fmul_rn(__fmul_rn(2.0f, i01), d_az);
                    for (int rr = bx.x + lr; rr <= bx.y; rr += rpi)
                    {
                        const float d_el = __fsub_rn(elc[rr], el);
                        const float u0 = __fmul_rn(d_el, inv_l1);
                        if (__fmul_rn(u0, u0) > cut2)
                            continue;
                        const float q_c = __fmul_rn(__fmul_rn(i00, d_el), d_el);
                        const float q = __fadd_rn(__fadd_rn(q_c, __fmul_rn(d_el, w2)), w1);
                        if (q > cut2)
                            continue;
                        const float e = expf(__fmul_rn(-0.5f, q));
                        const float k = __fmul_rn(delta, e);
                        const float2 gv = up[rr * T + cc];
                        const float gdot = __fadd_rn(__fmul_rn(gv.x, re), __fmul_rn(gv.y, im));
                        a[6] = __fadd_rn(a[6], __fmul_rn(gv.x, k));
                        a[7] = __fadd_rn(a[7], __fmul_rn(gv.y, k));
                        a[5] = __fadd_rn(a[5], __fmul_rn(gdot, e));
                        const float tq = __fmul_rn(__fmul_rn(-0.5f, gdot), k);
                        const float u1 = __fmul_rn(__fsub_rn(d_az, __fmul_rn(l2, u0)), inv_l3);
                        a[2] = __fadd_rn(a[2], __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(tq, 2.0f), u0), inv_l1),
                                                         __fadd_rn(-u0, __fmul_rn(__fmul_rn(u1, l2), inv_l3))));
                        a[3] = __fadd_rn(a[3], __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(tq, -2.0f), u1), u0), inv_l3));
                        a[4] = __fadd_rn(a[4], __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(tq, -2.0f), u1), u1), inv_l3));
                        const float s0 = __fadd_rn(__fmul_rn(i00, d_el), __fmul_rn(i01, d_az));
                        const float s1 = __fadd_rn(__fmul_rn(i01, d_el), __fmul_rn(i11, d_az));
                        a[0] = __fadd_rn(a[0], __fmul_rn(__fmul_rn(tq, -2.0f), s0));
                        a[1] = __fadd_rn(a[1], __fmul_rn(__fmul_rn(tq, -2.0f), s1));
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; k++)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
                        a[k] = __fadd_rn(a[k], __shfl_down_sync(0xffffffffu, a[k], o));
            }
            if (lane == 0) // the pair's partials in its CSR slot (splat.cpp:587-595)
            {
                float4 *dst = reinterpret_cast<float4 *>(slots + (lb + c0 + j) * 8);
                dst[0] = make_float4(a[0], a[1], a[2], a[3]);
                dst[1] = make_float4(a[4], a[5], a[6], a[7]);
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

// out layouts per position s (the reference's RenderGrads): center_raw [n][2],
// cholesky [n][3], atten_logit [n], response [n][2], d_center [n][2],
// d_response [n][2], d_atten [n]; each array [nb][n...]
__global__ void bwd_merge_kernel(Grid g, SceneDev sd, const float *__restrict__ res, int64_t plane, int with_res,
                                 const int *__restrict__ cnt, const int *__restrict__ poff,
                                 const int64_t *__restrict__ seg, const uint16_t *__restrict__ keys,
                                 const int *__restrict__ perm, const float *__restrict__ slots, int nb,
                                 float *__restrict__ center_raw, float *__restrict__ cholesky,
                                 float *__restrict__ atten_logit, float *__restrict__ response,
                                 float *__restrict__ d_center, float *__restrict__ d_response,
                                 float *__restrict__ d_atten)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nb * g.n)
        return;
    const int s = (int)(idx / g.n), p = (int)(idx % g.n);
    const int64_t pe = (int64_t)s * g.np + p;
    const int m = cnt[pe];
    const int64_t e0 = seg[s] + poff[pe];
    // the primitive's slots, summed in ascending tile order (splat.cpp:601-610):
    // selection by tile key (a primitive's tiles are distinct; m is small)
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int prev = -1;
    for (int it = 0; it < m; it++)
    {
        int best = 0x7fffffff, bi = 0;
        for (int i = 0; i < m; i++)
        {
            const int tk = keys[e0 + i];
            if (tk > prev && tk < best)
            {
                best = tk;
                bi = i;
            }
        }
        prev = best;
        const float *src = slots + (int64_t)perm[e0 + bi] * 8;
        for (int q = 0; q < 8; q++)
            a[q] = __fadd_rn(a[q], src[q]);
    }
    // splat.cpp:612-664
    const float4 bw = sd.bwd[p];
    const float pi4 = 0.785398163397448309616f, pi = 3.14159265358979323846f;
    center_raw[2 * idx] = __fmul_rn(__fmul_rn(a[0], pi4), bw.x);
    center_raw[2 * idx + 1] = __fmul_rn(__fmul_rn(a[1], pi), bw.y);
    d_center[2 * idx] = a[0];
    d_center[2 * idx + 1] = a[1];
    cholesky[3 * idx] = bw.z != 0.f ? a[2] : 0.f;
    cholesky[3 * idx + 1] = a[3];
    cholesky[3 * idx + 2] = bw.w != 0.f ? a[4] : 0.f;
    response[2 * idx] = a[6];
    response[2 * idx + 1] = a[7];
    d_response[2 * idx] = a[6];
    d_response[2 * idx + 1] = a[7];
    const float delta0 = sd.delta0[p];
    float mask = 1.f;
    if (with_res)
    {
        const float pre = __fadd_rn(delta0, res[4 * plane + pe]);
        mask = (pre > 0.f && pre < 1.f) ? 1.f : 0.f;
    }
    d_atten[idx] = __fmul_rn(a[5], mask);
    atten_logit[idx] = __fmul_rn(__fmul_rn(__fmul_rn(a[5], mask), delta0), __fsub_rn(1.0f, delta0));
}
} // namespace

void launch_raster_backward(Ctx &c, int nb, const float *d_state, const float *d_upstream, float *d_slots,
                            cudaStream_t st)
{
    // few positions (training: one) leave most SMs idle with a CTA per tile: split
    // each tile's pair list over enough CTAs for ~4 per SM
    int split = std::max(1, std::min(8, (4 * 148 + c.g.tiles * nb - 1) / (c.g.tiles * nb)));
    if (const char *e = std::getenv("SWR_BWD_SPLIT"))
        split = std::max(1, std::atoi(e));
    dim3 grid(c.g.tiles, nb * split);
    const size_t smem = (size_t)c.g.tile * c.g.tile * sizeof(float2) + kBwdWarps * 32 * sizeof(BwdRec);
    static DeviceOnce once;
    once.get(c.device, [] {
        // the largest variant (tiles up to 32 x 32)
        const size_t mx = (size_t)32 * 32 * sizeof(float2) + kBwdWarps * 32 * sizeof(BwdRec);
        check_cuda(cudaFuncSetAttribute(raster_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx),
                   "raster backward smem");
        return 1;
    });
    raster_bwd_kernel<<<grid, 32 * kBwdWarps, smem, st>>>(c.g, c.s, d_state, c.w.rng, c.w.seg, c.w.tile_off,
                                                          c.w.sorted, d_upstream, d_slots, split);
    c.launches++;
}

void launch_bwd_merge(Ctx &c, int nb, bool with_res, const float *d_slots, float *const out[7], cudaStream_t st)
{
    const int64_t total = (int64_t)nb * c.g.n;
    bwd_merge_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        c.g, c.s, c.w.res, (int64_t)c.w.cap_b * c.g.np, with_res ? 1 : 0, c.w.cnt, c.w.poff, c.w.seg, c.w.keys,
        c.w.perm, d_slots, nb, out[0], out[1], out[2], out[3], out[4], out[5], out[6]);
    c.launches++;
}

} // namespace swr
