// Deformation MLP, FP32 FMA path, plus the per-position and per-scene
// encoding terms it consumes.
//
// Reference: deform::predict_residuals (/root/reference/proj/src/deform.cpp:140-207).
// Row (g, s) of the reference input matrix is [encode(centre_g) | encode(pos_s)]
// (deform.cpp:158-171); trunk layers 0, 2, 4, 6 read that row (layer 0 alone,
// 2/4/6 concatenated after the hidden state, deform.cpp:41,177-192). Because
// the encoding splits into a per-Gaussian block and a per-position block, the
// product W x splits into W_c x_c[g] (precomputed once per scene, `cg`) and
// W_p x_p[s] (+ bias, computed once per position, `pterm`). The fused kernel
// then only runs the seven hidden->hidden 156x156 products per row and adds
// cg[g] + pterm[s] in the epilogue of layers 0/2/4/6. Same real-number
// function; FP32 summation order differs from Eigen's (~1e-7 relative).
#include "swr_internal.h"

#include <cstdio>
#include <cmath>
#include <cstring>

namespace swr
{

// ------------------------------------------------------------------ per position

struct PosArgs
{
    const float *pos;   // [nb][3] metres (or already normalized)
    float *pos01;       // [nb][4]
    float *pterm;       // [nb][4][wp]
    const float *wpos;  // [4][wp][dp]
    const float *bias;  // [8][wp]
    double bmin0, bmin1, bmin2, bmax0, bmax1, bmax2;
    int normalized, bands_p, dp, wp, width;
    float pscale[4]; // powers of two: the tensor-core MLP's activation scales 2^k_l of layers 0/2/4/6, else 1
    const int64_t *gate; // non-null: run only if *gate != 0 (device-side FP32 re-run, capi.cpp run_chunk)
};

__global__ void __launch_bounds__(256) pos_prep_kernel(PosArgs a)
{
    __shared__ float v[3];
    __shared__ float xp[64];
    if (a.gate && *a.gate == 0)
        return;
    const int s = blockIdx.x;
    const int t = threadIdx.x;
    if (t < 3)
    {
        const float p = a.pos[3 * s + t];
        float out;
        if (a.normalized)
            out = p;
        else
        {
            // training.cpp:178-187 (IEEE double ops, identical on the device)
            const double lo = t == 0 ? a.bmin0 : (t == 1 ? a.bmin1 : a.bmin2);
            const double hi = t == 0 ? a.bmax0 : (t == 1 ? a.bmax1 : a.bmax2);
            const double range = hi - lo;
            out = range > 0.0 ? (float)(((double)p - lo) / range) : 0.5f;
        }
        v[t] = out;
        a.pos01[4 * s + t] = out;
    }
    __syncthreads();
    // deform.cpp:54-70: [v | sin(f_k v) | cos(f_k v)]_k, f_k = float(2^k pi)
    if (t < a.dp)
    {
        float x;
        if (t < 3)
            x = v[t];
        else
        {
            const int k = (t - 3) / 6, w = (t - 3) % 6;
            const float f = (float)(kPi * (double)(1 << k));
            x = w < 3 ? sinf(f * v[w]) : cosf(f * v[w - 3]);
        }
        xp[t] = x;
    }
    __syncthreads();
    for (int idx = t; idx < 4 * a.wp; idx += blockDim.x)
    {
        const int j = idx / a.wp, n = idx % a.wp;
        const int layer = 2 * j;
        float acc = 0.0f;
        const float *wr = a.wpos + ((size_t)j * a.wp + n) * a.dp;
        for (int k = 0; k < a.dp; k++)
            acc = __fmaf_rn(wr[k], xp[k], acc);
        a.pterm[((size_t)s * 4 + j) * a.wp + n] = n < a.width ? (acc + a.bias[layer * a.wp + n]) * a.pscale[j] : 0.0f;
    }
}

void launch_pos_prep(Ctx &c, const float *d_pos, int nb, bool normalized, cudaStream_t st)
{
    PosArgs a;
    a.pos = d_pos;
    a.pos01 = c.w.pos01;
    a.pterm = c.w.pterm;
    a.wpos = c.net.wpos;
    a.bias = c.net.bias;
    a.bmin0 = c.bbox_min[0];
    a.bmin1 = c.bbox_min[1];
    a.bmin2 = c.bbox_min[2];
    a.bmax0 = c.bbox_max[0];
    a.bmax1 = c.bbox_max[1];
    a.bmax2 = c.bbox_max[2];
    a.normalized = normalized;
    a.bands_p = c.net.bands_p;
    a.dp = c.net.dp;
    a.wp = c.net.wp;
    a.width = c.net.width;
    for (int j = 0; j < 4; j++)
        a.pscale[j] = mlp_uses_tc(c) ? std::ldexp(1.0f, c.net.tc_ascale[2 * j]) : 1.0f;
    a.gate = c.gate;
    pos_prep_kernel<<<nb, 256, 0, st>>>(a);
    c.launches++;
}

// ------------------------------------------------------------------- per scene

__global__ void center_terms_kernel(const float *__restrict__ cenc, const float *__restrict__ wcen,
                                    float *__restrict__ cg, int np, int wp, int dc, int width)
{
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= np * 4 * wp)
        return;
    const int n = idx % wp, j = (idx / wp) % 4, g = idx / (4 * wp);
    float acc = 0.0f;
    if (n < width)
    {
        const float *x = cenc + (size_t)g * dc;
        const float *wr = wcen + ((size_t)j * wp + n) * dc;
        for (int k = 0; k < dc; k++)
            acc = __fmaf_rn(wr[k], x[k], acc);
    }
    cg[idx] = acc;
}

void launch_center_terms(Ctx &c, const float *d_cenc, cudaStream_t st)
{
    const float *wcen = c.net.wcen;
    const int total = c.g.np * 4 * c.net.wp;
    if (total == 0)
        return;
    center_terms_kernel<<<(total + 255) / 256, 256, 0, st>>>(d_cenc, wcen, c.net.cg, c.g.np, c.net.wp,
                                                               c.net.dc, c.net.width);
    c.launches++;
}

// -------------------------------------------------------------- fused MLP (FP32)

struct MlpArgs
{
    const float *whT;    // [7][wp][wp] k-major
    const float *bias;   // [8][wp]
    const float *cg;     // [np][4][wp]
    const float *pterm;  // [nb][4][wp]
    const float *heads;  // [5][wp]
    const float *hbias;  // [5]
    float *res;          // [5][cap_b][np]
    int n, np, nb, cap_b, width, n_gblk, n_sblk;
    unsigned *amax;      // optional [8]: max activation of each trunk layer (float bits; scene-load probe)
    const int64_t *gate; // non-null: run only if *gate != 0 (device-side FP32 re-run)
    unsigned long long *reruns; // with gate: bumped once per gated launch that runs
};

// Tile = GB Gaussians x 8 positions = TM rows; 256 threads as 16 row groups x
// 16 column groups; each thread owns (TM/16) rows x (2*NJ) columns.
template <int TM, int NJ>
__global__ void __launch_bounds__(256) mlp_fp32_kernel(MlpArgs a)
{
    constexpr int WP = 32 * NJ;
    constexpr int RT = TM / 16;   // rows per thread
    constexpr int SB = 8;
    constexpr int GB = TM / SB;
    constexpr int TMP = TM + 4;   // padded row stride of the k-major activation buffer
    constexpr int KC = 16;        // weight rows per pipeline stage
    extern __shared__ __align__(16) float smem[];
    float *act = smem;                   // [WP][TMP]
    float *wbuf = act + WP * TMP;        // [2][KC][WP]
    const int tid = threadIdx.x;
    const int cg = tid & 15, rg = tid >> 4;
    const int ntiles = a.n_gblk * a.n_sblk;
    if (a.gate)
    {
        if (*a.gate == 0)
            return;
        if (blockIdx.x == 0 && tid == 0 && a.reruns)
            atomicAdd(a.reruns, 1ull);
    }

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
    {
        const int g0 = (tile / a.n_sblk) * GB, s0 = (tile % a.n_sblk) * SB;
        // layer 0: ReLU(cg[g][0] + pterm[s][0])   (no hidden input)
        for (int idx = tid; idx < WP * TM; idx += 256)
        {
            const int nn = idx / TM, r = idx % TM;
            const int g = g0 + r / SB, s = s0 + r % SB;
            float v = 0.0f;
            if (g < a.n && s < a.nb)
                v = a.cg[((size_t)g * 4) * WP + nn] + a.pterm[((size_t)s * 4) * WP + nn];
            act[nn * TMP + r] = v > 0.0f ? v : 0.0f;
            if (a.amax && v > 0.0f)
                atomicMax(&a.amax[0], __float_as_uint(v));
        }
        __syncthreads();

        for (int l = 1; l < kTrunk; l++)
        {
            const float *wl = a.whT + (size_t)(l - 1) * WP * WP;
            float acc[RT][2 * NJ];
#pragma unroll
            for (int i = 0; i < RT; i++)
#pragma unroll
                for (int j = 0; j < 2 * NJ; j++)
                    acc[i][j] = 0.0f;

            auto load_stage = [&](int kc, int buf) {
                const float4 *src = reinterpret_cast<const float4 *>(wl + (size_t)kc * KC * WP);
                float4 *dst = reinterpret_cast<float4 *>(wbuf + buf * KC * WP);
                for (int i = tid; i < KC * WP / 4; i += 256)
                {
                    const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst + i);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(src + i));
                }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            constexpr int NKC = WP / KC;
            load_stage(0, 0);
            for (int kc = 0; kc < NKC; kc++)
            {
                if (kc + 1 < NKC)
                {
                    load_stage(kc + 1, (kc + 1) & 1);
                    asm volatile("cp.async.wait_group 1;\n" ::);
                }
                else
                    asm volatile("cp.async.wait_group 0;\n" ::);
                __syncthreads();
                const float *wb = wbuf + (kc & 1) * KC * WP;
#pragma unroll 4
                for (int kk = 0; kk < KC; kk++)
                {
                    const int k = kc * KC + kk;
                    float av[RT];
#pragma unroll
                    for (int q = 0; q < RT / 4; q++)
                    {
                        const float4 t4 = *reinterpret_cast<const float4 *>(act + k * TMP + q * 64 + rg * 4);
                        av[4 * q] = t4.x;
                        av[4 * q + 1] = t4.y;
                        av[4 * q + 2] = t4.z;
                        av[4 * q + 3] = t4.w;
                    }
                    float wv[2 * NJ];
#pragma unroll
                    for (int j = 0; j < NJ; j++)
                    {
                        const float2 t2 = *reinterpret_cast<const float2 *>(wb + kk * WP + j * 32 + cg * 2);
                        wv[2 * j] = t2.x;
                        wv[2 * j + 1] = t2.y;
                    }
#pragma unroll
                    for (int i = 0; i < RT; i++)
#pragma unroll
                        for (int j = 0; j < 2 * NJ; j++)
                            acc[i][j] = __fmaf_rn(av[i], wv[j], acc[i][j]);
                }
                __syncthreads();
            }
            // epilogue: + bias (layers 1,3,5,7) or + cg[g] + pterm[s] (2,4,6); ReLU
            const bool skip = (l == 2 || l == 4 || l == 6);
#pragma unroll
            for (int i = 0; i < RT; i++)
            {
                const int r = (i / 4) * 64 + rg * 4 + (i % 4);
                const int g = g0 + r / SB, s = s0 + r % SB;
                const bool live = g < a.n && s < a.nb;
#pragma unroll
                for (int j = 0; j < 2 * NJ; j++)
                {
                    const int nn = (j / 2) * 32 + cg * 2 + (j & 1);
                    float e;
                    if (skip)
                        e = live ? a.cg[((size_t)g * 4 + l / 2) * WP + nn] + a.pterm[((size_t)s * 4 + l / 2) * WP + nn] : 0.0f;
                    else
                        e = a.bias[l * WP + nn];
                    const float v = acc[i][j] + e;
                    acc[i][j] = v > 0.0f ? v : 0.0f;
                }
            }
            if (a.amax)
            {
                float m = 0.0f;
#pragma unroll
                for (int i = 0; i < RT; i++)
#pragma unroll
                    for (int j = 0; j < 2 * NJ; j++)
                        m = fmaxf(m, acc[i][j]);
                atomicMax(&a.amax[l], __float_as_uint(m));
            }
#pragma unroll
            for (int j = 0; j < 2 * NJ; j++)
            {
                const int nn = (j / 2) * 32 + cg * 2 + (j & 1);
#pragma unroll
                for (int q = 0; q < RT / 4; q++)
                    *reinterpret_cast<float4 *>(act + nn * TMP + q * 64 + rg * 4) =
                        make_float4(acc[4 * q][j], acc[4 * q + 1][j], acc[4 * q + 2][j], acc[4 * q + 3][j]);
            }
            __syncthreads();
        }
        // heads (deform.cpp:203-206): 5 linear outputs per row
        for (int o = tid; o < 5 * TM; o += 256)
        {
            const int r = o % TM, h = o / TM;
            const int g = g0 + r / SB, s = s0 + r % SB;
            float acc = 0.0f;
            const float *hw = a.heads + h * WP;
            for (int k = 0; k < a.width; k++)
                acc = __fmaf_rn(act[k * TMP + r], hw[k], acc);
            if (g < a.n && s < a.nb)
                a.res[((size_t)h * a.cap_b + s) * a.np + g] = acc + a.hbias[h];
        }
        __syncthreads();
    }
}

template <int TM, int NJ>
static void run_mlp(Ctx &c, int nb, cudaStream_t st, unsigned *amax = nullptr)
{
    constexpr int WP = 32 * NJ;
    constexpr int smem = (WP * (TM + 4) + 2 * 16 * WP) * 4;
    static DeviceOnce once;
    once.get(c.device, [] {
        check_cuda(cudaFuncSetAttribute(mlp_fp32_kernel<TM, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                   "mlp smem attribute");
        return 1;
    });
    MlpArgs a;
    a.whT = c.net.whT;
    a.bias = c.net.bias;
    a.cg = c.net.cg;
    a.pterm = c.w.pterm;
    a.heads = c.net.heads;
    a.hbias = c.net.hbias;
    a.res = c.w.res;
    a.n = c.g.n;
    a.np = c.g.np;
    a.nb = nb;
    a.cap_b = (int)c.w.cap_b;
    a.width = c.net.width;
    a.n_gblk = (c.g.n + TM / 8 - 1) / (TM / 8);
    a.n_sblk = (nb + 7) / 8;
    a.amax = amax;
    a.gate = c.gate;
    a.reruns = c.w.reruns;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c.device);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mlp_fp32_kernel<TM, NJ>, 256, smem);
    const long tiles = (long)a.n_gblk * a.n_sblk;
    const long grid = std::min<long>(tiles, (long)dev_sms * std::max(per_sm, 1));
    if (grid == 0)
        return;
    mlp_fp32_kernel<TM, NJ><<<(unsigned)grid, 256, smem, st>>>(a);
    c.launches++;
}

bool mlp_uses_tc(const Ctx &c)
{
    return c.mlp_precision != 0 && mlp_tc_available() &&
           ((c.net.wp == 160 && c.net.w_tc2 != nullptr) || (c.net.wp == 512 && c.net.w_wide != nullptr));
}

// Largest ReLU output of every trunk layer over all Gaussians x the first nb
// positions already prepared (pos_prep, unscaled), on the FP32 kernel.
void probe_activations(Ctx &c, int nb, float out[8], cudaStream_t st)
{
    unsigned *d = dalloc<unsigned>(c, 8);
    check_cuda(cudaMemsetAsync(d, 0, 8 * sizeof(unsigned), st), "probe reset");
    if (c.net.wp <= 160)
        run_mlp<128, 5>(c, nb, st, d);
    else
        run_mlp<64, 16>(c, nb, st, d);
    unsigned h[8];
    check_cuda(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st), "probe read");
    check_cuda(cudaStreamSynchronize(st), "probe");
    dfree(c, d);
    for (int l = 0; l < 8; l++)
        std::memcpy(&out[l], &h[l], 4);
}

void launch_mlp(Ctx &c, int nb, cudaStream_t st)
{
    if (mlp_uses_tc(c))
    {
        if (c.net.wp == 512)
            launch_mlp_wide(c, nb, st);
        else
            launch_mlp_tc2(c, nb, st);
        return;
    }
    if (c.net.wp <= 160)
        run_mlp<128, 5>(c, nb, st);
    else
        run_mlp<64, 16>(c, nb, st);
}

} // namespace swr
