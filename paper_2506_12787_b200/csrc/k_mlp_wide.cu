// Deformation MLP for wide nets (padded width 512: TrainConfig.width up to 512,
// training.hpp:100; BASELINE config 5) on tcgen05, layer by layer.
//
// Function: deform::predict_residuals (/root/reference/proj/src/deform.cpp:140-207),
// the same factoring as k_mlp_tc2.cu: W x = W_c xc[g] (per scene, cg) + W_p xp[s]
// + b (per position, pterm), FP32-grade products (a_hi w_hi + a_lo w_hi + a_hi w_lo,
// fp16 hi/lo of power-of-two-scaled operands, FP32 accumulation, cross terms
// first).
//
// Why not the fused kernel: a 512-wide layer's FP32 accumulator for 128 rows is
// 512 TMEM columns -- all of TMEM -- and its converted A operand (hi + lo) would
// take as much again, so the layers cannot stay on chip between UMMAs. Here each
// trunk layer is one persistent GEMM over a block of rows: A (activations, fp16
// hi/lo in the UMMA canonical K-major layout) streams from global memory with
// bulk copies, B (the layer's weights, same layout, half of the N columns per
// CTA of the pair) from L2, the CTA pair runs cta_group::2 UMMAs with M = 256
// (128 rows per CTA) and N = 256 (one output half at a time, double-buffered in
// TMEM so the epilogue of one half overlaps the UMMAs of the next), and the
// epilogue writes the next layer's A in the same canonical layout (ReLU,
// + bias or + position and centre terms, scale, split). Layer 0 (no UMMA:
// ReLU(cterm0 + pterm0)) is an elementwise kernel; layer 7's epilogue folds in
// the five heads (FP32 dot products of its output rows) and writes the residual
// planes.
//
// Rows are Gaussian-major, r = g * S + s (S positions of the chunk), so a 128-row
// tile holds whole Gaussians and each Gaussian's centre terms are read once per
// layer.
//
// Layouts (fp16 elements):
//   activations  [row block of 128][K step of 16 (32)][hi | lo][2048]
//   weights      [layer 1..7][N half (2)][CTA rank (2)][K step (32)][hi | lo][2048]
//   a K-step block of 128 rows (or N columns) x 16 K: element (m, kk) at
//   ((kk / 8) * 16 + m / 8) * 64 + (m % 8) * 8 + kk % 8 (core matrices of 8 x 8,
//   LBO = 2048 B between the K halves, SBO = 128 B between 8-row groups).
#include "swr_internal.h"
#include "tc_ptx.cuh"

#include <cuda_fp16.h>
#include <cmath>

#ifdef SWR_TC_DEBUG_WAITS
#define MBAR_WAIT_W(b, p) tc::mbar_wait_dbg(b, p, __LINE__)
#else
#define MBAR_WAIT_W(b, p) tc::mbar_wait(b, p)
#endif

namespace swr
{
namespace
{
constexpr int WW = 512;            // padded width
constexpr int KS = WW / 16;        // K steps per layer
constexpr int BLK = 128 * 16;      // elements of one (K-step, part) block
constexpr int STAGE_BYTES = 4 * BLK * 2; // A hi, A lo, B hi, B lo: 16 KB
constexpr int NSTAGE_W = 8;
constexpr int EPI_W = 8;           // epilogue warps: 4 TMEM lane quarters x 2 column halves
constexpr int THREADS_W = 32 * (EPI_W + 2);
constexpr int kProdW = EPI_W, kMmaW = EPI_W + 1;
constexpr int SMEM_W = NSTAGE_W * STAGE_BYTES + 1024 + 512 + 5 * 128 * 4;

struct WideArgs
{
    const uint16_t *act_in;   // [rows / 128][KS][2][BLK]
    uint16_t *act_out;        // same layout (layers 1..6)
    const uint16_t *w;        // this layer: [2 halves][2 ranks][KS][2][BLK]
    const float *add_bias;    // [512] x 2^k_l (odd layers) or null
    const float *pterm;       // [nb][4][512] x 2^k_l (even layers; bias included)
    const float *cg;          // [np][4][512] centre terms, unscaled
    int cg_j;                 // cg layer slot (l / 2) for even layers, -1 otherwise
    float cscale;             // 2^k_l for the centre terms
    float unscale;            // 2^(k_l - e_l - k_(l-1))
    int rows, S, g0, n, np;   // rows of this block (multiple of 256), positions per Gaussian, first Gaussian
    // heads (layer 7): res planes and weights
    int heads;
    const float *hw;          // [5][512] head weights (FP32)
    const float *hb;          // [5]
    float hscale;             // 2^-k_7: the activations carry 2^k_7
    float *res;               // [5][cap_b][np]
    int cap_b;
};

__device__ __forceinline__ uint32_t pack2(float lo, float hi)
{
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float relu_nan(float x)
{
    float r;
    asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
    return r;
}

// 16 values of row m (within its 128-row block) at K step ks -> hi / lo blocks
__device__ __forceinline__ void store_split16(uint16_t *act, size_t rblk, int ks, int m, const float (&v)[16])
{
    uint32_t h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; i++)
    {
        h[i] = pack2(v[2 * i], v[2 * i + 1]);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&h[i]));
        l[i] = pack2(v[2 * i] - hf.x, v[2 * i + 1] - hf.y); // exact: at most 13 significant bits
    }
    uint16_t *base = act + (rblk * KS + ks) * 2 * BLK;
#pragma unroll
    for (int half = 0; half < 2; half++)
    {
        const size_t off = (size_t)((half * 16 + m / 8) * 64 + (m % 8) * 8);
        *reinterpret_cast<uint4 *>(base + off) = make_uint4(h[4 * half], h[4 * half + 1], h[4 * half + 2], h[4 * half + 3]);
        *reinterpret_cast<uint4 *>(base + BLK + off) =
            make_uint4(l[4 * half], l[4 * half + 1], l[4 * half + 2], l[4 * half + 3]);
    }
}

// Layer 0: ReLU(cterm0[g] + pterm0[s]) x 2^k_0 -> A of layer 1. One thread per
// (row, K step).
__global__ void __launch_bounds__(256) wide_layer0_kernel(const float *__restrict__ cg,
                                                         const float *__restrict__ pterm, float cscale, int rows,
                                                         int S, int g0, int np, uint16_t *__restrict__ act)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)rows * KS)
        return;
    const int r = (int)(idx % rows), ks = (int)(idx / rows); // consecutive threads: consecutive rows
    const int g = g0 + r / S, s = r % S;
    const float *c = cg + ((size_t)min(g, np - 1) * 4 + 0) * WW + ks * 16; // padding rows: any valid Gaussian
    const float *p = pterm + ((size_t)s * 4 + 0) * WW + ks * 16;
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4)
    {
        const float4 a = *reinterpret_cast<const float4 *>(c + i), b = *reinterpret_cast<const float4 *>(p + i);
        v[i] = relu_nan(__fadd_rn(__fmul_rn(a.x, cscale), b.x));
        v[i + 1] = relu_nan(__fadd_rn(__fmul_rn(a.y, cscale), b.y));
        v[i + 2] = relu_nan(__fadd_rn(__fmul_rn(a.z, cscale), b.z));
        v[i + 3] = relu_nan(__fadd_rn(__fmul_rn(a.w, cscale), b.w));
    }
    store_split16(act, (size_t)(r / 128), ks, r % 128, v);
}

// One trunk layer over a block of rows: persistent CTA pairs, pair tile = 256 rows.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS_W, 1) mlp_wide_kernel(WideArgs a)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ring = smem;
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + NSTAGE_W * STAGE_BYTES);
    uint64_t *full = bars, *empty = bars + NSTAGE_W;
    uint64_t *acc_full = empty + NSTAGE_W, *acc_empty = acc_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
    float *hpart = reinterpret_cast<float *>(bars + 64); // [5][128] heads partials of column half 0

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_rank();
    if (threadIdx.x == 0)
    {
        for (int s = 0; s < NSTAGE_W; s++)
        {
            tc::mbar_init(&full[s], rank == 0 ? 2 : 1); // leader: own bytes + the peer's relay
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++)
        {
            tc::mbar_init(&acc_full[b], 1);
            tc::mbar_init(&acc_empty[b], 2 * EPI_W);
        }
        tc::fence_mbar_init();
    }
    if (warp == kMmaW)
        tc::tmem_alloc2<512>(tmem_slot);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int ntiles = a.rows / 256;
    const int mine = cluster < ntiles ? (ntiles - 1 - cluster) / nclusters + 1 : 0;

    if (warp == kProdW)
    {
        int stage = 0;
        uint32_t ph = 0;
        for (int it = 0; it < mine; it++)
        {
            const int t = cluster + it * nclusters;
            const size_t rblk = (size_t)t * 2 + rank;
            for (int nh = 0; nh < 2; nh++)
                for (int ks = 0; ks < KS; ks++)
                {
                    MBAR_WAIT_W(&empty[stage], ph ^ 1);
                    if (tc::elect_one())
                    {
                        uint8_t *dst = ring + stage * STAGE_BYTES;
                        tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                        tc::bulk_g2s(dst, a.act_in + (rblk * KS + ks) * 2 * BLK, 2 * BLK * 2, &full[stage]);
                        tc::bulk_g2s(dst + 2 * BLK * 2, a.w + (((size_t)nh * 2 + rank) * KS + ks) * 2 * BLK,
                                     2 * BLK * 2, &full[stage]);
                    }
                    __syncwarp();
                    if (++stage == NSTAGE_W)
                    {
                        stage = 0;
                        ph ^= 1;
                    }
                }
        }
    }
    else if (warp == kMmaW && rank != 0)
    {
        int stage = 0;
        uint32_t ph = 0;
        for (int j = 0; j < mine * 2 * KS; j++)
        {
            MBAR_WAIT_W(&full[stage], ph);
            if (tc::elect_one())
                tc::mbar_arrive_remote_relaxed(tc::mapa(&full[stage], 0));
            __syncwarp();
            if (++stage == NSTAGE_W)
            {
                stage = 0;
                ph ^= 1;
            }
        }
    }
    else if (warp == kMmaW)
    {
        constexpr uint32_t IDESC = tc::make_idesc(0, 256, 256);
        constexpr uint32_t LBO = 2048;
        constexpr uint32_t DH = tc::desc_hi(128);
        int stage = 0;
        uint32_t ph = 0, eph = 0;
        const uint32_t r_base = tc::smem_u32(ring);
        int nacc = 0;
        for (int it = 0; it < mine; it++)
            for (int nh = 0; nh < 2; nh++, nacc++)
            {
                const int buf = nh;
                if (nacc >= 2)
                {
                    MBAR_WAIT_W(&acc_empty[buf], (eph >> buf) & 1);
                    eph ^= 1u << buf;
                }
                tc::tc_fence_after();
                const uint32_t d = tmem + buf * 256;
                for (int ks = 0; ks < KS; ks++)
                {
                    MBAR_WAIT_W(&full[stage], ph);
                    tc::tc_fence_after();
                    if (tc::elect_one())
                    {
                        const uint32_t s0 = r_base + stage * STAGE_BYTES;
                        const uint64_t ahi = tc::desc_of(tc::desc_lo(s0, LBO), DH);
                        const uint64_t alo = tc::desc_of(tc::desc_lo(s0 + BLK * 2, LBO), DH);
                        const uint64_t bhi = tc::desc_of(tc::desc_lo(s0 + 2 * BLK * 2, LBO), DH);
                        const uint64_t blo = tc::desc_of(tc::desc_lo(s0 + 3 * BLK * 2, LBO), DH);
                        // cross terms first (small while the accumulator is small), then hi x hi
                        tc::mma2_f16(d, alo, bhi, IDESC, ks > 0 ? 1u : 0u);
                        tc::mma2_f16(d, ahi, blo, IDESC, 1u);
                        tc::mma2_f16(d, ahi, bhi, IDESC, 1u);
                        tc::mma2_commit(&empty[stage], 3);
                        if (ks == KS - 1)
                            tc::mma2_commit(&acc_full[buf], 3);
                    }
                    __syncwarp();
                    if (++stage == NSTAGE_W)
                    {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
    }
    else
    {
        // epilogue: warp w -> TMEM lane quarter q (rows 32q..32q+31 of the CTA's 128),
        // column half ch (columns 128 ch .. 128 ch + 127 of the 256-wide output half)
        const int q = warp & 3, ch = warp >> 2;
        const int m = 32 * q + lane; // row within the CTA block
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        uint32_t fph = 0;
        float hacc[5];
        for (int it = 0; it < mine; it++)
        {
            const int t = cluster + it * nclusters;
            const size_t rblk = (size_t)t * 2 + rank;
            const int r = (int)rblk * 128 + m; // row within the launch block
            const int g = a.g0 + r / a.S, s = r % a.S;
#pragma unroll
            for (int h = 0; h < 5; h++)
                hacc[h] = 0.0f;
            for (int nh = 0; nh < 2; nh++)
            {
                MBAR_WAIT_W(&acc_full[nh], (fph >> nh) & 1);
                fph ^= 1u << nh;
                tc::tc_fence_after();
                for (int c = 0; c < 8; c++)
                {
                    const int n0 = nh * 256 + ch * 128 + c * 16; // output column
                    float v[16];
                    tc::tmem_ld16(tmem + nh * 256 + ch * 128 + c * 16 + lane_off, v);
                    float add[16];
                    if (a.cg_j >= 0)
                    {
                        const float *cp = a.cg + ((size_t)min(g, a.np - 1) * 4 + a.cg_j) * WW + n0;
                        const float *pp = a.pterm + ((size_t)s * 4 + a.cg_j) * WW + n0;
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                        {
                            const float4 cv = *reinterpret_cast<const float4 *>(cp + i);
                            const float4 pv = *reinterpret_cast<const float4 *>(pp + i);
                            add[i] = __fadd_rn(__fmul_rn(cv.x, a.cscale), pv.x);
                            add[i + 1] = __fadd_rn(__fmul_rn(cv.y, a.cscale), pv.y);
                            add[i + 2] = __fadd_rn(__fmul_rn(cv.z, a.cscale), pv.z);
                            add[i + 3] = __fadd_rn(__fmul_rn(cv.w, a.cscale), pv.w);
                        }
                    }
                    else
                    {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                        {
                            const float4 bv = *reinterpret_cast<const float4 *>(a.add_bias + n0 + i);
                            add[i] = bv.x;
                            add[i + 1] = bv.y;
                            add[i + 2] = bv.z;
                            add[i + 3] = bv.w;
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 16; i++)
                        v[i] = relu_nan(__fmaf_rn(v[i], a.unscale, add[i]));
                    if (a.heads)
                    {
#pragma unroll
                        for (int h = 0; h < 5; h++)
                        {
                            const float *wr = a.hw + (size_t)h * WW + n0;
                            float acc = hacc[h];
#pragma unroll
                            for (int i = 0; i < 16; i++)
                                acc = __fmaf_rn(v[i], wr[i], acc);
                            hacc[h] = acc;
                        }
                    }
                    else
                        store_split16(a.act_out, rblk, n0 / 16, m, v);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    tc::mbar_arrive_remote_relaxed(tc::mapa(&acc_empty[nh], 0));
            }
            if (a.heads)
            {
                // combine the two column halves of each row, then the residual planes
                if (ch == 0)
#pragma unroll
                    for (int h = 0; h < 5; h++)
                        hpart[h * 128 + m] = hacc[h];
                tc::named_bar(1 + q, 64);
                if (ch == 1 && g < a.n)
                {
                    const size_t plane = (size_t)a.cap_b * a.np;
#pragma unroll
                    for (int h = 0; h < 5; h++)
                        a.res[h * plane + (size_t)s * a.np + g] =
                            __fadd_rn(__fmul_rn(__fadd_rn(hpart[h * 128 + m], hacc[h]), a.hscale), a.hb[h]);
                }
                tc::named_bar(1 + q, 64);
            }
        }
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == kMmaW)
    {
        tc::tc_fence_after();
        tc::tmem_dealloc2<512>(tmem);
    }
}

uint16_t f16b(float x) { return __half_as_ushort(__float2half_rn(x)); }
float f16f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

int scale_exp_w(float max_abs)
{
    if (!(max_abs > 0.0f) || !std::isfinite(max_abs))
        return 0;
    int e2 = 0;
    std::frexp(max_abs, &e2);
    return 14 - e2;
}
} // namespace

// Packed weights of layers 1..7 (whT: [7][512][512] k-major, zero padded), the
// heads (FP32, [5][512]) and the scaled biases.
void prepare_wide_weights(Ctx &c, const std::vector<float> &whT, const std::vector<float> &heads,
                          const std::vector<float> &bias)
{
    NetDev &nt = c.net;
    for (int l = 1; l < 8; l++)
    {
        float m = 0.0f;
        for (size_t i = 0; i < (size_t)WW * WW; i++)
            m = std::max(m, std::fabs(whT[(size_t)(l - 1) * WW * WW + i]));
        nt.tc_exp[l] = scale_exp_w(m);
    }
    nt.tc_exp[0] = 0;
    nt.tc_exp[8] = 0;
    const size_t per_layer = (size_t)2 * 2 * KS * 2 * BLK;
    std::vector<uint16_t> packed(7 * per_layer);
    for (int l = 1; l < 8; l++)
    {
        const float sc = std::ldexp(1.0f, nt.tc_exp[l]);
        uint16_t *L = packed.data() + (size_t)(l - 1) * per_layer;
        for (int nh = 0; nh < 2; nh++)
            for (int rk = 0; rk < 2; rk++)
                for (int ks = 0; ks < KS; ks++)
                {
                    uint16_t *hi = L + (((size_t)nh * 2 + rk) * KS + ks) * 2 * BLK, *lo = hi + BLK;
                    for (int nl = 0; nl < 128; nl++)
                        for (int kk = 0; kk < 16; kk++)
                        {
                            const int n = nh * 256 + rk * 128 + nl, k = ks * 16 + kk;
                            const float ws = whT[((size_t)(l - 1) * WW + k) * WW + n] * sc;
                            const size_t idx = (size_t)((kk / 8) * 16 + nl / 8) * 64 + (nl % 8) * 8 + kk % 8;
                            hi[idx] = f16b(ws);
                            lo[idx] = f16b(ws - f16f(hi[idx]));
                        }
                }
    }
    void *d = nullptr;
    check_cuda(cudaMalloc(&d, packed.size() * 2), "cudaMalloc wide weights");
    c.allocs.push_back(d);
    check_cuda(cudaMemcpy(d, packed.data(), packed.size() * 2, cudaMemcpyHostToDevice), "upload wide weights");
    nt.w_wide = static_cast<uint16_t *>(d);
    const int *k = nt.tc_ascale;
    std::vector<float> bs(bias.size());
    for (size_t i = 0; i < bias.size(); i++)
        bs[i] = std::ldexp(bias[i], k[i / WW]);
    nt.bias_tc = upload(c, bs);
    (void)heads; // the heads run in FP32 from nt.heads
}

void launch_mlp_wide(Ctx &c, int nb, cudaStream_t st)
{
    static DeviceOnce once;
    const int max_clusters = once.get(c.device, [] {
        check_cuda(cudaFuncSetAttribute(mlp_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_W),
                   "wide mlp smem attribute");
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2, 1, 1);
        cfg.blockDim = dim3(THREADS_W, 1, 1);
        cfg.dynamicSmemBytes = SMEM_W;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int mc = 0;
        check_cuda(cudaOccupancyMaxActiveClusters(&mc, mlp_wide_kernel, &cfg), "wide mlp cluster occupancy");
        if (mc < 1)
            check_cuda(cudaErrorLaunchOutOfResources, "wide mlp: no CTA pair fits on this device");
        return mc;
    });
    NetDev &nt = c.net;
    const int S = nb;
    // rows r = g * S + s in blocks of whole Gaussians, a multiple of 256 rows
    const int64_t block_rows_target = c.wide_block_rows; // default 2M rows: 2 x 4 GiB activation buffers
    int gper = int(std::max<int64_t>(1, block_rows_target / S));
    while ((int64_t(gper) * S) % 256)
        gper++;
    const int64_t brows = int64_t(gper) * S;
    if (c.w.wide_rows < brows)
    {
        dfree(c, c.w.wide_act[0]);
        dfree(c, c.w.wide_act[1]);
        c.w.wide_act[0] = dalloc<uint16_t>(c, size_t(brows) * WW * 2);
        c.w.wide_act[1] = dalloc<uint16_t>(c, size_t(brows) * WW * 2);
        c.w.wide_rows = brows;
    }
    const int *k = nt.tc_ascale;
    for (int g0 = 0; g0 < c.g.n; g0 += gper)
    {
        const int gcnt = std::min(gper, c.g.n - g0);
        int64_t rows = int64_t(gcnt) * S;
        rows = (rows + 255) / 256 * 256; // the last block's padding rows are computed, never written out
        {
            const int64_t total = rows * KS;
            wide_layer0_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
                nt.cg, c.w.pterm, std::ldexp(1.0f, k[0]), int(rows), S, g0, c.g.np, c.w.wide_act[0]);
            c.launches++;
        }
        for (int l = 1; l < 8; l++)
        {
            WideArgs a{};
            a.act_in = c.w.wide_act[(l - 1) & 1];
            a.act_out = c.w.wide_act[l & 1];
            a.w = nt.w_wide + (size_t)(l - 1) * 2 * 2 * KS * 2 * BLK;
            const bool even = (l % 2) == 0;
            a.add_bias = even ? nullptr : nt.bias_tc + (size_t)l * WW;
            a.pterm = c.w.pterm;
            a.cg = nt.cg;
            a.cg_j = even ? l / 2 : -1;
            a.cscale = std::ldexp(1.0f, k[l]);
            a.unscale = std::ldexp(1.0f, k[l] - nt.tc_exp[l] - k[l - 1]);
            a.rows = int(rows);
            a.S = S;
            a.g0 = g0;
            a.n = c.g.n;
            a.np = c.g.np;
            a.heads = l == 7;
            a.hw = nt.heads;
            a.hb = nt.hbias;
            a.hscale = std::ldexp(1.0f, -k[7]);
            a.res = c.w.res;
            a.cap_b = int(c.w.cap_b);
            const int grid = 2 * std::min<int>(max_clusters, int(rows / 256));
            mlp_wide_kernel<<<grid, THREADS_W, SMEM_W, st>>>(a);
            c.launches++;
        }
    }
}

} // namespace swr
