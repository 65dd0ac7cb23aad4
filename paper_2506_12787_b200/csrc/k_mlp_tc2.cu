// Deformation MLP on tcgen05, CTA pairs, TWO TILES IN FLIGHT ("ping-pong").
// The tensor-core MLP of libswr (mlp_precision SWR_MLP_FP16X3 / SWR_MLP_FP16).
//
// Function: deform::predict_residuals (/root/reference/proj/src/deform.cpp:140-207).
// The input row x = [xc[g] | xp[s]] splits W x into W_c xc[g] (cterm: a
// per-Gaussian FP32 constant computed once per scene) + W_p xp[s] + b (pterm:
// per position, FP32, added in the epilogue). The seven hidden->hidden products
// and the heads run on the tensor core with FP32 accumulation in TMEM; A
// operands are converted in place in TMEM.
//
// Precision (SWR_MLP_FP16X3, FP32-grade): every product is a_hi w_hi + a_lo w_hi
// + a_hi w_lo with fp16 hi/lo splits (11 + 11 significant bits, ~2^-22 per
// product, the dropped a_lo w_lo term included). Weights are pre-scaled per
// layer by a power of two 2^e_l (max |w| 2^e_l in [2^13, 2^14)) so both halves
// stay in fp16's normal range; the accumulator then holds 2^e_l W h, and the
// epilogue re-scales it exactly (fma(acc, 2^(k_l - e_l - k_(l-1)), add): the
// power-of-two product is exact, so one rounding, as in acc + add). Each trunk
// layer's output carries a scale 2^k_l, chosen at scene load so that 2^k_l
// times the largest ReLU output of that layer the FP32 kernel sees over all
// Gaussians x 16 probe positions is <= 65504 / 64: small activations then keep
// both fp16 halves normal (an unscaled 0.05 would leave its lo half subnormal,
// ~2^-20 instead of 2^-22) and large ones stay below fp16's 65504. The 2^k_l are
// folded into the position terms (pos_prep), the biases (bias_tc) and the cterm
// blocks, and taken out in the heads readout (2^-(e_h + k_7)). An activation that still overflows
// fp16 turns into NaN in every product it feeds (hi = inf, lo = -inf); the ReLU
// is max.NaN so the NaN reaches the residuals, where the setup kernel flags it
// and the host re-runs the chunk on the FP32 CUDA-core kernel (capi.cpp).
// SWR_MLP_FP16 runs the a_hi w_hi pass only (~2^-11, a fast tier not used for
// reported numbers).
//
// Why two tiles: one tile's layers back to back leave the tensor core waiting
// for the epilogue's conversion of layer l before layer l+1. Here a CTA pair
// alternates two tiles X and Y of the same 32 Gaussians (positions
// s0..s0+7 and s0+8..s0+15): while the tensor core runs layer l of X, the
// epilogue converts layer l-1 of Y and vice versa, so each conversion has a
// whole layer of the other tile (2,400 cycles at 3 passes) to finish in. Three
// 160-column TMEM regions suffice: step m (tile m%2, layer (m/2)%8) writes
// region m%3 and reads region (m-2)%3 (the same tile's previous layer, converted
// in place); region (m-1)%3 is the other tile's accumulator being converted
// meanwhile. Each weight stage (one per layer, full N = 160, half the columns
// per CTA) serves both tiles.
//
// Heads: each tile has its own N = 16 heads accumulator (TMEM columns 480-495 / 496-511),
// so heads Y never waits for heads X's readout, and the group-0 warps read the previous
// super-tile's heads out while the tensor core runs the next layer 1 (round 2; the
// clock64 trace, tools/tc2_trace.py: super-tile period 40.8k -> 40.6k cycles).
//
// Layer 0 has no UMMA: the epilogue writes ReLU(cterm0 + pterm0) (fp16 hi/lo)
// straight into TMEM from a cterm block in shared memory. Layers 2, 4, 6 add
// their cterm block in the epilogue too (round 1 seeded those accumulators with
// tcgen05.cp; starting every accumulator from zero lets the cross-term passes
// run first, see issue_layer, and cost < 1% in time). The five heads run
// on the tensor core (N = 32, heads 0-4 real) from layer 7's converted output
// into TMEM columns 480-511, their B operand resident in shared memory; issue
// order at a super-tile boundary is ... X7, Y7, heads X, heads Y, X'1 ... (X'0 /
// Y'0 are written by the epilogue once heads X / Y have read the regions they
// reuse).
//
// Measured (round 1, bf16 splits -- same instruction count as fp16; one
// 256-position chunk, 50k Gaussians): 8.2-8.3 ms (33.0 ms per 1,024 spectra in
// bench.py). A clock64 timeline (tools/tc2_trace.py, hooks build) shows ~2,500
// cycles per layer step against 2,400 for the UMMAs alone and ~4,000 cycles lost
// per super-tile boundary; the epilogue (40 16-column conversions per step on
// 20 warps) is the limiting chain, and the UMMA issuer shares its SM
// sub-partition with it.
//
// Warps (704 threads per CTA with the default 5 column groups): 0-19 epilogue
// (5 column groups x 4 TMEM lane quarters; group g converts 16-column chunks g
// and g + 5), 20 producer (TMA of this CTA's half of each weight stage + cterm
// blocks), 21 UMMA issuer (leader CTA) / stage relay (peer CTA).
#include "swr_internal.h"
#include "tc_ptx.cuh"

#include <cuda_fp16.h>
#include <cmath>
#include <cstdlib>
#include <cstring>

#ifdef SWR_TC_DEBUG_WAITS
#define MBAR_WAIT_PLAIN(b, p) tc::mbar_wait_dbg(b, p, __LINE__)
#else
#define MBAR_WAIT_PLAIN(b, p) tc::mbar_wait(b, p)
#endif

namespace swr
{

namespace
{
constexpr int TM = 128;                   // rows per CTA: 32 Gaussians x 4 positions
constexpr int TG = 32, TS = 4;
constexpr int SUPER_S = 16;               // positions per super-tile (tiles X, Y x 2 CTAs x 4)
constexpr int WPC = 160, KSTEPS = 10, NL = 8, NHEADS = 5;
constexpr int NHEAD_N = 16;               // heads UMMA N (5 real columns; the N granularity of a CTA pair)
constexpr int HEAD_COL = 3 * WPC;         // heads accumulators: TMEM columns 480-495 (tile X), 496-511 (tile Y)
constexpr int HB_BYTES = KSTEPS * 2 * (NHEAD_N / 2) * 16 * 2; // heads B operand per CTA: 5 KB
constexpr int KB = WPC / 2 * 16 * 2;      // one K step, one operand (hi or lo), this CTA's 80 columns: 2.5 KB
constexpr int W_BYTES = KSTEPS * 2 * KB;  // one layer's weights per CTA: 50 KB
constexpr int C_BLOCK = WPC * TG * 4;     // one layer's cterm block: [40 column groups][32 rows][4] f32
constexpr int SLOT = W_BYTES;             // weight stage
constexpr int NSTAGE = 2;                 // weight stages (layers 1..7), each serving both tiles
constexpr int NCSTAGE = 2;                // cterm blocks of layers 0/2/4/6, read by the epilogue
#ifndef SWR_TC2_GROUPS
#define SWR_TC2_GROUPS 5 // 5: every epilogue warp converts two chunks (measured ~1% faster than 6 and 7)
#endif
constexpr int NGRP = SWR_TC2_GROUPS;
constexpr int EPI_WARPS = 4 * NGRP, EPI_THREADS = 32 * EPI_WARPS;
constexpr int THREADS = 32 * (EPI_WARPS + 2);
constexpr int kProducerWarp = EPI_WARPS, kMmaWarp = EPI_WARPS + 1;
constexpr int PROW = 4 * WPC;             // pterm row of one position (layers 0, 2, 4, 6)
constexpr int SMEM_RING = NSTAGE * SLOT;
constexpr int SMEM_CRING = NCSTAGE * C_BLOCK;
constexpr int SMEM_P = 2 * 2 * TS * PROW * 4;         // [buffer][tile][4 positions][640]
constexpr int SMEM_CONST = (8 * WPC + 8) * 4;
// w_full[2], w_empty[2], c_full[2], c_empty[2], acc[2 tiles], a_ready[2 tiles], acc_h[2 tiles], h_free[2 tiles]
constexpr int NBARS = 2 * NSTAGE + 2 * NCSTAGE + 2 + 2 + 2 + 2;
constexpr int SMEM_BYTES = SMEM_RING + SMEM_CRING + SMEM_P + HB_BYTES + SMEM_CONST + NBARS * 8 + 16 + 1024;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

__host__ __device__ constexpr bool has_xc(int l) { return (l & 1) == 0; } // layers 0, 2, 4, 6 read x

struct Tc2Args
{
    const uint16_t *w;     // packed weights, layers 1..7: [layer][rank][10 K][hi | lo][80 cols x 16] fp16 (x 2^e_l)
    const float *cterm;    // [n/32 blocks][4 layers][40][32][4] x 2^k (cterm_pack_kernel)
    const float *bias;     // [8][160]
    const float *pterm;    // [nb][4][160]
    const uint16_t *wh;    // heads B operand: [rank][10 K][hi | lo][16 cols x 16] fp16 (x 2^e_h)
    const float *hbias;    // [5]
    float *res;            // [5][cap_b][np]
    int n, np, nb, cap_b, n_sblk, ntiles;
    float unscale[9];      // 2^-e_l of trunk layers 1..7 (index l), [8] = heads; [0] unused (layer 0: no UMMA)
    long long *trace;      // -DSWR_TC_DEBUG_HOOKS builds: [4][48] clock64 stamps of CTA 0 (steps 16..63)
};
#ifdef SWR_TC_DEBUG_HOOKS
constexpr bool kHooks = true;
#else
constexpr bool kHooks = false;
#endif
__device__ __forceinline__ void stamp2(const Tc2Args &a, int kind, int m)
{
    if (kHooks && a.trace && blockIdx.x == 0 && m >= 16 && m < 64)
        a.trace[kind * 48 + m - 16] = clock64(); // kinds 0-2 MMA warp, 3-6 epilogue (tools/tc2_trace.py)
    (void)kind;
}

__device__ __forceinline__ uint32_t pack_f16(float lo, float hi)
{
    __half2 h = __floats2half2_rn(lo, hi); // cvt.rn.f16x2.f32: lo -> bits 0-15
    return *reinterpret_cast<uint32_t *>(&h);
}
// ReLU that keeps NaN (max.NaN): an fp16 overflow upstream stays visible in the residuals
__device__ __forceinline__ float relu_nan(float x)
{
    float r;
    asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
    return r;
}

// v = ReLU(acc * unscale + add) -> 8 columns of fp16 hi pairs, then 8 columns of
// lo pairs (lo = v - float(hi) is exact in FP32: at most 13 significant bits)
__device__ __forceinline__ void relu_split16(const float (&acc)[16], const float (&add)[16], float unscale,
                                             uint32_t (&o)[16])
{
#pragma unroll
    for (int i = 0; i < 8; i++)
    {
        float2 v = __ffma2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), make_float2(unscale, unscale),
                              make_float2(add[2 * i], add[2 * i + 1]));
        v.x = relu_nan(v.x);
        v.y = relu_nan(v.y);
        const uint32_t h = pack_f16(v.x, v.y);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&h));
        const float2 lo = __ffma2_rn(hf, make_float2(-1.0f, -1.0f), v);
        o[i] = h;
        o[8 + i] = pack_f16(lo.x, lo.y);
    }
}

__device__ __forceinline__ void lds16(const float *p, float (&v)[16])
{
    const uint32_t a = tc::smem_u32(p);
#pragma unroll
    for (int i = 0; i < 4; i++)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[4 * i]), "=f"(v[4 * i + 1]), "=f"(v[4 * i + 2]), "=f"(v[4 * i + 3])
                     : "r"(a + 16 * i));
}

__device__ __forceinline__ void super_origin(const Tc2Args &a, int tile, int &g0, int &s0)
{
    g0 = (tile / a.n_sblk) * TG;
    s0 = (tile % a.n_sblk) * SUPER_S;
}

// all UMMAs of one layer step, A from TMEM: the two cross-term passes (a_lo w_hi,
// a_hi w_lo) first, then a_hi w_hi. The tensor core's FP32 accumulation truncates
// at each UMMA relative to the running sum, so summing the small cross terms
// while the accumulator is still small leaves ~10 full-size truncations per
// layer instead of 30.
template <bool SPLIT>
__device__ __forceinline__ void issue_layer(uint32_t d, uint32_t bh, uint32_t areg)
{
    constexpr uint32_t LBO = WPC / 2 / 8 * 128;
    constexpr uint32_t IDESC = tc::make_idesc(0, 2 * TM, WPC); // f16 x f16 -> f32
    constexpr uint32_t DH = tc::desc_hi(128);
    const uint32_t b0 = tc::desc_lo(bh, LBO);
    if (SPLIT)
    {
#pragma unroll
        for (int k = 0; k < KSTEPS; k++)
            tc::mma2_f16_ts(d, areg + 16 * k + 8, tc::desc_of(b0 + (k * 2 * KB >> 4), DH), IDESC, k > 0 ? 1u : 0u);
#pragma unroll
        for (int k = 0; k < KSTEPS; k++)
            tc::mma2_f16_ts(d, areg + 16 * k, tc::desc_of(b0 + ((k * 2 + 1) * KB >> 4), DH), IDESC, 1u);
    }
#pragma unroll
    for (int k = 0; k < KSTEPS; k++)
        tc::mma2_f16_ts(d, areg + 16 * k, tc::desc_of(b0 + (k * 2 * KB >> 4), DH), IDESC, (SPLIT || k > 0) ? 1u : 0u);
}
// the heads: N = 32, A = layer 7's converted output in TMEM, B resident in shared
// memory; same pass order as issue_layer
template <bool SPLIT>
__device__ __forceinline__ void issue_heads(uint32_t d, uint32_t bh, uint32_t areg)
{
    constexpr uint32_t KBH = NHEAD_N / 2 * 16 * 2, LBO = NHEAD_N / 2 / 8 * 128;
    constexpr uint32_t IDESC = tc::make_idesc(0, 2 * TM, NHEAD_N);
    constexpr uint32_t DH = tc::desc_hi(128);
    const uint32_t b0 = tc::desc_lo(bh, LBO);
    if (SPLIT)
    {
#pragma unroll
        for (int k = 0; k < KSTEPS; k++)
            tc::mma2_f16_ts(d, areg + 16 * k + 8, tc::desc_of(b0 + (k * 2 * KBH >> 4), DH), IDESC, k > 0 ? 1u : 0u);
#pragma unroll
        for (int k = 0; k < KSTEPS; k++)
            tc::mma2_f16_ts(d, areg + 16 * k, tc::desc_of(b0 + ((k * 2 + 1) * KBH >> 4), DH), IDESC, 1u);
    }
#pragma unroll
    for (int k = 0; k < KSTEPS; k++)
        tc::mma2_f16_ts(d, areg + 16 * k, tc::desc_of(b0 + (k * 2 * KBH >> 4), DH), IDESC, (SPLIT || k > 0) ? 1u : 0u);
}
// per lane (row = Gaussian g0 + lane): 16 cterm columns of a chunk from a cterm
// block in shared memory ([40 column groups][32 rows][4] f32; 512 contiguous bytes
// per 4 columns, so each ld.shared.v4 of a warp is conflict-free)
__device__ __forceinline__ void lds_cterm16(const uint8_t *blk, int chunk, int lane, float (&v)[16])
{
    const uint32_t a0 = tc::smem_u32(blk) + (uint32_t)(chunk * 4 * TG * 16 + lane * 16);
#pragma unroll
    for (int i = 0; i < 4; i++)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[4 * i]), "=f"(v[4 * i + 1]), "=f"(v[4 * i + 2]), "=f"(v[4 * i + 3])
                     : "r"(a0 + i * TG * 16));
}

template <bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) mlp_tc2_kernel(Tc2Args a)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ring = smem;                                    // weight stages (layers 1..7)
    uint8_t *cring = ring + SMEM_RING;                       // cterm blocks (layers 0/2/4/6)
    float *pbuf = reinterpret_cast<float *>(cring + SMEM_CRING); // [2][2][4][640]
    uint8_t *hb = reinterpret_cast<uint8_t *>(pbuf + 2 * 2 * TS * PROW); // heads B operand (this CTA's 16 columns)
    float *sbias = reinterpret_cast<float *>(hb + HB_BYTES);            // [8][160]
    float *shb = sbias + 8 * WPC;                                       // [8]
    uint64_t *bars = reinterpret_cast<uint64_t *>(shb + 8);
    uint64_t *w_full = bars, *w_empty = bars + NSTAGE;  // w_full (leader) also counts the peer's relay
    uint64_t *c_full = w_empty + NSTAGE, *c_empty = c_full + NCSTAGE; // this CTA's cterm blocks (epilogue)
    uint64_t *acc = c_empty + NCSTAGE;                  // [tile]: a layer's accumulator complete
    uint64_t *a_ready = acc + 2;                        // [tile] (leader): a layer converted, both CTAs
    uint64_t *acc_h = a_ready + 2;                      // [tile]: heads accumulator complete
    uint64_t *h_free = acc_h + 2;                       // [tile] (leader) heads accumulator read out, both CTAs
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + NBARS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_rank();
    if (threadIdx.x == 0)
    {
        for (int s = 0; s < NSTAGE; s++)
        {
            tc::mbar_init(&w_full[s], rank == 0 ? 2 : 1);
            tc::mbar_init(&w_empty[s], 1);
        }
        for (int s = 0; s < NCSTAGE; s++)
        {
            tc::mbar_init(&c_full[s], 1);
            tc::mbar_init(&c_empty[s], EPI_WARPS);
        }
        for (int t = 0; t < 2; t++)
        {
            tc::mbar_init(&acc[t], 1);
            tc::mbar_init(&a_ready[t], 2 * EPI_WARPS);
            tc::mbar_init(&acc_h[t], 1);
        }
        for (int t = 0; t < 2; t++)
            tc::mbar_init(&h_free[t], 2 * 4); // the 4 group-0 warps of both CTAs
        tc::fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 8 * WPC; i += THREADS)
        sbias[i] = a.bias[i];
    for (int i = threadIdx.x; i < HB_BYTES / 16; i += THREADS)
        reinterpret_cast<uint4 *>(hb)[i] = reinterpret_cast<const uint4 *>(a.wh + (size_t)rank * HB_BYTES / 2)[i];
    tc::fence_proxy_async_smem(); // read by the tensor core
    if (threadIdx.x < NHEADS)
        shb[threadIdx.x] = a.hbias[threadIdx.x];
    if (warp == kMmaWarp)
        tc::tmem_alloc2<512>(tmem_slot);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int mine = cluster < a.ntiles ? (a.ntiles - 1 - cluster) / nclusters + 1 : 0;

    if (warp == kProducerWarp)
    {
        int stage = 0, cstage = 0;
        uint32_t ph = 0, cph = 0;
        for (int it = 0; it < mine; it++)
        {
            int g0, s0;
            super_origin(a, cluster + it * nclusters, g0, s0);
            for (int l = 0; l < NL; l++)
            {
                if (has_xc(l))
                {
                    MBAR_WAIT_PLAIN(&c_empty[cstage], cph ^ 1);
                    if (tc::elect_one())
                    {
                        tc::mbar_arrive_expect_tx(&c_full[cstage], C_BLOCK);
                        tc::bulk_g2s(cring + cstage * C_BLOCK,
                                     reinterpret_cast<const uint8_t *>(a.cterm) + ((size_t)(g0 / TG) * 4 + l / 2) * C_BLOCK,
                                     C_BLOCK, &c_full[cstage]);
                    }
                    __syncwarp();
                    if (++cstage == NCSTAGE)
                    {
                        cstage = 0;
                        cph ^= 1;
                    }
                }
                if (l >= 1)
                {
                    MBAR_WAIT_PLAIN(&w_empty[stage], ph ^ 1);
                    if (tc::elect_one())
                    {
                        tc::mbar_arrive_expect_tx(&w_full[stage], W_BYTES);
                        tc::bulk_g2s(ring + stage * SLOT,
                                     reinterpret_cast<const uint8_t *>(a.w) + ((size_t)(l - 1) * 2 + rank) * W_BYTES,
                                     W_BYTES, &w_full[stage]);
                    }
                    __syncwarp();
                    if (++stage == NSTAGE)
                    {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    }
    else if (warp == kMmaWarp && rank != 0)
    {
        // peer CTA: tell the leader when this CTA's half of each weight stage has landed
        int stage = 0;
        uint32_t ph = 0;
        for (int j = 0; j < mine * (NL - 1); j++)
        {
            MBAR_WAIT_PLAIN(&w_full[stage], ph);
            if (tc::elect_one())
                tc::mbar_arrive_remote_relaxed(tc::mapa(&w_full[stage], 0));
            __syncwarp();
            if (++stage == NSTAGE)
            {
                stage = 0;
                ph ^= 1;
            }
        }
    }
    else if (warp == kMmaWarp)
    {
        int stage = 0;
        uint32_t ph = 0, aph = 0, hph = 0; // aph / hph bit t: phase of a_ready[t] / h_free[t]
        int nheads = 0;                    // super-tiles whose heads were issued
        const uint32_t r_base = tc::smem_u32(ring), hb_base = tc::smem_u32(hb);
        auto wait_ready = [&](int t) {
            MBAR_WAIT_PLAIN(&a_ready[t], (aph >> t) & 1);
            aph ^= 1u << t;
        };
        // heads of tile t, whose layer 7 ran at step m7 (its converted output is A)
        auto heads = [&](int t, int m7) {
            wait_ready(t); // layer 7 of this tile converted
            if (nheads > 0)
            {
                MBAR_WAIT_PLAIN(&h_free[t], (hph >> t) & 1); // this tile's previous heads were read out
                hph ^= 1u << t;
            }
            tc::tc_fence_after();
            if (tc::elect_one())
            {
                issue_heads<SPLIT>(tmem + HEAD_COL + NHEAD_N * t, hb_base, tmem + (m7 % 3) * WPC);
                tc::mma2_commit(&acc_h[t], 3);
            }
            __syncwarp();
            if (t == 1)
                nheads++;
        };
        int m = 0; // layer steps (tile = m & 1; layer 0 steps are the epilogue's alone)
        for (int it = 0; it < mine; it++)
        {
            m += 2; // layer 0 of X and Y
            for (int l = 1; l < NL; l++)
            {
                MBAR_WAIT_PLAIN(&w_full[stage], ph);
                const uint32_t b = r_base + stage * SLOT;
                for (int t = 0; t < 2; t++, m++)
                {
                    if (lane == 0)
                        stamp2(a, 0, m);
                    wait_ready(t); // this tile's layer l-1 converted (both CTAs)
                    tc::tc_fence_after();
                    if (lane == 0)
                        stamp2(a, 1, m);
                    if (tc::elect_one())
                    {
                        const uint32_t d = tmem + (m % 3) * WPC;
                        issue_layer<SPLIT>(d, b, tmem + ((m + 1) % 3) * WPC);
                        tc::mma2_commit(&acc[t], 3);
                        if (t == 1)
                            tc::mma2_commit(&w_empty[stage], 3);
                    }
                    __syncwarp();
                    if (lane == 0)
                        stamp2(a, 2, m);
                }
                if (++stage == NSTAGE)
                {
                    stage = 0;
                    ph ^= 1;
                }
            }
            heads(0, m - 2); // X7 ran at step m - 2
            heads(1, m - 1); // Y7 at step m - 1
        }
    }
    else
    {
        const int e = warp, et = threadIdx.x;
        const int q = e & 3;          // TMEM lane quarter = position within the tile (CTA)
        const int grp = e >> 2;       // column group: chunks grp and grp + 6 (< 10)
        const int c1 = grp + NGRP;
        const bool two = c1 < KSTEPS;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        uint32_t fph = 0, hph = 0, cph = 0; // acc[t] phases (bit t), acc_h[t] phases (bit t), c_full phase
        int cstage = 0;
        int cur_m = 0; // the step being converted (trace stamps of the hooks build)

        auto prefetch = [&](int it) {
            int g0, s0;
            super_origin(a, cluster + it * nclusters, g0, s0);
            float *dst = pbuf + (it & 1) * 2 * TS * PROW;
            for (int i = et; i < 2 * TS * PROW / 4; i += EPI_THREADS)
            {
                const int row = i / (PROW / 4), k = (i % (PROW / 4)) * 4; // row = tile * 4 + CTA position
                const int s = s0 + (row / TS) * 2 * TS + (int)rank * TS + row % TS;
                const bool ok = s < a.nb;
                tc::cp_async16(dst + row * PROW + k, a.pterm + (size_t)(ok ? s : 0) * PROW + k, ok);
            }
            tc::cp_async_commit();
        };
        auto operands_ready = [&]() {
            tc::cp_async_wait_all();
            tc::named_bar(1, EPI_THREADS);
        };
        // one 16-column chunk: v = [acc * 2^-e_l +] add (+ cterm) -> ReLU -> fp16 hi/lo -> TMEM (in place)
        auto convert = [&](uint32_t reg, int chunk, const float *add, const uint8_t *cblk, bool from_acc,
                           float unscale) {
            const int n0 = chunk * 16;
            uint32_t raw[16];
            if (from_acc)
                tc::tmem_ld16_issue(reg + n0, raw);
            float x[16];
            lds16(add + n0, x);
            if (cblk)
            {
                float cv[16];
                lds_cterm16(cblk, chunk, lane, cv);
#pragma unroll
                for (int i = 0; i < 8; i++)
                {
                    const float2 sum = __fadd2_rn(make_float2(x[2 * i], x[2 * i + 1]), make_float2(cv[2 * i], cv[2 * i + 1]));
                    x[2 * i] = sum.x;
                    x[2 * i + 1] = sum.y;
                }
            }
            float v[16];
            if (from_acc)
            {
                tc::tmem_ld_wait();
                if (e == 0 && lane == 0 && chunk == grp)
                    stamp2(a, 4, cur_m); // first chunk's accumulator in registers
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = __uint_as_float(raw[i]);
            }
            else
            {
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = 0.0f;
            }
            uint32_t o[16];
            relu_split16(v, x, unscale, o);
            tc::tmem_st16(reg + n0, o);
        };
        // heads readout (group-0 warps: one TMEM lane quarter each) of tile t of the
        // super-tile at (g0, s0); acc_h[t] already waited
        auto heads_out = [&](int t, int g0, int s0) {
            float v[16];
            tc::tmem_ld16(tmem + HEAD_COL + NHEAD_N * t + lane_off, v);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0)
                tc::mbar_arrive_remote_relaxed(tc::mapa(&h_free[t], 0));
            const int g = g0 + lane, s = s0 + t * 2 * TS + (int)rank * TS + q;
            if (g < a.n && s < a.nb)
            {
                SWR_DCHECK(s < a.cap_b && g < a.np, "mlp heads: residual index outside the work buffer");
                const size_t plane = (size_t)a.cap_b * a.np;
#pragma unroll
                for (int h = 0; h < NHEADS; h++)
                    a.res[h * plane + (size_t)s * a.np + g] = __fmaf_rn(v[h], a.unscale[8], shb[h]);
            }
        };
        auto wait_heads = [&](int t) {
            MBAR_WAIT_PLAIN(&acc_h[t], (hph >> t) & 1);
            hph ^= 1u << t;
            tc::tc_fence_after();
        };

        if (mine > 0)
        {
            prefetch(0);
            operands_ready();
            if (mine > 1)
                prefetch(1);
        }
        int m = 0;
        int pg0 = 0, ps0 = 0; // previous super-tile
        for (int it = 0; it < mine; it++)
        {
            int g0, s0;
            super_origin(a, cluster + it * nclusters, g0, s0);
            for (int l = 0; l < NL; l++)
            {
                const uint8_t *cblk = nullptr;
                if (has_xc(l))
                {
                    MBAR_WAIT_PLAIN(&c_full[cstage], cph);
                    cblk = cring + cstage * C_BLOCK;
                }
                for (int t = 0; t < 2; t++, m++)
                {
                    if (l == 0)
                    {
                        // layer 0 = ReLU(cterm + pterm), no UMMA. X0's region held the previous
                        // super-tile's Y6 (read by Y7, done: acc[Y] waited before Y7's conversion),
                        // Y0's held X7 (read by heads X); waiting for the previous super-tile's
                        // heads here also keeps a_ready at most one phase ahead of its waiter.
                        // Each tile has its own heads accumulator, so heads Y never waits
                        // for heads X's readout
                        if (it > 0)
                        {
                            wait_heads(t);
                        }
                    }
                    else
                    {
                        // the previous super-tile's heads of this tile, read out while the
                        // tensor core runs this tile's layer 1 (the group-0 warps would
                        // otherwise wait here anyway): off the path from layer 7 to the next
                        // layer 1 (~1,600 cycles per boundary measured in that position)
                        if (l == 1 && it > 0 && grp == 0)
                            heads_out(t, pg0, ps0);
                        MBAR_WAIT_PLAIN(&acc[t], (fph >> t) & 1);
                        fph ^= 1u << t;
                        tc::tc_fence_after();
                    }
                    if (e == 0 && lane == 0)
                        stamp2(a, 3, m);
                    const uint32_t reg = tmem + (m % 3) * WPC + lane_off;
                    const float *prow = pbuf + ((it & 1) * 2 + t) * TS * PROW + q * PROW;
                    const float *add = has_xc(l) ? prow + (l / 2) * WPC : sbias + l * WPC; // warp-uniform
                    const float us = a.unscale[l]; // warp-uniform (layer 0: acc is not read)
                    cur_m = m;
                    convert(reg, grp, add, cblk, l > 0, us);
                    if (two)
                        convert(reg, c1, add, cblk, l > 0, us);
                    tc::tmem_st_wait();
                    if (lane == 0 && (e == 0 || e == EPI_WARPS - 1))
                        stamp2(a, e == 0 ? 5 : 6, m); // this warp's conversion stored
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        tc::mbar_arrive_remote_relaxed(tc::mapa(&a_ready[t], 0));
                }
                if (has_xc(l))
                {
                    // both tiles have read this cterm block
                    if (lane == 0)
                        tc::mbar_arrive(&c_empty[cstage]);
                    if (++cstage == NCSTAGE)
                    {
                        cstage = 0;
                        cph ^= 1;
                    }
                }
                if (l == 3 && it + 1 < mine)
                    operands_ready(); // next super-tile's pterm rows (prefetched a super-tile ahead)
            }
            pg0 = g0;
            ps0 = s0;
            // this super-tile's pterm buffer is free (all its conversions are done)
            if (it + 2 < mine)
                prefetch(it + 2);
        }
        if (mine > 0)
            for (int t = 0; t < 2; t++)
            {
                wait_heads(t);
                if (grp == 0)
                    heads_out(t, pg0, ps0);
            }
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == kMmaWarp)
    {
        tc::tc_fence_after();
        tc::tmem_dealloc2<512>(tmem);
    }
}

// fp16 bits of x, round to nearest even (host; subnormals and overflow as IEEE)
uint16_t f16_bits(float x) { return __half_as_ushort(__float2half_rn(x)); }
float f16_float(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// power-of-two exponent e with max_abs * 2^e in [2^13, 2^14) (0 for an all-zero block)
int scale_exp(float max_abs)
{
    if (!(max_abs > 0.0f) || !std::isfinite(max_abs))
        return 0;
    int e2 = 0;
    std::frexp(max_abs, &e2); // max_abs = m 2^e2, m in [0.5, 1)
    return 14 - e2;
}

// w * 2^e split into fp16 hi + lo (both stored at the UMMA K-major slot idx)
void put_split(uint16_t *hi, uint16_t *lo, size_t idx, float w, float scale)
{
    const float ws = w * scale; // exact (power of two)
    const uint16_t hb = f16_bits(ws);
    hi[idx] = hb;
    lo[idx] = f16_bits(ws - f16_float(hb));
}
} // namespace

// cterm blocks from the per-Gaussian centre terms cg [np][4][160] (W_c xc of
// layers 0,2,4,6, FP32, center_terms_kernel): block b, layer j, column group
// n / 4, row = Gaussian % 32 -> the tcgen05.cp source layout (zero rows past np).
// All four are added by the epilogue and carry the activation scale 2^k (exact).
__global__ void cterm_pack_kernel(const float *__restrict__ cg, float *__restrict__ ct, int np, int nblk, float s0,
                                  float s2, float s4, float s6)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nblk * TG * 4 * WPC)
        return;
    const int n = (int)(idx % WPC), j = (int)((idx / WPC) % 4);
    const int g = (int)(idx / (4 * WPC));
    const int blk = g / TG, row = g % TG;
    const size_t dst = ((size_t)blk * 4 + j) * (C_BLOCK / 4) + ((size_t)(n / 4) * TG + row) * 4 + n % 4;
    const float sc = j == 0 ? s0 : (j == 1 ? s2 : (j == 2 ? s4 : s6));
    ct[dst] = g < np ? cg[((size_t)g * 4 + j) * WPC + n] * sc : 0.0f;
}

bool mlp_tc_available() { return true; }

// Packed weights: per layer l = 1..7, pair rank 0 then 1 (each its 80 of the 160
// output columns), 10 K steps x (hi, lo) fp16 of w * 2^e_l in UMMA K-major
// core-matrix order: element (n_local, kk) of a K step at
// ((kk/8)*(80/8) + n_local/8)*64 + (n_local%8)*8 + kk%8. Also the heads' B
// operand (scale 2^e_h) and the cterm blocks.
void prepare_tc2_weights(Ctx &c, const std::vector<float> &whT, const std::vector<float> &heads,
                         const std::vector<float> &bias)
{
    const int WP = c.net.wp;
    constexpr int NC = WPC / 2;
    // per-layer scales from the largest |w| of the layer (zero padding included: harmless)
    for (int l = 1; l < NL; l++)
    {
        float m = 0.0f;
        for (size_t i = 0; i < (size_t)WP * WP; i++)
            m = std::max(m, std::fabs(whT[(size_t)(l - 1) * WP * WP + i]));
        c.net.tc_exp[l] = scale_exp(m);
    }
    {
        float m = 0.0f;
        for (int h = 0; h < NHEADS; h++)
            for (int k = 0; k < WP; k++)
                m = std::max(m, std::fabs(heads[(size_t)h * WP + k]));
        c.net.tc_exp[8] = scale_exp(m);
    }
    c.net.tc_exp[0] = 0;
    std::vector<uint16_t> packed((size_t)7 * 2 * W_BYTES / 2);
    size_t at = 0;
    for (int l = 1; l < NL; l++)
    {
        const float sc = std::ldexp(1.0f, c.net.tc_exp[l]);
        for (int rk = 0; rk < 2; rk++)
            for (int k = 0; k < KSTEPS; k++)
            {
                uint16_t *hi = packed.data() + at, *lo = hi + NC * 16;
                for (int nl = 0; nl < NC; nl++)
                    for (int kk = 0; kk < 16; kk++)
                    {
                        const float w = whT[((size_t)(l - 1) * WP + (k * 16 + kk)) * WP + rk * NC + nl];
                        put_split(hi, lo, (size_t)((kk / 8) * (NC / 8) + nl / 8) * 64 + (nl % 8) * 8 + kk % 8, w, sc);
                    }
                at += 2 * NC * 16;
            }
    }
    // heads B operand: per rank its NHEAD_N / 2 of the UMMA columns (heads 0-4 real, all in rank 0's)
    constexpr int HN = NHEAD_N / 2;
    const float hsc = std::ldexp(1.0f, c.net.tc_exp[8]);
    std::vector<uint16_t> hpk((size_t)2 * HB_BYTES / 2, 0);
    for (int rk = 0; rk < 2; rk++)
        for (int k = 0; k < KSTEPS; k++)
        {
            uint16_t *hi = hpk.data() + ((size_t)rk * KSTEPS + k) * 2 * HN * 16, *lo = hi + HN * 16;
            for (int nl = 0; nl < HN; nl++)
                for (int kk = 0; kk < 16; kk++)
                {
                    const int h = rk * HN + nl;
                    const float w = h < NHEADS ? heads[(size_t)h * WP + k * 16 + kk] : 0.0f;
                    put_split(hi, lo, (size_t)((kk / 8) * (HN / 8) + nl / 8) * 64 + (nl % 8) * 8 + kk % 8, w, hsc);
                }
        }
    void *dh = nullptr;
    check_cuda(cudaMalloc(&dh, hpk.size() * 2), "cudaMalloc tc2 heads");
    c.allocs.push_back(dh);
    check_cuda(cudaMemcpy(dh, hpk.data(), hpk.size() * 2, cudaMemcpyHostToDevice), "upload tc2 heads");
    c.net.wh_tc2 = static_cast<uint16_t *>(dh);
    void *d = nullptr;
    check_cuda(cudaMalloc(&d, packed.size() * 2), "cudaMalloc tc2 weights");
    c.allocs.push_back(d);
    check_cuda(cudaMemcpy(d, packed.data(), packed.size() * 2, cudaMemcpyHostToDevice), "upload tc2 weights");
    c.net.w_tc2 = static_cast<uint16_t *>(d);

    const int nblk = (c.g.n + TG - 1) / TG;
    const size_t total = (size_t)nblk * TG * 4 * WPC;
    check_cuda(cudaMalloc(&d, total * sizeof(float)), "cudaMalloc cterm blocks");
    c.allocs.push_back(d);
    c.net.c_tc = static_cast<float *>(d);
    const int *k = c.net.tc_ascale;
    cterm_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c.stream>>>(
        c.net.cg, c.net.c_tc, c.g.np, nblk, std::ldexp(1.0f, k[0]), std::ldexp(1.0f, k[2]), std::ldexp(1.0f, k[4]),
        std::ldexp(1.0f, k[6]));
    std::vector<float> bs(bias.size());
    for (size_t i = 0; i < bias.size(); i++)
        bs[i] = std::ldexp(bias[i], k[i / WP]);
    c.net.bias_tc = upload(c, bs);
    check_cuda(cudaStreamSynchronize(c.stream), "cterm blocks");
}

static long long *g_trace2 = nullptr;
int mlp_tc2_trace(long long *out)
{
    if (!g_trace2)
        return 1;
    cudaDeviceSynchronize();
    return cudaMemcpy(out, g_trace2, 8 * 48 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}

void launch_mlp_tc2(Ctx &c, int nb, cudaStream_t st)
{
    static DeviceOnce once;
    const int max_clusters = once.get(c.device, [] {
        for (auto k : {mlp_tc2_kernel<true>, mlp_tc2_kernel<false>})
        {
            check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
                       "tc2 mlp smem attribute"); // SMEM_BYTES + the optional pad (mlp_smem_pad)
            check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            (int)cudaSharedmemCarveoutMaxShared),
                       "tc2 mlp carveout");
        }
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2, 1, 1);
        cfg.blockDim = dim3(THREADS, 1, 1);
        cfg.dynamicSmemBytes = SMEM_BYTES;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int mc = 0;
        check_cuda(cudaOccupancyMaxActiveClusters(&mc, mlp_tc2_kernel<true>, &cfg), "tc2 mlp cluster occupancy");
        if (mc < 1)
            check_cuda(cudaErrorLaunchOutOfResources, "tc2 mlp: no CTA pair fits on this device");
        return mc;
    });
    Tc2Args a;
    a.w = c.net.w_tc2;
    a.cterm = c.net.c_tc;
    a.bias = c.net.bias_tc;
    a.pterm = c.w.pterm;
    a.wh = c.net.wh_tc2;
    a.hbias = c.net.hbias;
    a.res = c.w.res;
    a.n = c.g.n;
    a.np = c.g.np;
    a.nb = nb;
    a.cap_b = (int)c.w.cap_b;
    a.n_sblk = (nb + SUPER_S - 1) / SUPER_S;
    a.ntiles = ((c.g.n + TG - 1) / TG) * a.n_sblk;
    // layer l's accumulator holds 2^(e_l + k_(l-1)) W h; its output carries 2^k_l
    const int *k = c.net.tc_ascale;
    a.unscale[0] = 1.0f;
    for (int l = 1; l < 8; l++)
        a.unscale[l] = std::ldexp(1.0f, k[l] - c.net.tc_exp[l] - k[l - 1]);
    a.unscale[8] = std::ldexp(1.0f, -(c.net.tc_exp[8] + k[7])); // heads: back to true residuals
    a.trace = nullptr;
    if (kHooks && getenv("SWR_TC_DEBUG"))
    {
        static long long *buf = nullptr;
        if (!buf)
            check_cuda(cudaMalloc(&buf, 8 * 48 * sizeof(long long)), "trace buffer");
        cudaMemsetAsync(buf, 0, 8 * 48 * sizeof(long long), st);
        a.trace = buf;
        g_trace2 = buf;
    }
    const int cap = c.mlp_max_clusters > 0 ? std::min(c.mlp_max_clusters, max_clusters) : max_clusters;
    const int grid = 2 * std::min(cap, a.ntiles);
    if (grid == 0)
        return;
    const int smem = std::min(SMEM_BYTES + std::max(c.mlp_smem_pad, 0), 227 * 1024);
    if (c.mlp_precision == 1)
        mlp_tc2_kernel<true><<<grid, THREADS, smem, st>>>(a);
    else
        mlp_tc2_kernel<false><<<grid, THREADS, smem, st>>>(a);
    c.launches++;
}

} // namespace swr
