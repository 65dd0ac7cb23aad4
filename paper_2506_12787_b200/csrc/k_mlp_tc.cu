// Deformation MLP on the 5th-generation tensor cores (tcgen05), split precision,
// CTA pairs (cta_group::2).
//
// Function: deform::predict_residuals (/root/reference/proj/src/deform.cpp:140-207).
// Row (g, s) of the reference's input matrix is x = [xc[g] | xp[s]], the
// sinusoidal encodings of Gaussian g's materialised centre (42 values) and of
// TX position s (39 values) (deform.cpp:54-70, 158-171). Trunk layers 0, 2, 4, 6
// read x (layer 0 alone, 2/4/6 after the hidden state, deform.cpp:41,177-192).
// Here W x is split into W_c xc[g] + (W_p xp[s] + b):
//   * W_c xc[g] depends on the Gaussian only: it is computed once per scene in
//     FP32 (center_terms_kernel, k_mlp.cu) and stored per 32-Gaussian block in
//     the tcgen05.cp source layout ("cterm"). Each layer 0/2/4/6 accumulator
//     STARTS from it: the issuer copies the block into TMEM with
//     tcgen05.cp.32x128b.warpx4 (one 32-row copy broadcast to the 4 lane
//     quarters = the 4 positions of the CTA), and the layer's UMMAs accumulate on
//     top (cp and mma from one thread execute in issue order). Layer 0 thus needs
//     no UMMA at all, and layers 2/4/6 only their 10 hidden K steps;
//   * W_p xp[s] + b ("pterm", computed per position by pos_prep_kernel) is added in
//     the epilogue; a CTA's 128 rows are 32 Gaussians x 4 positions with the TMEM
//     lane quarter = the position, so this addend is warp-uniform.
// The five heads (deform.cpp:194-206) run on the tensor cores too, as a ninth
// MMA layer (N = 32, heads 0-4 real) reading layer 7's converted output.
// All products use bf16 hi/lo splits with FP32 accumulation in TMEM:
//   a.w ~= a_hi.w_hi + a_lo.w_hi + a_hi.w_lo        ("bf16x3", 3 UMMAs per K step)
// (~16 significant bits per product; residuals within ~2e-5 relative of the FP64
// oracle). SWR_MLP_BF16 issues only a_hi.w_hi.
//
// Why CTA pairs: every tile streams all weights (hi + lo, ~0.8 MB) through
// shared memory; with one CTA per tile the TMA writes plus the tensor core's B
// reads nearly saturate the 128 B/clk shared-memory port. A cluster of 2 CTAs
// runs M = 256 UMMAs: each CTA holds its own 128 rows (A) and HALF of every B
// tile, so per-SM weight traffic halves while each SM still computes 128 rows.
//
// Structure (one persistent 2-CTA cluster per TPC, 22 warps per CTA):
//   warps 0-19  epilogue (both CTAs): 5 column groups x 4 TMEM lane quarters. Layer
//               l's FP32 accumulator is converted IN PLACE into layer l+1's bf16
//               hi/lo A operand (tcgen05.ld -> + bias / pterm -> ReLU -> split ->
//               tcgen05.st), then the warp arrives on the leader's barrier;
//   warp 20     producer (both CTAs): streams this CTA's half of each weight stage
//               from L2 into a shared-memory ring (cp.async.bulk, complete_tx);
//   warp 21     leader CTA: UMMA issuer (converged warp, one elected lane) --
//               tcgen05.mma.cta_group::2 M=256, K=16, two output parts N = 96, 64
//               committed separately; peer CTA: relays "my half of stage s
//               landed" to the leader (remote mbarrier arrive).
// Output parts 0/1 (columns 0-95, 96-159) are exactly the next layer's K steps
// 0-5 and 6-9: the epilogue converts part 0 while the tensor core runs part 1,
// and the next layer's first 6 K steps run while part 1 is converted.
// TMEM: three 160-column regions used round-robin (accumulator / A operand of the
// next layer / free) plus 32 columns for the heads accumulator.
// Issue-loop lessons (measured): descriptors must be compile-time offsets from
// one base (a runtime K loop halves UMMA throughput); remote arrivals on the
// critical path are .relaxed (a .release.cluster arrive costs a MEMBAR.GPU).
#include "swr_internal.h"
#include "tc_ptx.cuh"

#include <cstdio>
#ifdef SWR_TC_DEBUG_WAITS
#define MBAR_WAIT(b, p, tag) tc::mbar_wait_dbg(b, p, tag)
#define MBAR_WAIT_CL(b, p, tag) tc::mbar_wait_cluster_dbg(b, p, tag)
#else
#define MBAR_WAIT(b, p, tag) tc::mbar_wait(b, p)
#define MBAR_WAIT_CL(b, p, tag) tc::mbar_wait(b, p)
#endif

#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

namespace swr
{

namespace
{
constexpr int TM = 128;                 // rows per CTA: 32 Gaussians x 4 positions
constexpr int TG = 32, TS = 4;
constexpr int PAIR_S = 2 * TS;          // positions per pair tile
constexpr int WPC = 160;                // padded width (N and K of the hidden layers)
constexpr int KSTEPS = WPC / 16;        // 10 UMMA K steps per hidden layer
constexpr int NPART = 2;
constexpr int NL = 8;                   // trunk layers per tile: 0 (cterm copy only), 1..7; then the heads
constexpr int NHEAD_N = 32;             // heads UMMA N (5 real columns)
// output part p: N = npart(p) columns from pcol(p) (N multiple of 32 for cta_group::2
// with A in TMEM); feeds the next layer's K steps pcol/16 .. Each part's conversion
// (epilogue) overlaps the UMMAs of the later part and of the next layer's K steps
// that do not read it. Finer parts (64/32/32/32 was tried) spread the epilogue's
// issue pressure over the whole layer, and the single-thread UMMA issuer, which
// shares its SM sub-partition with 6 epilogue warps, then falls behind the tensor
// pipe (tools/umma_parts_bench.cu: the pipe alone runs every split at N/2 clk per
// UMMA; with busy neighbour warps the issue rate collapses): 96/64 measured best.
__host__ __device__ constexpr int npart(int p) { return p == 0 ? 96 : 64; }
__host__ __device__ constexpr int pcol(int p) { return p == 0 ? 0 : 96; }
__host__ __device__ constexpr int part_of_chunk(int c) { return c < 6 ? 0 : 1; }
// one operand (hi or lo), one K step, this CTA's half of N output columns
__host__ __device__ constexpr int kstep_bytes_n(int n) { return n / 2 * 16 * 2; }
__host__ __device__ constexpr int kstep_bytes(int p) { return kstep_bytes_n(npart(p)); }
// cterm segment of output part p: npart(p) / 4 groups of [32 rows][4 f32] (one
// tcgen05.cp.32x128b each), full N (both CTAs of a pair hold the same Gaussians)
__host__ __device__ constexpr int cseg_bytes(int p) { return npart(p) * TG * 4; }
// cterm block layout: [160 / 4 column groups][32 rows][4] f32, so part p's segment
// starts at byte pcol(p) * TG * 4
__host__ __device__ constexpr int cseg_off(int p) { return pcol(p) * TG * 4; }
constexpr int C_BLOCK = WPC * TG * 4;   // one layer's cterm of a 32-Gaussian block: 20 KB
constexpr int W_MAX = KSTEPS * 2 * kstep_bytes(0); // largest weight stage: 10 K steps x (hi, lo) = 30 KB
constexpr int SLOT = W_MAX + cseg_bytes(0);        // + the cterm segment at W_MAX: 42 KB
#ifndef SWR_TC_NSTAGE
#define SWR_TC_NSTAGE 3
#endif
constexpr int NSTAGE = SWR_TC_NSTAGE;
#ifndef SWR_TC_GROUPS
#define SWR_TC_GROUPS 6
#endif
constexpr int NGRP = SWR_TC_GROUPS;     // epilogue column groups (5 or 6)
constexpr int EPI_WARPS = 4 * NGRP;     // column groups x 4 TMEM lane quarters
constexpr int EPI_THREADS = 32 * EPI_WARPS;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int NREG = 3;                 // TMEM regions of 160 columns
constexpr int HEAD_COL = NREG * WPC;    // heads accumulator: TMEM columns 480-511
// The warp scheduler prefers higher warp ids: the producer and the MMA issuer
// sit above the epilogue warps.
constexpr int kProducerWarp = EPI_WARPS, kMmaWarp = EPI_WARPS + 1;
constexpr int PROW = 4 * WPC;           // pterm row of one position (4 layers)
constexpr int SMEM_RING = NSTAGE * SLOT;
constexpr int SMEM_P = 2 * TS * PROW * 4;
constexpr int SMEM_CONST = (8 * WPC + 8) * 4;
// w_full[NSTAGE], w_empty[NSTAGE], a_ready[2 sets][2 parts], acc[2 sets][2 parts],
// acc_h
constexpr int NBARS = 2 * NSTAGE + 2 * NPART + 2 * NPART + 1;
constexpr int SMEM_BYTES = SMEM_RING + SMEM_P + SMEM_CONST + NBARS * 8 + 16 + 1024;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
static_assert(NPART == 2 && pcol(NPART - 1) + npart(NPART - 1) == WPC, "output parts cover the width");
// epilogue column group g converts 16-column chunks g and g + NGRP (if < 10), in
// that order (= part order). With 6 groups: part 0 (chunks 0-5) one chunk per
// group, part 1 (chunks 6-9) by groups 0-3. part_warps(p): warps (x 4 lane quarters) that report part p, one
// arrival per warp and part.
__host__ __device__ constexpr int part_warps(int p)
{
    int w = 0;
    for (int g = 0; g < NGRP; g++)
        w += (part_of_chunk(g) == p || (g + NGRP < KSTEPS && part_of_chunk(g + NGRP) == p)) ? 4 : 0;
    return w;
}

// layers whose input includes the centre encoding (deform.cpp:41: layer 0 and the
// skip layers 2, 4, 6): their accumulator starts from the cterm
__host__ __device__ constexpr bool has_xc(int l) { return l == 0 || l == 2 || l == 4 || l == 6; }
// weight stream per tile: one stage per (trunk layer, part): the 10 hidden K steps
// (layers 1..7; layer 0 has none), each K step hi then lo, rank 0's half of the
// part's columns then rank 1's; finally the heads stage. A stage of a layer with
// a cterm also receives the tile's cterm segment (at W_MAX, both CTAs in full).
__host__ __device__ constexpr int stage_bytes(int l, int p)
{
    return (l >= 1 ? KSTEPS : 0) * 2 * kstep_bytes(p);
}
constexpr int HEAD_STAGE = KSTEPS * 2 * (NHEAD_N / 2) * 16 * 2; // 10 KB per CTA
// byte offset of stage (l, p) (l = NL: the heads) in the packed stream, both ranks
__host__ __device__ constexpr size_t stream_offset(int l, int p)
{
    size_t off = 0;
    for (int j = 0; j < l * NPART + (l < NL ? p : 0); j++)
        off += 2 * (size_t)stage_bytes(j / NPART, j % NPART);
    return off;
}

struct TcArgs
{
    const uint16_t *w_tc;  // packed weights in consumption order (prepare_tc_weights)
    const float *cterm;    // [n/32 blocks][4 layers][part 0 | part 1][npart/4][32 rows][4] f32 (W_c xc, no bias)
    const float *bias;     // [8][160]
    const float *pterm;    // [nb][4][160] position term of layers 0,2,4,6 (bias included)
    const float *hbias;    // [5]
    float *res;            // [5][cap_b][np]
    int n, np, nb, cap_b, n_sblk, ntiles, split, debug;
    long long *trace;      // debug: [3 tiles][9 layers][128 slots] clock64 stamps of block 0
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi)
{
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi); // .x -> low 16 bits
    return *reinterpret_cast<uint32_t *>(&h);
}

// 16 consecutive K elements -> 8 columns of hi pairs, then 8 columns of lo pairs.
// v = ReLU(acc + add): packed f32x2 arithmetic (FADD2/FFMA2) halves the FP
// instruction count of the conversion.
__device__ __forceinline__ void relu_split16(const float (&acc)[16], const float (&add)[16], uint32_t (&o)[16])
{
#pragma unroll
    for (int i = 0; i < 8; i++)
    {
        float2 v = __fadd2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), make_float2(add[2 * i], add[2 * i + 1]));
        v.x = fmaxf(v.x, 0.0f);
        v.y = fmaxf(v.y, 0.0f);
        const uint32_t h = pack_bf16(v.x, v.y);
        const float2 hf = make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u));
        const float2 lo = __ffma2_rn(hf, make_float2(-1.0f, -1.0f), v);
        o[i] = h;
        o[8 + i] = pack_bf16(lo.x, lo.y);
    }
}

// 16 floats from shared memory (explicit ld.shared; generic loads would be slower)
__device__ __forceinline__ void lds16(const float *p, float (&v)[16])
{
    const uint32_t a = tc::smem_u32(p);
#pragma unroll
    for (int i = 0; i < 4; i++)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[4 * i]), "=f"(v[4 * i + 1]), "=f"(v[4 * i + 2]), "=f"(v[4 * i + 3])
                     : "r"(a + 16 * i));
}

// pair tile `tile` (32 Gaussians x 8 positions) -> this CTA's Gaussian and position origin
__device__ __forceinline__ void tile_origin(const TcArgs &a, int tile, uint32_t rank, int &g0, int &s0)
{
    g0 = (tile / a.n_sblk) * TG;
    s0 = (tile % a.n_sblk) * PAIR_S + (int)rank * TS;
}

// cp.async the CTA's 4 pterm rows (zero-filled outside the problem); issued by
// all epilogue threads
__device__ __forceinline__ void prefetch_tile(const TcArgs &a, int tile, uint32_t rank, float *p_buf, int et)
{
    int g0, s0;
    tile_origin(a, tile, rank, g0, s0);
    for (int i = et; i < TS * PROW / 4; i += EPI_THREADS)
    {
        const int sl = i / (PROW / 4), k = (i % (PROW / 4)) * 4;
        const int s = s0 + sl;
        const bool ok = s < a.nb;
        tc::cp_async16(p_buf + sl * PROW + k, a.pterm + (size_t)(ok ? s : 0) * PROW + k, ok);
    }
    tc::cp_async_commit();
}

// Debug hooks (SWR_TC_DEBUG bits: 1 stale weights, 2 skip the conversion math, 8
// clock64 trace) exist only in builds with -DSWR_TC_DEBUG_HOOKS (tools/
// build_variant.py): every instruction they add to the epilogue lengthens the
// conversion chain between layers.
#ifdef SWR_TC_DEBUG_HOOKS
constexpr bool kHooks = true;
#else
constexpr bool kHooks = false;
#endif
__device__ __forceinline__ void stamp(const TcArgs &a, int it, int l, int slot)
{
    if (kHooks && a.trace && blockIdx.x == 0 && it < 3)
        a.trace[(it * 9 + l) * 128 + slot] = clock64();
}

// UMMA issue (one elected thread), descriptors compile-time offsets from one base.
// cterm of an N-column output part: N / 4 copies of [32 rows][4 f32] from the
// stage's cterm segment into the accumulator columns, each broadcast to the 4
// TMEM lane quarters (the 4 positions); both CTAs copy from their own segment
template <int N>
__device__ __forceinline__ void issue_cterm(uint32_t d, uint32_t cseg)
{
    constexpr uint32_t DH = tc::desc_hi(128); // 8-row groups of 16 B rows: 128 B apart (contiguous)
    const uint32_t c0 = tc::desc_lo(cseg, 16);
#pragma unroll
    for (int g = 0; g < N / 4; g++)
        tc::cp2_32x128b_x4(d + 4 * g, tc::desc_of(c0 + (g * TG * 16 >> 4), DH));
}
// hidden K steps [K0, K0 + NK) of an N-column output: A = previous layer's
// converted output in TMEM
template <int N, int K0, int NK, bool SPLIT>
__device__ __forceinline__ void issue_hidden(uint32_t d, uint32_t bh, uint32_t areg, bool first)
{
    constexpr uint32_t KB = kstep_bytes_n(N), LBO = N / 2 / 8 * 128;
    constexpr uint32_t IDESC = tc::make_idesc(1, 2 * TM, N);
    constexpr uint32_t DH = tc::desc_hi(128);
    const uint32_t b0 = tc::desc_lo(bh, LBO);
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
    {
        const int k = K0 + kk;
        const uint64_t dbh = tc::desc_of(b0 + (k * 2 * KB >> 4), DH);
        const uint32_t ahi = areg + 16 * k;
        tc::mma2_f16_ts(d, ahi, dbh, IDESC, (kk == 0 && first) ? 0u : 1u);
        if (SPLIT)
        {
            tc::mma2_f16_ts(d, ahi + 8, dbh, IDESC, 1u);
            tc::mma2_f16_ts(d, ahi, tc::desc_of(b0 + ((k * 2 + 1) * KB >> 4), DH), IDESC, 1u);
        }
    }
}
// hidden K steps fed by input part J (= the previous layer's output part J),
// after waiting for its conversion (WAITS)
template <int N, int J, bool WAITS, bool SPLIT>
__device__ __forceinline__ void mma_from_part(uint32_t d, uint32_t bh, uint32_t areg, bool first, uint64_t *ready,
                                              uint32_t ready_ph)
{
    if (WAITS)
    {
        MBAR_WAIT_CL(&ready[J], (ready_ph >> J) & 1, 101 + J);
        tc::tc_fence_after();
    }
    if (tc::elect_one())
        issue_hidden<N, pcol(J) / 16, npart(J) / 16, SPLIT>(d, bh, areg, J == 0 && first);
    __syncwarp();
    if constexpr (J + 1 < NPART)
        mma_from_part<N, J + 1, WAITS, SPLIT>(d, bh, areg, first, ready, ready_ph);
}
// the 10 hidden K steps of one output (whole warp); WAITS: wait for each converted
// part of the previous layer before the K steps that read it
template <int N, bool WAITS, bool SPLIT>
__device__ __forceinline__ void mma_hidden(uint32_t d, uint32_t bh, uint32_t areg, bool first, uint64_t *ready,
                                           uint32_t ready_ph)
{
    mma_from_part<N, 0, WAITS, SPLIT>(d, bh, areg, first, ready, ready_ph);
}
// output part P of trunk layer l from one stage at b: the cterm copy (layers
// 0/2/4/6), then the hidden UMMAs (layers 1..7) accumulating on top of it
template <int P, bool SPLIT>
__device__ __forceinline__ void mma_part(int l, uint32_t d, uint32_t areg, uint32_t b, uint64_t *ready,
                                         uint32_t ready_ph)
{
    const bool xc = has_xc(l);
    if (xc)
    {
        if (tc::elect_one())
            issue_cterm<npart(P)>(d, b + W_MAX);
        __syncwarp();
    }
    if (l >= 1)
        mma_hidden<npart(P), P == 0, SPLIT>(d, b, areg, !xc, ready, ready_ph);
}

template <bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) mlp_tc_kernel(TcArgs a)
{
    extern __shared__ uint8_t smem_raw[];
    // identical offsets in both CTAs (UMMA descriptors of the pair address both)
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ring = smem;
    float *pbuf = reinterpret_cast<float *>(ring + SMEM_RING);         // [2][4][4][160]
    float *sbias = pbuf + 2 * TS * PROW;                               // [8][160]
    float *shb = sbias + 8 * WPC;                                      // [8]
    uint64_t *bars = reinterpret_cast<uint64_t *>(shb + 8);
    uint64_t *w_full = bars, *w_empty = bars + NSTAGE; // w_full (leader) also counts the peer's relay
    uint64_t *a_ready = bars + 2 * NSTAGE; // [set][part] (leader): a converted output part, both CTAs
    uint64_t *acc = a_ready + 2 * NPART;   // [set][part]: a layer's accumulator part complete (commit multicast)
    uint64_t *acc_h = acc + 2 * NPART;     // heads accumulator complete
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
        for (int k = 0; k < 2 * NPART; k++)
        {
            tc::mbar_init(&a_ready[k], 2 * part_warps(k % NPART));
            tc::mbar_init(&acc[k], 1);
        }
        tc::mbar_init(acc_h, 1);
        tc::fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 8 * WPC; i += THREADS)
        sbias[i] = a.bias[i];
    if (threadIdx.x < 5)
        shb[threadIdx.x] = a.hbias[threadIdx.x];
    if (warp == kMmaWarp)
        tc::tmem_alloc2<512>(tmem_slot);
    tc::tc_fence_before();
    tc::cluster_sync(); // barriers of both CTAs initialised before any remote arrival
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int ntiles_mine = cluster < a.ntiles ? (a.ntiles - 1 - cluster) / nclusters + 1 : 0;

    // Issue order (= weight-stream order = conversion order): layer 0 of the first
    // tile, then per tile layers 1..7, layer 0 of the NEXT tile (a cterm copy that
    // needs nothing from this tile), then the heads.
    auto stage_count = [&](int it) { return NL * NPART - (it + 1 < ntiles_mine ? 0 : NPART) + 1; };
    if (warp == kProducerWarp)
    {
        // whole warp converged; one elected lane issues; this CTA copies its half
        // of every stage
        int stage = 0;
        uint32_t ph = 0;
        auto load = [&](int l, int p, int it) {
            const uint32_t bytes = l < NL ? stage_bytes(l, p) : HEAD_STAGE;
            const uint32_t cbytes = l < NL && has_xc(l) ? cseg_bytes(p) : 0;
            const size_t off = stream_offset(l, p);
            MBAR_WAIT(&w_empty[stage], ph ^ 1, 1);
            if (tc::elect_one())
            {
                if (kHooks && (a.debug & 1) && it > 0)
                    tc::mbar_arrive(&w_full[stage]); // debug: stale weights, no TMA traffic
                else
                {
                    tc::mbar_arrive_expect_tx(&w_full[stage], bytes + cbytes);
                    if (bytes)
                        tc::bulk_g2s(ring + stage * SLOT,
                                     reinterpret_cast<const uint8_t *>(a.w_tc) + off + rank * bytes, bytes,
                                     &w_full[stage]);
                    if (cbytes)
                    {
                        int g0, s0;
                        tile_origin(a, cluster + it * nclusters, rank, g0, s0);
                        const uint8_t *src = reinterpret_cast<const uint8_t *>(a.cterm) +
                                             ((size_t)(g0 / TG) * 4 + l / 2) * C_BLOCK + cseg_off(p);
                        tc::bulk_g2s(ring + stage * SLOT + W_MAX, src, cbytes, &w_full[stage]);
                    }
                }
            }
            __syncwarp();
            if (++stage == NSTAGE)
            {
                stage = 0;
                ph ^= 1;
            }
        };
        if (ntiles_mine > 0)
            for (int p = 0; p < NPART; p++)
                load(0, p, 0);
        for (int it = 0; it < ntiles_mine; it++)
        {
            for (int l = 1; l < NL; l++)
                for (int p = 0; p < NPART; p++)
                    load(l, p, it);
            if (it + 1 < ntiles_mine)
                for (int p = 0; p < NPART; p++)
                    load(0, p, it + 1);
            load(NL, 0, it);
        }
    }
    else if (warp == kMmaWarp && rank != 0)
    {
        // peer CTA: tell the leader when this CTA's half of each stage has landed
        int stage = 0;
        uint32_t ph = 0;
        const int total = ntiles_mine > 0 ? NPART + [&] {
            int t = 0;
            for (int it = 0; it < ntiles_mine; it++)
                t += stage_count(it);
            return t;
        }() : 0;
        for (int j = 0; j < total; j++)
        {
            MBAR_WAIT(&w_full[stage], ph, 4);
            if (tc::elect_one())
                tc::mbar_arrive_remote_relaxed(tc::mapa(&w_full[stage], 0)); // payload: completed TMA bytes
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
        // leader: whole warp converged (waits by all lanes), UMMAs and commits by
        // one elected lane: keeps the issue loop free of YIELD/divergence overhead
        int stage = 0;
        uint32_t ph = 0, aph = 0; // phase bits: aph bit set*NPART+part
        constexpr uint32_t PMASK = (1u << NPART) - 1;
        int ct = 0;                        // trunk layers issued: acc set = ct & 1
        int k = 0;                         // layers that read a converted layer: a_ready set = k & 1
        const uint32_t r_base = tc::smem_u32(ring);
        auto next_stage = [&]() {
            if (++stage == NSTAGE)
            {
                stage = 0;
                ph ^= 1;
            }
        };
        // trunk layer l of local tile it
        auto trunk = [&](int it, int l) {
            const int m = 8 * it + l; // TMEM region rotation
            const uint32_t dreg = tmem + (m % NREG) * WPC;
            const uint32_t areg = tmem + ((m + NREG - 1) % NREG) * WPC;
            const int ks = k & 1;
            const uint32_t rph = (aph >> (ks * NPART)) & PMASK;
#pragma unroll
            for (int p = 0; p < NPART; p++)
            {
                if (lane == 0)
                    stamp(a, it, l, 112 + p);
                MBAR_WAIT_CL(&w_full[stage], ph, 2);
                tc::tc_fence_after();
                if (lane == 0)
                    stamp(a, it, l, 116 + p);
                const uint32_t b = r_base + stage * SLOT;
                if (p == 0)
                    mma_part<0, SPLIT>(l, dreg, areg, b, &a_ready[ks * NPART], rph);
                else
                    mma_part<1, SPLIT>(l, dreg + pcol(1), areg, b, &a_ready[ks * NPART], rph);
                if (tc::elect_one())
                {
                    tc::mma2_commit(&w_empty[stage], 3);
                    tc::mma2_commit(&acc[(ct & 1) * NPART + p], 3);
                }
                __syncwarp();
                if (lane == 0)
                    stamp(a, it, l, 120 + p);
                next_stage();
            }
            ct++;
            if (l >= 1)
            {
                aph ^= PMASK << (ks * NPART);
                k++;
            }
        };
        if (ntiles_mine > 0)
            trunk(0, 0);
        for (int it = 0; it < ntiles_mine; it++)
        {
            for (int l = 1; l < NL; l++)
                trunk(it, l);
            if (it + 1 < ntiles_mine)
                trunk(it + 1, 0);
            // heads: A = layer 7's converted output, D = the heads columns
            const int ks = k & 1;
            if (lane == 0)
                stamp(a, it, NL, 112);
            MBAR_WAIT_CL(&w_full[stage], ph, 2);
            tc::tc_fence_after();
            mma_hidden<NHEAD_N, true, SPLIT>(tmem + HEAD_COL, r_base + stage * SLOT, tmem + ((8 * it + 7) % NREG) * WPC,
                                             true, &a_ready[ks * NPART], (aph >> (ks * NPART)) & PMASK);
            if (tc::elect_one())
            {
                tc::mma2_commit(&w_empty[stage], 3);
                tc::mma2_commit(acc_h, 3);
            }
            __syncwarp();
            if (lane == 0)
                stamp(a, it, NL, 120);
            next_stage();
            aph ^= PMASK << (ks * NPART);
            k++;
        }
    }
    else
    {
        const int e = warp;           // 0 .. EPI_WARPS - 1
        const int et = threadIdx.x;
        const int q = warp & 3;       // TMEM lane quarter = position of the tile
        const int grp = NGRP - 1 - (e >> 2); // column group: chunks grp (part 0) and grp + NGRP (if < 10)
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int c1 = grp + NGRP; // second chunk (none when >= 10)
        const int pc0 = part_of_chunk(grp), pc1 = c1 < KSTEPS ? part_of_chunk(c1) : -1;
        uint32_t fph = 0; // phase bits of acc[set][part] (this warp waits every completion of its parts)
        int ct = 0;       // trunk layers converted (= the issuer's trunk count): set = ct & 1

        // convert chunk `chunk` (16 columns, part p) of trunk layer (it, l) in place
        // and report it to the leader
        auto convert = [&](int it, int l, int chunk, int p, bool wait, bool arrive) {
            const int m = 8 * it + l;
            const uint32_t reg = tmem + (m % NREG) * WPC + lane_off;
            const float *prow = pbuf + (it & 1) * TS * PROW + q * PROW; // pterm row of this warp's position
            if (wait)
            {
                const int bit = (ct & 1) * NPART + p;
                MBAR_WAIT(&acc[bit], (fph >> bit) & 1, 10 + p);
                fph ^= 1u << bit;
                tc::tc_fence_after();
            }
            if (lane == 0) // debug trace: first chunk 16 + e / 40 + e, second 64 + e / 88 + e
                stamp(a, it, l, (chunk < NGRP ? 16 : 64) + e);
            if (!kHooks || !(a.debug & 2))
            {
                const float *add = has_xc(l) ? prow + (l / 2) * WPC : sbias + l * WPC; // warp-uniform addend
                const int n0 = chunk * 16;
                uint32_t raw[16];
                tc::tmem_ld16_issue(reg + n0, raw);
                float x[16];
                lds16(add + n0, x);
                tc::tmem_ld_wait();
                float v[16];
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = __uint_as_float(raw[i]);
                uint32_t o[16];
                relu_split16(v, x, o);
                tc::tmem_st16(reg + n0, o);
                tc::tmem_st_wait();
            }
            if (!arrive)
                return;
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0)
            {
                tc::mbar_arrive_remote_relaxed(tc::mapa(&a_ready[(ct & 1) * NPART + p], 0)); // read by the next consumer
                stamp(a, it, l, (chunk < NGRP ? 40 : 88) + e);
            }
        };
        auto convert_layer = [&](int it, int l) {
            convert(it, l, grp, pc0, true, pc1 != pc0);
            if (pc1 >= 0)
                convert(it, l, c1, pc1, pc1 != pc0, true);
            ct++;
        };
        // heads of local tile `it` (group 0 warps: one lane quarter each)
        auto heads = [&](int it) {
            if (grp != 0)
                return;
            MBAR_WAIT(acc_h, it & 1, 20);
            tc::tc_fence_after();
            float v[16];
            tc::tmem_ld16(tmem + HEAD_COL + lane_off, v);
            int g0, s0;
            tile_origin(a, cluster + it * nclusters, rank, g0, s0);
            const int g = g0 + lane, s = s0 + q;
            if (g < a.n && s < a.nb)
            {
                const size_t plane = (size_t)a.cap_b * a.np;
#pragma unroll
                for (int hh = 0; hh < 5; hh++)
                    a.res[hh * plane + (size_t)s * a.np + g] = v[hh] + shb[hh];
            }
        };
        // pterm rows of local tile `it` (buffer it & 1) have landed
        auto operands_ready = [&](int it) {
            (void)it;
            tc::cp_async_wait_all();
            tc::named_bar(1, EPI_THREADS); // pterm rows copied by other warps are visible
        };
        auto prefetch = [&](int it) {
            prefetch_tile(a, cluster + it * nclusters, rank, pbuf + (it & 1) * TS * PROW, et);
        };

        if (ntiles_mine > 0)
        {
            prefetch(0);
            operands_ready(0);
            if (ntiles_mine > 1)
                prefetch(1);
            convert_layer(0, 0);
        }
        for (int it = 0; it < ntiles_mine; it++)
        {
            for (int l = 1; l < NL; l++)
            {
                convert_layer(it, l);
                if (l == 3 && it + 1 < ntiles_mine)
                    operands_ready(it + 1);
            }
            if (it + 1 < ntiles_mine)
                convert_layer(it + 1, 0);
            heads(it);
            // tile it's buffers are free (its layers 0-7 are converted, layer 6 done)
            if (it + 2 < ntiles_mine)
                prefetch(it + 2);
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

uint16_t bf16_bits(float f)
{
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u)
        return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float bf16_float(uint16_t h)
{
    const uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// one K step (16 k) x `nc` output columns of a weight matrix as UMMA K-major core
// matrices, hi then lo: element (n_local, kk) at ((kk/8)*(nc/8) + n_local/8)*64 + (n_local%8)*8 + kk%8
template <class F>
void pack_kstep(uint16_t *dst, int nc, F &&w_of)
{
    uint16_t *hi = dst, *lo = dst + nc * 16;
    for (int nl = 0; nl < nc; nl++)
        for (int kk = 0; kk < 16; kk++)
        {
            const float w = w_of(nl, kk);
            const uint16_t hb = bf16_bits(w);
            const size_t idx = (size_t)((kk / 8) * (nc / 8) + nl / 8) * 64 + (nl % 8) * 8 + kk % 8;
            hi[idx] = hb;
            lo[idx] = bf16_bits(w - bf16_float(hb));
        }
}
} // namespace

bool mlp_tc_available() { return true; }

static long long *g_trace_buf = nullptr;
int mlp_tc_trace(long long *out)
{
    if (!g_trace_buf)
        return 1;
    cudaDeviceSynchronize();
    return cudaMemcpy(out, g_trace_buf, 3 * 9 * 128 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}

// cterm blocks from the per-Gaussian centre terms cg [np][4][160] (W_c xc of
// layers 0,2,4,6, FP32, center_terms_kernel): block b, layer j, column group
// n / 4, row = Gaussian % 32 -> the tcgen05.cp source layout (zero rows past np)
__global__ void cterm_pack_kernel(const float *__restrict__ cg, float *__restrict__ ct, int np, int nblk)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nblk * TG * 4 * WPC)
        return;
    const int n = (int)(idx % WPC), j = (int)((idx / WPC) % 4);
    const int g = (int)(idx / (4 * WPC));
    const int blk = g / TG, row = g % TG;
    const size_t dst = ((size_t)blk * 4 + j) * (C_BLOCK / 4) + ((size_t)(n / 4) * TG + row) * 4 + n % 4;
    ct[dst] = g < np ? cg[((size_t)g * 4 + j) * WPC + n] : 0.0f;
}

// Pack the weights in the kernel's consumption order (see stage_bytes): per trunk
// layer l = 1..7 and output part p, for pair rank 0 then 1 (each its half of the
// part's columns): the 10 hidden K steps; finally the heads (N = 32, columns 0-4
// real). Layer 0 streams no weights (its accumulator is the cterm alone).
// whT: [7][k][n] hidden weights (k-major); heads: [5][wp]. The cterm blocks are
// repacked on the device from c.net.cg.
void prepare_tc_weights(Ctx &c, const std::vector<float> &whT, const std::vector<float> &heads)
{
    const int WP = c.net.wp;
    std::vector<uint16_t> packed;
    auto kstep = [&](int nc, auto &&w_of) {
        const size_t at = packed.size();
        packed.resize(at + 2 * nc * 16);
        pack_kstep(packed.data() + at, nc, w_of);
    };
    for (int l = 1; l < NL; l++)
        for (int p = 0; p < NPART; p++)
            for (int rk = 0; rk < 2; rk++)
            {
                const int nc = npart(p) / 2, cbase = pcol(p) + rk * nc;
                for (int k = 0; k < KSTEPS; k++)
                    kstep(nc, [&](int nl, int k16) {
                        return whT[((size_t)(l - 1) * WP + (k * 16 + k16)) * WP + cbase + nl];
                    });
            }
    for (int rk = 0; rk < 2; rk++)
        for (int k = 0; k < KSTEPS; k++)
            kstep(NHEAD_N / 2, [&](int nl, int k16) {
                const int n = rk * (NHEAD_N / 2) + nl;
                return n < 5 ? heads[(size_t)n * WP + k * 16 + k16] : 0.0f;
            });
    if (packed.size() * 2 != stream_offset(NL, 0) + 2 * (size_t)HEAD_STAGE)
        throw std::logic_error("tc weight stream size");
    void *d = nullptr;
    check_cuda(cudaMalloc(&d, packed.size() * 2), "cudaMalloc tc weights");
    c.allocs.push_back(d);
    check_cuda(cudaMemcpy(d, packed.data(), packed.size() * 2, cudaMemcpyHostToDevice), "upload tc weights");
    c.net.w_tc = static_cast<uint16_t *>(d);

    const int nblk = (c.g.n + TG - 1) / TG;
    const size_t total = (size_t)nblk * TG * 4 * WPC;
    check_cuda(cudaMalloc(&d, total * sizeof(float)), "cudaMalloc cterm blocks");
    c.allocs.push_back(d);
    c.net.c_tc = static_cast<float *>(d);
    cterm_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c.stream>>>(c.net.cg, c.net.c_tc, c.g.np, nblk);
    check_cuda(cudaStreamSynchronize(c.stream), "cterm blocks");
}

void launch_mlp_tc(Ctx &c, int nb, cudaStream_t st)
{
    static int max_clusters = 0;
    if (!max_clusters)
    {
        check_cuda(cudaFuncSetAttribute(mlp_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES),
                   "tc mlp smem attribute");
        check_cuda(cudaFuncSetAttribute(mlp_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES),
                   "tc mlp smem attribute");
        // all 228 KB as shared memory: the SM then has room for a raster CTA next to
        // this persistent CTA (without it the driver sizes the carveout to this
        // kernel alone and nothing else can share the SM)
        for (auto k : {mlp_tc_kernel<true>, mlp_tc_kernel<false>})
            check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            (int)cudaSharedmemCarveoutMaxShared),
                       "tc mlp carveout");
        // persistent grid: as many CTA pairs as can be co-resident (TPCs whose two
        // SMs are both available), never more -- a second wave would double the time
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
        check_cuda(cudaOccupancyMaxActiveClusters(&max_clusters, mlp_tc_kernel<true>, &cfg),
                   "tc mlp cluster occupancy");
        if (max_clusters < 1)
            check_cuda(cudaErrorLaunchOutOfResources, "tc mlp: no CTA pair fits on this device");
    }
    TcArgs a;
    a.w_tc = c.net.w_tc;
    a.cterm = c.net.c_tc;
    a.bias = c.net.bias;
    a.pterm = c.w.pterm;
    a.hbias = c.net.hbias;
    a.res = c.w.res;
    a.n = c.g.n;
    a.np = c.g.np;
    a.nb = nb;
    a.cap_b = (int)c.w.cap_b;
    a.n_sblk = (nb + PAIR_S - 1) / PAIR_S;
    const int n_gblk = (c.g.n + TG - 1) / TG;
    a.ntiles = n_gblk * a.n_sblk;
    a.split = c.mlp_precision == 1 ? 1 : 0;
    a.debug = getenv("SWR_TC_DEBUG") ? atoi(getenv("SWR_TC_DEBUG")) : 0;
    a.trace = nullptr;
    if (a.debug & 8)
    {
        static long long *buf = nullptr;
        if (!buf)
            check_cuda(cudaMalloc(&buf, 3 * 9 * 128 * sizeof(long long)), "trace buffer");
        cudaMemsetAsync(buf, 0, 3 * 9 * 128 * sizeof(long long), st);
        a.trace = buf;
        g_trace_buf = buf;
    }
    const int grid = 2 * std::min(max_clusters, a.ntiles);
    if (a.split)
        mlp_tc_kernel<true><<<grid, THREADS, SMEM_BYTES, st>>>(a);
    else
        mlp_tc_kernel<false><<<grid, THREADS, SMEM_BYTES, st>>>(a);
    c.launches++;
}

} // namespace swr
