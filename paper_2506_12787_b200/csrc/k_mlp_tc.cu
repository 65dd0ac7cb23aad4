// Deformation MLP on the 5th-generation tensor cores (tcgen05), split precision.
//
// Same function as the FP32 kernel in k_mlp.cu (deform.cpp:140-207 with the
// encoding blocks factored into cg[g] + pterm[s]); the seven hidden->hidden
// 160x160 products run on the tensor cores with FP32 accumulators in TMEM:
//
//   a = a_hi + a_lo, w = w_hi + w_lo  (bf16 pairs, |a - a_hi - a_lo| <= 2^-17 |a|)
//   a.w ~= a_hi.w_hi + a_lo.w_hi + a_hi.w_lo        ("bf16x3", 3 UMMAs per K step)
//
// which keeps ~16 significant bits per product (measured: residuals within
// ~1e-5 relative of the FP64 oracle); SWR_MLP_BF16 issues only a_hi.w_hi.
//
// Structure (one persistent CTA per SM, 18 warps, one 128-row tile in flight):
//   warp 16     producer: streams each layer's packed weight K-chunks (hi+lo,
//               10 KB) from L2 into a shared-memory ring (cp.async.bulk, mbarrier
//               complete_tx);
//   warp 17     MMA issuer (one thread): tcgen05.mma M=128 N=160 K=16 with the
//               A operand in TMEM ("TS" form) and B from shared memory;
//   warps 0-15  epilogue, 4 column groups x 4 TMEM lane quarters. Layer l's FP32
//               accumulator is converted IN PLACE into layer l+1's bf16 hi/lo A
//               operand (tcgen05.ld -> + bias or cg[g] + pterm[s] -> ReLU -> split
//               -> tcgen05.st), 16 columns at a time; each converted chunk is
//               published on its own mbarrier so the next layer's UMMAs start on
//               chunk 0 while later chunks are still being converted.
// TMEM holds three 160-column regions used round-robin (accumulator / A of the
// next layer / the previous tile's layer-7 accumulator being reduced by the
// heads), so the heads of tile i overlap the first UMMAs of tile i+1. Shared
// memory carries only the weight ring and the tile's cg/pterm rows (double
// buffered, cp.async prefetch one tile ahead).
#include "swr_internal.h"
#include "tc_ptx.cuh"

#include <cstdio>
#ifdef SWR_TC_DEBUG_WAITS
#define MBAR_WAIT(b, p, tag) tc::mbar_wait_dbg(b, p, tag)
#else
#define MBAR_WAIT(b, p, tag) tc::mbar_wait(b, p)
#endif
#ifdef SWR_TC_DEBUG_WAITS
#define MBAR_POLL(b, p, tag) tc::mbar_wait_dbg(b, p, tag)
#else
#define MBAR_POLL(b, p, tag) tc::mbar_poll(b, p)
#endif

#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

namespace swr
{

namespace
{
constexpr int TM = 128;                 // rows per tile (16 Gaussians x 8 positions)
constexpr int WPC = 160;                // padded width (N and K of the hidden layers)
constexpr int KSTEPS = WPC / 16;        // 10 UMMA K steps per layer
constexpr int NL = 7;                   // hidden->hidden layers 1..7
constexpr int B_CHUNK = WPC * 16 * 2;   // one K step of one weight operand: 5 KB
constexpr int B_LBO = (WPC / 8) * 128;
constexpr int B_SBO = 128;
constexpr int KPS = 2;                  // UMMA K steps per ring stage / per epilogue chunk
constexpr int NCH = KSTEPS / KPS;       // 5 stages (and 32-column chunks) per layer
constexpr int STAGE = KPS * 2 * B_CHUNK; // hi + lo of KPS K steps: 20 KB
constexpr int NSTAGE = 4;
constexpr int LK_ELEMS = 2 * B_CHUNK / 2; // bf16 elements (hi + lo) of one (layer, K step) block
constexpr int EPI_WARPS = 16;
constexpr int EPI_THREADS = 32 * EPI_WARPS;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int NREG = 3;                 // TMEM regions of 160 columns
// The warp scheduler prefers higher warp ids: the single-thread producer and
// MMA issuer sit above the 16 epilogue warps so they are never starved.
constexpr int kProducerWarp = EPI_WARPS, kMmaWarp = EPI_WARPS + 1;
// per-tile addend block in shared memory: cg rows of 16 Gaussians and pterm rows
// of 8 positions, 4 layers each, rows skewed by 8 / 4 floats against bank conflicts
constexpr int CROW = 4 * WPC;
constexpr int CS_FLOATS = 16 * CROW + 16 * 8;
constexpr int PS_FLOATS = 8 * CROW + 8 * 4;
constexpr int CP_FLOATS = CS_FLOATS + PS_FLOATS;
constexpr int SMEM_RING = NSTAGE * STAGE;
constexpr int SMEM_CP = 2 * CP_FLOATS * 4;
constexpr int SMEM_CONST = (8 * WPC + 5 * WPC + 8) * 4;
constexpr int SMEM_HX = 4 * TM * 5 * 4;
constexpr int NBARS = 2 * NSTAGE + 2 * NCH + 2;
constexpr int SMEM_BYTES = SMEM_RING + SMEM_CP + SMEM_CONST + SMEM_HX + NBARS * 8 + 16 + 1024;

struct TcArgs
{
    const uint16_t *w_tc;  // [7][10][hi 2560 | lo 2560] bf16 bits, UMMA core-matrix layout
    const float *bias;     // [8][160]
    const float *cg;       // [np][4][160]
    const float *pterm;    // [nb][4][160]
    const float *heads;    // [5][160]
    const float *hbias;    // [5]
    float *res;            // [5][cap_b][np]
    int n, np, nb, cap_b, n_sblk, ntiles, split, debug;
    long long *trace; // debug: [3 tiles][8 layers][80 slots] clock64 stamps of block 0
    uint32_t idesc;
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi)
{
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi); // .x -> low 16 bits
    return *reinterpret_cast<uint32_t *>(&h);
}

// 16 consecutive K elements -> 8 columns of hi pairs, then 8 columns of lo pairs
__device__ __forceinline__ void split16(const float (&v)[16], uint32_t (&o)[16])
{
#pragma unroll
    for (int i = 0; i < 8; i++)
    {
        const uint32_t h = pack_bf16(v[2 * i], v[2 * i + 1]);
        const float h0 = __uint_as_float(h << 16), h1 = __uint_as_float(h & 0xffff0000u);
        o[i] = h;
        o[8 + i] = pack_bf16(v[2 * i] - h0, v[2 * i + 1] - h1);
    }
}

// 16 floats from shared memory (explicit ld.shared: the pointer arithmetic
// below loses the address space, generic loads would be slower)
__device__ __forceinline__ void lds16(const float *p, float (&v)[16])
{
    const uint32_t a = tc::smem_u32(p);
#pragma unroll
    for (int i = 0; i < 4; i++)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[4 * i]), "=f"(v[4 * i + 1]), "=f"(v[4 * i + 2]), "=f"(v[4 * i + 3])
                     : "r"(a + 16 * i));
}

__device__ __forceinline__ void tile_origin(const TcArgs &a, int tile, int &g0, int &s0)
{
    g0 = (tile / a.n_sblk) * 16;
    s0 = (tile % a.n_sblk) * 8;
}

// cp.async the tile's cg / pterm rows into one buffer (zero-fill outside the
// problem); issued by all epilogue threads
__device__ __forceinline__ void prefetch_cp(const TcArgs &a, int tile, float *buf, int et)
{
    int g0, s0;
    tile_origin(a, tile, g0, s0);
    constexpr int C16 = CROW / 4; // 16-byte pieces per row
    for (int i = et; i < 16 * C16; i += EPI_THREADS)
    {
        const int gl = i / C16, k = (i % C16) * 4;
        const int g = g0 + gl;
        const bool ok = g < a.n;
        tc::cp_async16(buf + gl * CROW + gl * 8 + k, a.cg + (size_t)(ok ? g : 0) * CROW + k, ok);
    }
    float *ps = buf + CS_FLOATS;
    for (int i = et; i < 8 * C16; i += EPI_THREADS)
    {
        const int sl = i / C16, k = (i % C16) * 4;
        const int s = s0 + sl;
        const bool ok = s < a.nb;
        tc::cp_async16(ps + sl * CROW + sl * 4 + k, a.pterm + (size_t)(ok ? s : 0) * CROW + k, ok);
    }
    tc::cp_async_commit();
}

__device__ __forceinline__ void stamp(const TcArgs &a, int it, int l, int slot)
{
    if (a.trace && blockIdx.x == 0 && it < 3)
        a.trace[(it * 8 + l) * 80 + slot] = clock64();
}

__global__ void __launch_bounds__(THREADS, 1) mlp_tc_kernel(TcArgs a)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ring = smem;
    float *cpbuf = reinterpret_cast<float *>(ring + SMEM_RING);       // [2][CP_FLOATS]
    float *sbias = cpbuf + 2 * CP_FLOATS;                             // [8][160]
    float *sheads = sbias + 8 * WPC;                                  // [5][160]
    float *shb = sheads + 5 * WPC;                                    // [8]
    float *hx = shb + 8;                                              // [4][128][5]
    uint64_t *bars = reinterpret_cast<uint64_t *>(hx + 4 * TM * 5);
    uint64_t *w_full = bars, *w_empty = bars + NSTAGE, *chunk_ready = bars + 2 * NSTAGE,
             *acc_full = bars + 2 * NSTAGE + 2 * NCH;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + NBARS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0)
    {
        for (int s = 0; s < NSTAGE; s++)
        {
            tc::mbar_init(&w_full[s], 1);
            tc::mbar_init(&w_empty[s], 1);
        }
        for (int k = 0; k < 2 * NCH; k++)
            tc::mbar_init(&chunk_ready[k], 8); // 2 column groups x 4 lane quarters per 32-column chunk
        tc::mbar_init(&acc_full[0], 1);
        tc::mbar_init(&acc_full[1], 1);
        tc::fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 8 * WPC; i += THREADS)
        sbias[i] = a.bias[i];
    for (int i = threadIdx.x; i < 5 * WPC; i += THREADS)
        sheads[i] = a.heads[i];
    if (threadIdx.x < 5)
        shb[threadIdx.x] = a.hbias[threadIdx.x];
    if (warp == kMmaWarp)
        tc::tmem_alloc<512>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int ntiles_mine = blockIdx.x < a.ntiles ? (a.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == kProducerWarp)
    {
        // whole warp converged; one elected lane issues (see tc::mbar_wait)
        int stage = 0;
        uint32_t ph = 0;
        for (int it = 0; it < ntiles_mine; it++)
            for (int l = 0; l < NL; l++)
                for (int k = 0; k < NCH; k++)
                {
                    MBAR_WAIT(&w_empty[stage], ph ^ 1, 1);
                    if (tc::elect_one())
                    {
                        if ((a.debug & 1) && it > 0)
                            tc::mbar_arrive(&w_full[stage]); // debug: stale weights, no TMA traffic
                        else
                        {
                            tc::mbar_arrive_expect_tx(&w_full[stage], STAGE);
                            tc::bulk_g2s(ring + stage * STAGE, a.w_tc + (size_t)(l * KSTEPS + k * KPS) * LK_ELEMS,
                                         STAGE, &w_full[stage]);
                        }
                    }
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
        // whole warp converged (waits by all lanes), UMMAs and commits by one
        // elected lane: keeps the issue loop free of YIELD/divergence overhead
        {
            int stage = 0;
            uint32_t ph = 0, cph[2] = {0, 0};
            const uint32_t r_base = tc::smem_u32(ring);
            for (int it = 0; it < ntiles_mine; it++)
                for (int l = 1; l <= NL; l++)
                {
                    const int u = 8 * it + l;
                    const uint32_t dreg = tmem + (u % NREG) * WPC;
                    const uint32_t areg = tmem + ((u + NREG - 1) % NREG) * WPC;
                    // chunk barriers alternate between two sets by conversion
                    // index (7 per tile: layers 0..6) so the layer-0 chunks of
                    // the next tile can never advance a set the UMMAs of this
                    // tile's layer 7 have not consumed yet
                    const int cs = (7 * it + l - 1) & 1;
                    uint64_t *cready = chunk_ready + cs * NCH;
                    for (int j = 0; j < NCH; j++)
                    {
                        MBAR_WAIT(&cready[j], cph[cs], 100 + j);
                        MBAR_WAIT(&w_full[stage], ph, 2);
                        tc::tc_fence_after();
                        if (lane == 0)
                            stamp(a, it, l, j);
                        const uint32_t b = r_base + stage * STAGE;
                        const bool leader = tc::elect_one();
#pragma unroll
                        for (int kk = 0; kk < KPS && leader; kk++)
                        {
                            const int k = j * KPS + kk;
                            const uint64_t dbh = tc::make_desc(b + kk * 2 * B_CHUNK, B_LBO, B_SBO);
                            const uint32_t ahi = areg + 16 * k;
                            tc::mma_f16_ts(dreg, ahi, dbh, a.idesc, k > 0 ? 1u : 0u);
                            if (a.split)
                            {
                                const uint64_t dbl = tc::make_desc(b + kk * 2 * B_CHUNK + B_CHUNK, B_LBO, B_SBO);
                                tc::mma_f16_ts(dreg, ahi + 8, dbh, a.idesc, 1u);
                                tc::mma_f16_ts(dreg, ahi, dbl, a.idesc, 1u);
                            }
                        }
                        if (leader)
                            tc::mma_commit(&w_empty[stage]);
                        __syncwarp();
                        if (++stage == NSTAGE)
                        {
                            stage = 0;
                            ph ^= 1;
                        }
                    }
                    cph[cs] ^= 1;
                    // accumulators alternate between two barriers (MMA layer
                    // index parity) so neither can run two phases ahead of
                    // the epilogue's waits
                    if (tc::elect_one())
                        tc::mma_commit(&acc_full[(7 * it + l - 1) & 1]);
                    __syncwarp();
                    if (lane == 0)
                        stamp(a, it, l, 10);
                }
        }
    }
    else
    {
        const int e = warp;           // 0..15
        const int et = threadIdx.x;
        const int q = warp & 3;       // TMEM lane quarter this warp may access
        // column group: 16-column units grp, grp+4, grp+8. Group 0 (units 0, 4, 8)
        // sits on the highest epilogue warp ids: the scheduler favours it, so the
        // first chunk of each layer is ready as early as possible.
        const int grp = 3 - (e >> 2);
        const int r = q * 32 + lane;  // row in tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int gl = r >> 3, sl = r & 7;
        uint32_t fph[2] = {0, 0};
        if (ntiles_mine > 0)
            prefetch_cp(a, blockIdx.x, cpbuf, et);

        // heads of the tile whose layer-7 accumulator sits in region `reg`
        auto wait_acc = [&](int m) {
            MBAR_WAIT(&acc_full[m & 1], fph[m & 1], 10 + (m & 1));
            fph[m & 1] ^= 1;
        };
        auto heads = [&](int tile, int reg, int m) {
            wait_acc(m);
            tc::tc_fence_after();
            float acc5[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
            for (int sc = grp; sc < KSTEPS; sc += 4) // 16-column units round robin over the groups
            {
                const int n0 = sc * 16;
                float v[16], x[16];
                tc::tmem_ld16(tmem + reg * WPC + lane_off + n0, v);
                lds16(sbias + NL * WPC + n0, x);
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = fmaxf(v[i] + x[i], 0.0f);
#pragma unroll
                for (int h = 0; h < 5; h++)
                {
                    lds16(sheads + h * WPC + n0, x);
#pragma unroll
                    for (int i = 0; i < 16; i++)
                        acc5[h] = __fmaf_rn(v[i], x[i], acc5[h]);
                }
            }
            tc::tc_fence_before();
#pragma unroll
            for (int h = 0; h < 5; h++)
                hx[(grp * TM + r) * 5 + h] = acc5[h];
            tc::named_bar(2, EPI_THREADS);
            if (grp == 0)
            {
                int g0, s0;
                tile_origin(a, tile, g0, s0);
                const int g = g0 + gl, s = s0 + sl;
                if (g < a.n && s < a.nb)
                {
                    const size_t plane = (size_t)a.cap_b * a.np;
#pragma unroll
                    for (int h = 0; h < 5; h++)
                    {
                        const float t = ((acc5[h] + hx[(1 * TM + r) * 5 + h]) + hx[(2 * TM + r) * 5 + h]) +
                                        hx[(3 * TM + r) * 5 + h];
                        a.res[h * plane + (size_t)s * a.np + g] = t + shb[h];
                    }
                }
            }
        };

        for (int it = 0; it < ntiles_mine; it++)
        {
            const int tile = blockIdx.x + it * gridDim.x;
            float *cp = cpbuf + (it & 1) * CP_FLOATS;
            const float *crow = cp + gl * CROW + gl * 8;            // cg rows of this row's Gaussian
            const float *prow = cp + CS_FLOATS + sl * CROW + sl * 4; // pterm rows of this row's position
            int g0, s0;
            tile_origin(a, tile, g0, s0);
            const bool live = g0 + gl < a.n && s0 + sl < a.nb;
            tc::cp_async_wait_all();
#ifdef SWR_TC_DEBUG_WAITS
            if (blockIdx.x == 0 && lane == 0)
                printf("epi warp %d tile %d before bar1\n", warp, it);
#endif
            tc::named_bar(1, EPI_THREADS);
#ifdef SWR_TC_DEBUG_WAITS
            if (blockIdx.x == 0 && lane == 0)
                printf("epi warp %d tile %d after bar1\n", warp, it);
#endif
            if (it + 1 < ntiles_mine)
                prefetch_cp(a, tile + gridDim.x, cpbuf + ((it + 1) & 1) * CP_FLOATS, et);
            // ---- layer 0: A = split(ReLU(cg[g][0] + pterm[s][0])) into region (8 it) % 3
            {
                const uint32_t reg = tmem + ((8 * it) % NREG) * WPC + lane_off;
                for (int sc = grp; sc < KSTEPS; sc += 4)
                {
                    const int c = sc >> 1; // 32-column chunk of this 16-column unit
                    {
                        const int n0 = sc * 16;
                        float v[16], x[16];
                        lds16(crow + n0, v);
                        lds16(prow + n0, x);
#pragma unroll
                        for (int i = 0; i < 16; i++)
                            v[i] = live ? fmaxf(v[i] + x[i], 0.0f) : 0.0f;
                        uint32_t o[16];
                        split16(v, o);
                        tc::tmem_st16(reg + n0, o);
                    }
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        tc::mbar_arrive(&chunk_ready[((7 * it) & 1) * NCH + c]);
#ifdef SWR_TC_DEBUG_WAITS
                    if (blockIdx.x == 0 && lane == 0)
                        printf("epi warp %d tile %d L0 chunk %d arrived\n", warp, it, c);
#endif
                }
            }
            if (it > 0)
                heads(tile - gridDim.x, (8 * it - 1) % NREG, 7 * it - 1);
            // ---- layers 1..6: accumulator -> next layer's A, in place
            for (int l = 1; l < NL; l++)
            {
                const bool skip = (l == 2 || l == 4 || l == 6);
                const int u = 8 * it + l;
                const uint32_t reg = tmem + (u % NREG) * WPC + lane_off;
                wait_acc(7 * it + l - 1);
                tc::tc_fence_after();
                if (lane == 0)
                    stamp(a, it, l, 16 + e);
                for (int sc = grp; sc < KSTEPS; sc += 4)
                {
                    const int c = sc >> 1; // 32-column chunk of this 16-column unit
                    {
                        const int n0 = sc * 16;
                        float v[16], x[16];
                        if (skip)
                        {
                            float y[16];
                            lds16(crow + (l / 2) * WPC + n0, x);
                            lds16(prow + (l / 2) * WPC + n0, y);
#pragma unroll
                            for (int i = 0; i < 16; i++)
                                x[i] += y[i];
                        }
                        else
                            lds16(sbias + l * WPC + n0, x);
                        tc::tmem_ld16(reg + n0, v);
#pragma unroll
                        for (int i = 0; i < 16; i++)
                            v[i] = fmaxf(v[i] + x[i], 0.0f);
                        uint32_t o[16];
                        split16(v, o);
                        tc::tmem_st16(reg + n0, o);
                    }
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                    {
                        tc::mbar_arrive(&chunk_ready[((7 * it + l) & 1) * NCH + c]);
                        stamp(a, it, l, 32 + c * 4 + q);
                    }
                }
            }
        }
        if (ntiles_mine > 0)
            heads(blockIdx.x + (ntiles_mine - 1) * gridDim.x, (8 * ntiles_mine - 1) % NREG, 7 * ntiles_mine - 1);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp)
    {
        tc::tc_fence_after();
        tc::tmem_dealloc<512>(tmem);
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
} // namespace

bool mlp_tc_available() { return true; }

static long long *g_trace_buf = nullptr;
int mlp_tc_trace(long long *out)
{
    if (!g_trace_buf)
        return 1;
    cudaDeviceSynchronize();
    return cudaMemcpy(out, g_trace_buf, 3 * 8 * 80 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}

// Pack the seven hidden->hidden layers (whT: [7][k][n], zero padded to 160)
// into UMMA K-major core-matrix chunks: per (layer, K step) 160 rows (n) x 16
// (k) of w_hi, then of w_lo; element (n, kk) of a chunk at
// ((kk/8)*20 + n/8)*64 + (n%8)*8 + kk%8.
void prepare_tc_weights(Ctx &c, const std::vector<float> &whT)
{
    const int WP = c.net.wp;
    std::vector<uint16_t> packed((size_t)NL * KSTEPS * LK_ELEMS);
    for (int l = 0; l < NL; l++)
        for (int k = 0; k < KSTEPS; k++)
        {
            uint16_t *hi = packed.data() + (size_t)(l * KSTEPS + k) * LK_ELEMS;
            uint16_t *lo = hi + B_CHUNK / 2;
            for (int n = 0; n < WPC; n++)
                for (int kk = 0; kk < 16; kk++)
                {
                    const float w = whT[((size_t)l * WP + (k * 16 + kk)) * WP + n];
                    const uint16_t h = bf16_bits(w);
                    const uint16_t lw = bf16_bits(w - bf16_float(h));
                    const size_t idx = (size_t)((kk / 8) * (WPC / 8) + n / 8) * 64 + (n % 8) * 8 + kk % 8;
                    hi[idx] = h;
                    lo[idx] = lw;
                }
        }
    void *d = nullptr;
    check_cuda(cudaMalloc(&d, packed.size() * 2), "cudaMalloc tc weights");
    c.allocs.push_back(d);
    check_cuda(cudaMemcpy(d, packed.data(), packed.size() * 2, cudaMemcpyHostToDevice), "upload tc weights");
    c.net.w_tc = static_cast<uint16_t *>(d);
}

void launch_mlp_tc(Ctx &c, int nb, cudaStream_t st)
{
    static bool configured = false;
    if (!configured)
    {
        check_cuda(cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES),
                   "tc mlp smem attribute");
        configured = true;
    }
    TcArgs a;
    a.w_tc = c.net.w_tc;
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
    a.n_sblk = (nb + 7) / 8;
    const int n_gblk = (c.g.n + 15) / 16;
    a.ntiles = n_gblk * a.n_sblk;
    a.split = c.mlp_precision == 1 ? 1 : 0;
    a.idesc = tc::make_idesc(1, TM, WPC);
    a.debug = getenv("SWR_TC_DEBUG") ? atoi(getenv("SWR_TC_DEBUG")) : 0;
    a.trace = nullptr;
    if (a.debug & 8)
    {
        static long long *buf = nullptr;
        if (!buf)
            check_cuda(cudaMalloc(&buf, 3 * 8 * 80 * sizeof(long long)), "trace buffer");
        cudaMemsetAsync(buf, 0, 3 * 8 * 80 * sizeof(long long), st);
        a.trace = buf;
        g_trace_buf = buf;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int grid = std::min(sms, a.ntiles);
    mlp_tc_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(a);
    c.launches++;
}

} // namespace swr
