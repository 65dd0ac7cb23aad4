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
// Structure (one persistent CTA per SM, 18 warps):
//   warp 0      TMA-engine producer: streams each layer's packed weight K-chunks
//               (hi+lo, 10 KB) from L2 into a 5-stage shared-memory ring
//               (cp.async.bulk + mbarrier complete_tx);
//   warp 1      MMA issuer (one thread): tcgen05.mma M=128 N=160 K=16 into TMEM,
//               tcgen05.commit releases ring slots / publishes accumulators;
//   warps 2-17  epilogue, 8 warps per tile slot (2 per TMEM lane quarter): TMEM
//               -> registers (tcgen05.ld), + bias or cg[g] + pterm[s], ReLU,
//               hi/lo split, st.shared straight into the next layer's A operand
//               (K-major core-matrix layout); after layer 7 the 5 heads in FP32.
// Two 128-row tiles ping-pong: while the tensor core runs tile 0's layer the
// epilogue warps of tile 1 turn its previous accumulator into the next A.
#include "swr_internal.h"
#include "tc_ptx.cuh"

#include <cuda_bf16.h>

#include <cstring>

namespace swr
{

namespace
{
constexpr int TM = 128;                 // rows per tile (16 Gaussians x 8 positions)
constexpr int WPC = 160;                // padded width (N and K of the hidden layers)
constexpr int KSTEPS = WPC / 16;        // 10 UMMA K steps per layer
constexpr int NL = 7;                   // hidden->hidden layers 1..7
constexpr int A_BYTES = TM * WPC * 2;   // one bf16 operand (hi or lo) of one tile: 40 KB
constexpr int A_LBO = (TM / 8) * 128;   // byte stride between K-adjacent core matrices
constexpr int A_SBO = 128;              // byte stride between 8-row groups
constexpr int B_CHUNK = WPC * 16 * 2;   // one K step of one weight operand: 5 KB
constexpr int B_LBO = (WPC / 8) * 128;
constexpr int B_SBO = 128;
constexpr int STAGE = 2 * B_CHUNK;      // hi + lo
constexpr int NSTAGE = 5;
constexpr int EPI_WARPS = 8;            // per tile slot
constexpr int THREADS = 32 * (2 + 2 * EPI_WARPS);
constexpr int SMEM_A = 2 * 2 * A_BYTES;
constexpr int SMEM_RING = NSTAGE * STAGE;
constexpr int SMEM_HX = 2 * TM * 5 * 4;
constexpr int SMEM_BYTES = SMEM_A + SMEM_RING + SMEM_HX + 256 + 1024; // + barriers + alignment slack

struct TcArgs
{
    const uint16_t *w_tc;  // [7][10][hi 2560 | lo 2560] bf16 bits, UMMA core-matrix layout
    const float *bias;     // [8][160]
    const float *cg;       // [np][4][160]
    const float *pterm;    // [nb][4][160]
    const float *heads;    // [5][160]
    const float *hbias;    // [5]
    float *res;            // [5][cap_b][np]
    int n, np, nb, cap_b, n_sblk, ntiles, npairs, split;
    uint32_t idesc;
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi)
{
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi); // .x -> low 16 bits
    return *reinterpret_cast<uint32_t *>(&h);
}

// write 16 consecutive columns [n0, n0+16) of row r as hi/lo bf16 into the
// K-major core-matrix layout of one tile's A operand
__device__ __forceinline__ void store_split(uint8_t *Ahi, uint8_t *Alo, int r, int n0, const float (&v)[16])
{
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; i++)
    {
        hi[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
        const float h0 = __uint_as_float(hi[i] << 16), h1 = __uint_as_float(hi[i] & 0xffff0000u);
        lo[i] = pack_bf16(v[2 * i] - h0, v[2 * i + 1] - h1);
    }
    const int off = (n0 >> 3) * A_LBO + (r >> 3) * A_SBO + (r & 7) * 16;
    *reinterpret_cast<uint4 *>(Ahi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4 *>(Ahi + off + A_LBO) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
    *reinterpret_cast<uint4 *>(Alo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    *reinterpret_cast<uint4 *>(Alo + off + A_LBO) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
}

__device__ __forceinline__ void ld16(const float *p, float (&v)[16])
{
#pragma unroll
    for (int i = 0; i < 4; i++)
    {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(p) + i);
        v[4 * i] = t.x;
        v[4 * i + 1] = t.y;
        v[4 * i + 2] = t.z;
        v[4 * i + 3] = t.w;
    }
}

__global__ void __launch_bounds__(THREADS, 1) mlp_tc_kernel(TcArgs a)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *A = smem;
    uint8_t *ring = smem + SMEM_A;
    float *hx = reinterpret_cast<float *>(ring + SMEM_RING);
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(hx) + SMEM_HX);
    uint64_t *w_full = bars, *w_empty = bars + NSTAGE, *a_ready = bars + 2 * NSTAGE, *acc_full = bars + 2 * NSTAGE + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NSTAGE + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0)
    {
        for (int s = 0; s < NSTAGE; s++)
        {
            tc::mbar_init(&w_full[s], 1);
            tc::mbar_init(&w_empty[s], 1);
        }
        for (int t = 0; t < 2; t++)
        {
            tc::mbar_init(&a_ready[t], EPI_WARPS);
            tc::mbar_init(&acc_full[t], 1);
        }
        tc::fence_mbar_init();
    }
    if (warp == 1)
        tc::tmem_alloc<512>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0)
    {
        if (lane == 0)
        {
            int stage = 0;
            uint32_t ph = 0;
            for (int p = blockIdx.x; p < a.npairs; p += gridDim.x)
                for (int l = 0; l < NL; l++)
                    for (int t = 0; t < 2; t++)
                        for (int k = 0; k < KSTEPS; k++)
                        {
                            tc::mbar_wait(&w_empty[stage], ph ^ 1);
                            tc::mbar_arrive_expect_tx(&w_full[stage], STAGE);
                            tc::bulk_g2s(ring + stage * STAGE, a.w_tc + (size_t)(l * KSTEPS + k) * (STAGE / 2), STAGE,
                                         &w_full[stage]);
                            if (++stage == NSTAGE)
                            {
                                stage = 0;
                                ph ^= 1;
                            }
                        }
        }
    }
    else if (warp == 1)
    {
        if (lane == 0)
        {
            int stage = 0;
            uint32_t ph = 0, aph[2] = {0, 0};
            const uint32_t a_base = tc::smem_u32(A), r_base = tc::smem_u32(ring);
            for (int p = blockIdx.x; p < a.npairs; p += gridDim.x)
                for (int l = 0; l < NL; l++)
                    for (int t = 0; t < 2; t++)
                    {
                        tc::mbar_wait(&a_ready[t], aph[t]);
                        aph[t] ^= 1;
                        tc::tc_fence_after();
                        const uint32_t d = tmem + t * WPC;
                        const uint32_t ahi = a_base + t * 2 * A_BYTES, alo = ahi + A_BYTES;
                        for (int k = 0; k < KSTEPS; k++)
                        {
                            tc::mbar_wait(&w_full[stage], ph);
                            tc::tc_fence_after();
                            const uint32_t b = r_base + stage * STAGE;
                            const uint64_t dah = tc::make_desc(ahi + 2 * k * A_LBO, A_LBO, A_SBO);
                            const uint64_t dbh = tc::make_desc(b, B_LBO, B_SBO);
                            tc::mma_f16(d, dah, dbh, a.idesc, k > 0 ? 1u : 0u);
                            if (a.split)
                            {
                                const uint64_t dal = tc::make_desc(alo + 2 * k * A_LBO, A_LBO, A_SBO);
                                const uint64_t dbl = tc::make_desc(b + B_CHUNK, B_LBO, B_SBO);
                                tc::mma_f16(d, dal, dbh, a.idesc, 1u);
                                tc::mma_f16(d, dah, dbl, a.idesc, 1u);
                            }
                            tc::mma_commit(&w_empty[stage]);
                            if (++stage == NSTAGE)
                            {
                                stage = 0;
                                ph ^= 1;
                            }
                        }
                        tc::mma_commit(&acc_full[t]);
                    }
        }
    }
    else
    {
        const int e = warp - 2;      // 0..15
        const int t = e / EPI_WARPS; // tile slot
        const int q = warp & 3;      // TMEM lane quarter this warp may access
        const int half = (e % EPI_WARPS) / 4;
        const int r = q * 32 + lane;
        uint8_t *Ahi = A + t * 2 * A_BYTES, *Alo = Ahi + A_BYTES;
        const uint32_t tacc = tmem + t * WPC + ((uint32_t)(q * 32) << 16);
        uint32_t fph = 0;
        for (int p = blockIdx.x; p < a.npairs; p += gridDim.x)
        {
            const int tile = 2 * p + t;
            const int g0 = (tile / a.n_sblk) * 16, s0 = (tile % a.n_sblk) * 8;
            const int g = g0 + (r >> 3), s = s0 + (r & 7);
            const bool live = tile < a.ntiles && g < a.n && s < a.nb;
            const float *cg_row = a.cg + (size_t)(live ? g : 0) * 4 * WPC;
            const float *pt_row = a.pterm + (size_t)(live ? s : 0) * 4 * WPC;
            // ---- layer 0: ReLU(cg[g][0] + pterm[s][0])
#pragma unroll 1
            for (int c = 0; c < 5; c++)
            {
                const int n0 = half * 80 + c * 16;
                float v[16], w[16];
                ld16(cg_row + n0, v);
                ld16(pt_row + n0, w);
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = live ? fmaxf(v[i] + w[i], 0.0f) : 0.0f;
                store_split(Ahi, Alo, r, n0, v);
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0)
                tc::mbar_arrive(&a_ready[t]);
            // ---- layers 1..7
#pragma unroll 1
            for (int l = 1; l <= NL; l++)
            {
                tc::mbar_wait(&acc_full[t], fph);
                fph ^= 1;
                tc::tc_fence_after();
                const bool skip = (l == 2 || l == 4 || l == 6);
                if (l < NL)
                {
#pragma unroll 1
                    for (int c = 0; c < 5; c++)
                    {
                        const int n0 = half * 80 + c * 16;
                        float v[16], x[16];
                        tc::tmem_ld16(tacc + n0, v);
                        if (skip)
                        {
                            float y[16];
                            ld16(cg_row + (l / 2) * WPC + n0, x);
                            ld16(pt_row + (l / 2) * WPC + n0, y);
#pragma unroll
                            for (int i = 0; i < 16; i++)
                                x[i] += y[i];
                        }
                        else
                            ld16(a.bias + l * WPC + n0, x);
#pragma unroll
                        for (int i = 0; i < 16; i++)
                            v[i] = fmaxf(v[i] + x[i], 0.0f);
                        store_split(Ahi, Alo, r, n0, v);
                    }
                    tc::fence_proxy_async_smem();
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        tc::mbar_arrive(&a_ready[t]);
                }
                else
                {
                    float acc5[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
                    for (int c = 0; c < 5; c++)
                    {
                        const int n0 = half * 80 + c * 16;
                        float v[16], x[16];
                        tc::tmem_ld16(tacc + n0, v);
                        ld16(a.bias + NL * WPC + n0, x);
#pragma unroll
                        for (int i = 0; i < 16; i++)
                            v[i] = fmaxf(v[i] + x[i], 0.0f);
#pragma unroll
                        for (int h = 0; h < 5; h++)
                        {
                            ld16(a.heads + h * WPC + n0, x);
#pragma unroll
                            for (int i = 0; i < 16; i++)
                                acc5[h] = __fmaf_rn(v[i], x[i], acc5[h]);
                        }
                    }
                    tc::tc_fence_before();
                    float *xr = hx + ((size_t)t * TM + r) * 5;
                    if (half == 1)
#pragma unroll
                        for (int h = 0; h < 5; h++)
                            xr[h] = acc5[h];
                    asm volatile("bar.sync %0, %1;" ::"r"(1 + t), "r"(EPI_WARPS * 32));
                    if (half == 0 && live)
                    {
                        const size_t plane = (size_t)a.cap_b * a.np;
#pragma unroll
                        for (int h = 0; h < 5; h++)
                            a.res[h * plane + (size_t)s * a.np + g] = acc5[h] + xr[h] + a.hbias[h];
                    }
                }
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1)
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

// Pack the seven hidden->hidden layers (whT: [7][k][n], zero padded to 160)
// into UMMA K-major core-matrix chunks: per (layer, K step) 160 rows (n) x 16
// (k) of w_hi, then of w_lo; element (n, kk) of a chunk at
// ((kk/8)*20 + n/8)*64 + (n%8)*8 + kk%8.
void prepare_tc_weights(Ctx &c, const std::vector<float> &whT)
{
    const int WP = c.net.wp;
    std::vector<uint16_t> packed((size_t)NL * KSTEPS * (STAGE / 2));
    for (int l = 0; l < NL; l++)
        for (int k = 0; k < KSTEPS; k++)
        {
            uint16_t *hi = packed.data() + (size_t)(l * KSTEPS + k) * (STAGE / 2);
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
    a.npairs = (a.ntiles + 1) / 2;
    a.split = c.mlp_precision == 1 ? 1 : 0;
    a.idesc = tc::make_idesc(1, TM, WPC);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int grid = std::min(sms, a.npairs);
    mlp_tc_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(a);
    c.launches++;
}

} // namespace swr
