// Deformation-network training GEMMs on the tensor cores at FP32 accuracy
// (deform.cpp:126-137 forward, 237-326 backward).
//
// 3xTF32: every operand is split x = hi + lo with hi = tf32(x), lo = tf32(x - hi)
// (11 + 11 significant bits), and a product is hi*hi + hi*lo + lo*hi with FP32
// accumulation — the FP32 reference's accuracy (the dropped lo*lo term is
// ~2^-22 relative), at the legacy mma.sync rate (m16n8k8 TF32 measured 279
// TF/s on this part, so ~93 TF/s of FP32-equivalent work against 74 TF/s for the
// whole FP32 SIMT pipe). Weights are split once per optimizer step
// (split_kernel); activations / gradients are split when their fragments are
// read from shared memory.
//
//   tc_gemm<...>  C[i][j] = sum_k A(i,k) B(k,j) over a CTA tile of
//                 (16 WM WARPS_M) x (8 WN WARPS_N), k-tiles of 16 through a
//                 3-stage cp.async ring; epilogues: +bias ReLU (trunk forward),
//                 ReLU-mask (dIN, deform.cpp:305-324), +bias into the residual
//                 planes (heads), split-K partial (dW, reduced in fixed chunk
//                 order by dw_reduce_kernel in k_train.cu)
#include "swr_internal.h"

namespace swr
{

namespace
{
constexpr int TBK = 16, TSTAGES = 3;

// two segments along one axis (the [h | x] concatenation of skip layers) plus
// an optional ones column (the dW kernel's db) at index `ones`
struct Seg
{
    const float *p1, *p2;
    int ld1, ld2, n1, n; // p1 covers [0, n1), p2 [n1, n); index == ones -> 1.0
    int ones;
};

__device__ const float c_one_tc = 1.0f;

__device__ __forceinline__ const float *seg_ptr(const Seg &s, int64_t outer, int inner)
{
    return inner < s.n1 ? s.p1 + outer * s.ld1 + inner : s.p2 + outer * s.ld2 + (inner - s.n1);
}

__device__ __forceinline__ void cpa4(float *dst, const float *src, bool pred)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 4 : 0));
}

__device__ __forceinline__ uint32_t tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void split(float x, uint32_t &hi, uint32_t &lo)
{
    hi = tf32(x);
    lo = tf32(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma8(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct TcArgs
{
    int M, N, K;      // C is M x N, reduction over K (split into chunks of `chunk`)
    int chunk;
    // A(i, k): A_KM ? a.p1[k * lda + i] : seg(a, i, k)
    Seg a;
    // B(k, j): B_KN ? seg(b, k, j) : b.p1[j * ldb + k]; presplit: bhi/blo same layout
    Seg b;
    const float *bhi, *blo;
    const float *bias, *mask;
    int ldm;
    float *out;
    int64_t ldo;
};

// MODE 0 +bias ReLU -> out[i][j]; 1 * (mask[i][j] > 0) -> out[i][j];
//      2 +bias -> out[j * ldo + i] (planes); 3 partial -> out[(chunk * M + i) * N + j]
template <int WM, int WN, int WARPS_M, int WARPS_N, bool A_KM, bool B_KN, bool PRESPLIT, int MODE>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N) tc_gemm(TcArgs p)
{
    constexpr int BM = 16 * WM * WARPS_M, BN = 8 * WN * WARPS_N, NT = 32 * WARPS_M * WARPS_N;
    constexpr int LD = TBK + 4; // k-contiguous rows, conflict-free fragment reads
    constexpr int NB = PRESPLIT ? 2 : 1;
    extern __shared__ __align__(16) float tc_smem[];
    // As[TSTAGES][BM][LD], then Bs[TSTAGES][NB][BN][LD]
    auto As = reinterpret_cast<float(*)[BM][LD]>(tc_smem);
    auto Bs = reinterpret_cast<float(*)[NB][BN][LD]>(tc_smem + TSTAGES * BM * LD);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    const int gid = lane >> 2, tig = lane & 3;
    const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
    const int kb = blockIdx.z * p.chunk, ke = min(p.K, kb + p.chunk);
    float acc[WM][WN][4];
#pragma unroll
    for (int a = 0; a < WM; a++)
#pragma unroll
        for (int b = 0; b < WN; b++)
#pragma unroll
            for (int c = 0; c < 4; c++)
                acc[a][b][c] = 0.0f;

    auto issue = [&](int k0, int stg) {
        // A tile: BM x TBK
        for (int e = t; e < BM * TBK; e += NT)
        {
            int ii, kk;
            if (A_KM)
            {
                ii = e % BM; // consecutive threads -> consecutive i (contiguous in global)
                kk = e / BM;
            }
            else
            {
                kk = e % TBK;
                ii = e / TBK;
            }
            const int i = i0 + ii, k = k0 + kk;
            const bool ok = i < p.M && k < ke;
            const float *src = p.a.p1;
            if (ok)
                src = A_KM ? p.a.p1 + int64_t(k) * p.a.ld1 + i : seg_ptr(p.a, i, k);
            cpa4(&As[stg][ii][kk], src, ok);
        }
        // B tile: TBK x BN, stored [j][k]
        for (int e = t; e < BN * TBK; e += NT)
        {
            int jj, kk;
            if (B_KN)
            {
                jj = e % BN;
                kk = e / BN;
            }
            else
            {
                kk = e % TBK;
                jj = e / TBK;
            }
            const int j = j0 + jj, k = k0 + kk;
            const bool ok = j < p.N && k < ke;
            if (PRESPLIT)
            {
                // presplit weights are always stored [j][k] (B_KN false) or [k][j] single segment
                const int64_t off = B_KN ? int64_t(k) * p.b.ld1 + j : int64_t(j) * p.b.ld1 + k;
                cpa4(&Bs[stg][0][jj][kk], ok ? p.bhi + off : p.bhi, ok);
                cpa4(&Bs[stg][NB - 1][jj][kk], ok ? p.blo + off : p.blo, ok);
            }
            else
            {
                const float *src = p.b.p1;
                if (ok)
                    src = j == p.b.ones ? &c_one_tc : (B_KN ? seg_ptr(p.b, k, j) : p.b.p1 + int64_t(j) * p.b.ld1 + k);
                cpa4(&Bs[stg][0][jj][kk], src, ok);
            }
        }
    };

    const int nt = (ke - kb + TBK - 1) / TBK;
#pragma unroll
    for (int s = 0; s < TSTAGES - 1; s++)
    {
        if (s < nt)
            issue(kb + s * TBK, s);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int kt = 0; kt < nt; kt++)
    {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(TSTAGES - 2));
        __syncthreads();
        if (kt + TSTAGES - 1 < nt)
            issue(kb + (kt + TSTAGES - 1) * TBK, (kt + TSTAGES - 1) % TSTAGES);
        asm volatile("cp.async.commit_group;\n" ::);
        const int stg = kt % TSTAGES;
#pragma unroll
        for (int k8 = 0; k8 < TBK; k8 += 8)
        {
            uint32_t ah[WM][4], al[WM][4];
#pragma unroll
            for (int mt = 0; mt < WM; mt++)
            {
                const int r = (wm * WM + mt) * 16 + gid;
                split(As[stg][r][k8 + tig], ah[mt][0], al[mt][0]);
                split(As[stg][r + 8][k8 + tig], ah[mt][1], al[mt][1]);
                split(As[stg][r][k8 + tig + 4], ah[mt][2], al[mt][2]);
                split(As[stg][r + 8][k8 + tig + 4], ah[mt][3], al[mt][3]);
            }
#pragma unroll
            for (int n8 = 0; n8 < WN; n8++)
            {
                const int cidx = (wn * WN + n8) * 8 + gid;
                uint32_t bh0, bh1, bl0, bl1;
                if (PRESPLIT)
                {
                    bh0 = __float_as_uint(Bs[stg][0][cidx][k8 + tig]);
                    bh1 = __float_as_uint(Bs[stg][0][cidx][k8 + tig + 4]);
                    bl0 = __float_as_uint(Bs[stg][NB - 1][cidx][k8 + tig]);
                    bl1 = __float_as_uint(Bs[stg][NB - 1][cidx][k8 + tig + 4]);
                }
                else
                {
                    split(Bs[stg][0][cidx][k8 + tig], bh0, bl0);
                    split(Bs[stg][0][cidx][k8 + tig + 4], bh1, bl1);
                }
#pragma unroll
                for (int mt = 0; mt < WM; mt++)
                {
                    mma8(acc[mt][n8], al[mt], bh0, bh1);
                    mma8(acc[mt][n8], ah[mt], bl0, bl1);
                    mma8(acc[mt][n8], ah[mt], bh0, bh1);
                }
            }
        }
    }
    // epilogue
#pragma unroll
    for (int mt = 0; mt < WM; mt++)
#pragma unroll
        for (int n8 = 0; n8 < WN; n8++)
#pragma unroll
            for (int h = 0; h < 4; h++)
            {
                const int i = i0 + (wm * WM + mt) * 16 + gid + (h >= 2 ? 8 : 0);
                const int j = j0 + (wn * WN + n8) * 8 + 2 * tig + (h & 1);
                if (i >= p.M || j >= p.N)
                    continue;
                const float v = acc[mt][n8][h];
                if (MODE == 0)
                {
                    const float z = v + p.bias[j];
                    p.out[int64_t(i) * p.ldo + j] = z > 0.0f ? z : 0.0f;
                }
                else if (MODE == 1)
                    p.out[int64_t(i) * p.ldo + j] = p.mask[int64_t(i) * p.ldm + j] > 0.0f ? v : 0.0f;
                else if (MODE == 2)
                    p.out[int64_t(j) * p.ldo + i] = v + p.bias[j];
                else
                    p.out[(int64_t(blockIdx.z) * p.M + i) * p.N + j] = v;
            }
}

// w -> (tf32 hi, tf32 lo) for the presplit operand
__global__ void split_kernel(const float *__restrict__ w, int64_t n, float *__restrict__ hi, float *__restrict__ lo)
{
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    {
        uint32_t h, l;
        split(w[i], h, l);
        hi[i] = __uint_as_float(h);
        lo[i] = __uint_as_float(l);
    }
}

inline unsigned cdiv(int64_t a, int64_t b) { return unsigned((a + b - 1) / b); }

template <int WM, int WN, int WARPS_M, int WARPS_N, bool A_KM, bool B_KN, bool PRESPLIT, int MODE>
void run_tc(const TcArgs &p, dim3 grid, cudaStream_t st)
{
    constexpr int BM = 16 * WM * WARPS_M, BN = 8 * WN * WARPS_N, LD = TBK + 4, NB = PRESPLIT ? 2 : 1;
    constexpr size_t smem = sizeof(float) * TSTAGES * LD * (BM + NB * BN);
    auto kern = tc_gemm<WM, WN, WARPS_M, WARPS_N, A_KM, B_KN, PRESPLIT, MODE>;
    static bool configured = false;
    if (!configured)
    {
        check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                   "tc gemm smem attribute");
        configured = true;
    }
    kern<<<grid, 32 * WARPS_M * WARPS_N, smem, st>>>(p);
}
} // namespace

void launch_split_weights(Ctx &c, const float *w, int64_t n, float *hi, float *lo, cudaStream_t st)
{
    split_kernel<<<std::min<int64_t>(cdiv(n, 256), 148 * 4), 256, 0, st>>>(w, n, hi, lo);
    c.launches++;
}

// trunk forward: h = relu([a1 | a2] W^T + b); W presplit (whi/wlo [width][K])
void launch_dense_fwd_tc(Ctx &c, const float *a1, int ld1, int ka, const float *a2, int ld2, int K, const float *whi,
                         const float *wlo, const float *b, int width, float *h, cudaStream_t st)
{
    TcArgs p{};
    p.M = c.g.n;
    p.N = width;
    p.K = K;
    p.chunk = K;
    p.a = Seg{a1, a2, ld1, ld2, ka, K, -1};
    p.b = Seg{whi, nullptr, K, 0, K, K, -1};
    p.bhi = whi;
    p.blo = wlo;
    p.bias = b;
    p.out = h;
    p.ldo = width;
    run_tc<1, 10, 2, 2, false, false, true, 0>(p, dim3(cdiv(p.M, 32), cdiv(p.N, 160), 1), st);
    c.launches++;
}

// heads: planes[j][i] = h7[i] . Wh[j] + bh[j], j < 5
void launch_heads_fwd_tc(Ctx &c, const float *h7, int width, const float *whi, const float *wlo, const float *bh,
                         float *planes, int64_t plane, cudaStream_t st)
{
    TcArgs p{};
    p.M = c.g.n;
    p.N = 5;
    p.K = width;
    p.chunk = width;
    p.a = Seg{h7, nullptr, width, 0, width, width, -1};
    p.b = Seg{whi, nullptr, width, 0, width, width, -1};
    p.bhi = whi;
    p.blo = wlo;
    p.bias = bh;
    p.out = planes;
    p.ldo = plane;
    run_tc<1, 1, 4, 1, false, false, true, 2>(p, dim3(cdiv(p.M, 64), 1, 1), st);
    c.launches++;
}

// dZ_prev = (dZ W[:, :width]) * (h_prev > 0); W presplit [width][cols]
void launch_dense_bwd_input_tc(Ctx &c, const float *dz, int width, const float *whi, const float *wlo, int cols,
                               const float *h_prev, float *dz_prev, cudaStream_t st)
{
    TcArgs p{};
    p.M = c.g.n;
    p.N = width;
    p.K = width;
    p.chunk = width;
    p.a = Seg{dz, nullptr, width, 0, width, width, -1};
    p.b = Seg{whi, nullptr, cols, 0, width, width, -1};
    p.bhi = whi;
    p.blo = wlo;
    p.mask = h_prev;
    p.ldm = width;
    p.out = dz_prev;
    p.ldo = width;
    run_tc<1, 10, 2, 2, false, true, true, 1>(p, dim3(cdiv(p.M, 32), cdiv(p.N, 160), 1), st);
    c.launches++;
}

// split-K partials of dW [R][K+1] = dZ^T [a1 | a2 | 1] over row chunks
void launch_dense_bwd_weights_tc(Ctx &c, const float *dz, int R, const float *a1, int ld1, int ka, const float *a2,
                                 int ld2, int K, int chunk, float *part, cudaStream_t st)
{
    TcArgs p{};
    p.M = R;
    p.N = K + 1;
    p.K = c.g.n;
    p.chunk = chunk;
    p.a = Seg{dz, nullptr, R, 0, R, R, -1};
    p.b = Seg{a1, a2, ld1, ld2, ka, K, K};
    p.out = part;
    const unsigned chunks = cdiv(c.g.n, chunk);
    if (R <= 16)
        run_tc<1, 2, 1, 4, true, true, false, 3>(p, dim3(1, cdiv(p.N, 64), chunks), st);
    else if (R <= 160)
        run_tc<5, 4, 2, 2, true, true, false, 3>(p, dim3(cdiv(R, 160), cdiv(p.N, 64), chunks), st);
    else
        throw std::invalid_argument("training supports deform-net widths up to 160");
    c.launches++;
}

} // namespace swr
