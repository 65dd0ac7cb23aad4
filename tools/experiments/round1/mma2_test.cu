// CTA-pair (cta_group::2) UMMA check: layout of B across the pair, SS and TS
// forms, and throughput. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_12787_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>
#include <cmath>
#include "tc_ptx.cuh"
using namespace swr::tc;

constexpr int N = 160;

// A [256][16], B [160][16] bf16 bits; D [256][160]
// mode 0: CTA r holds B columns [r*N/2, (r+1)*N/2); mode 1: both hold all N
template <int TS>
__global__ void __cluster_dims__(2, 1, 1) pair_test(const uint16_t *A, const uint16_t *B, float *D, int mode)
{
    __shared__ __align__(1024) uint16_t a_s[128 * 16];
    __shared__ __align__(1024) uint16_t b_s[N * 16];
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // core-matrix layout: element (row, k) at ((k/8)*(rows/8) + row/8)*64 + (row%8)*8 + k%8
    for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x)
    {
        const int row = i / 16, k = i % 16;
        a_s[((k / 8) * 16 + row / 8) * 64 + (row % 8) * 8 + k % 8] = A[(rank * 128 + row) * 16 + k];
    }
    const int nb = mode == 0 ? N / 2 : N, n0 = mode == 0 ? rank * N / 2 : 0;
    for (int i = threadIdx.x; i < nb * 16; i += blockDim.x)
    {
        const int n = i / 16, k = i % 16;
        b_s[((k / 8) * (nb / 8) + n / 8) * 64 + (n % 8) * 8 + k % 8] = B[(n0 + n) * 16 + k];
    }
    if (threadIdx.x == 0)
    {
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc2<512>(&tslot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (TS && warp < 4)
    {
        // A into TMEM columns 256..263: lane = row, column c = k pair (2c, 2c+1)
        uint32_t r[16];
        const int row = warp * 32 + lane;
        for (int c = 0; c < 8; c++)
            r[c] = (uint32_t)A[(rank * 128 + row) * 16 + 2 * c] | ((uint32_t)A[(rank * 128 + row) * 16 + 2 * c + 1] << 16);
        for (int c = 8; c < 16; c++)
            r[c] = 0;
        tmem_st16(tmem + 256 + ((uint32_t)(warp * 32) << 16), r);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && warp == 0)
    {
        const uint32_t idesc = make_idesc(1, 256, N);
        const uint64_t db = make_desc(smem_u32(b_s), (nb / 8) * 128, 128);
        if (elect_one())
        {
            if (TS)
                mma2_f16_ts(tmem, tmem + 256, db, idesc, 0);
            else
                mma2_f16(tmem, make_desc(smem_u32(a_s), 16 * 128, 128), db, idesc, 0);
            mma2_commit(&done, 3);
        }
        __syncwarp();
    }
    mbar_wait_cluster(&done, 0);
    tc_fence_after();
    if (warp < 4)
    {
        const int row = rank * 128 + warp * 32 + lane;
        for (int c = 0; c < N; c += 16)
        {
            float v[16];
            tmem_ld16(tmem + c + ((uint32_t)(warp * 32) << 16), v);
            for (int i = 0; i < 16; i++)
                D[row * N + c + i] = v[i];
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

// throughput: leader issues batches of BATCH TS UMMAs (M=256, N), commit multicast per batch
template <int NN, int BATCH, int NACC, int RANDOM>
__global__ void __cluster_dims__(2, 1, 1) pair_bench(long long *out, int batches)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, empty[4];
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
    {
        mbar_init(&full, 1);
        for (int k = 0; k < 4; k++)
            mbar_init(&empty[k], 1);
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc2<512>(&tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (RANDOM)
    {
        // random bf16 data in B (shared) and the A region (TMEM), like real weights/activations
        uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
        uint32_t *w = reinterpret_cast<uint32_t *>(sm);
        for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x)
        {
            x = x * 1664525u + 1013904223u;
            const uint32_t h0 = 0x3c00u + ((x >> 8) & 0x3ff) - 0x200, h1 = 0x3c00u + ((x >> 20) & 0x3ff) - 0x200;
            w[i] = (h0 & 0xffff) | ((h1 ^ ((x & 1) << 15)) << 16);
        }
        fence_proxy_async_smem();
        uint32_t r[16];
        for (int c = 0; c < 512; c += 16)
        {
            for (int i = 0; i < 16; i++)
            {
                x = x * 1664525u + 1013904223u;
                r[i] = (0x3c00u + ((x >> 8) & 0x3ff) - 0x200) | ((0x3c00u + ((x >> 20) & 0x3ff) - 0x200) << 16);
            }
            tmem_st16(tmem + c + ((uint32_t)(warp * 32) << 16), r);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && warp == 0)
    {
        const uint32_t idesc = make_idesc(1, 256, NN);
        const uint64_t db = make_desc(smem_u32(sm) + 65536, (NN / 16) * 128, 128);
        long long t0 = clock64();
        for (int j = 0; j < batches; j++)
        {
            tc_fence_after();
            if (elect_one())
            {
#pragma unroll
                for (int k = 0; k < BATCH; k++)
                    mma2_f16_ts(tmem + NN * (k % NACC), tmem + 320 + 16 * (k % 8) + 8 * (k & 1), db + 16 * (k % 4), idesc,
                                (j | k) > 0);
                mma2_commit(&empty[j & 3], 3);
            }
            __syncwarp();
        }
        if (elect_one())
            mma2_commit(&full, 3);
        __syncwarp();
        mbar_wait(&full, 0);
        if (threadIdx.x == 0)
            out[blockIdx.x / 2] = clock64() - t0;
    }
    else
        mbar_wait_cluster(&full, 0);
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}


// the MLP kernel's hidden-layer issue pattern (no waits): per layer m, part 0
// (N=96, D = region m%3) then part 1 (N=64, D = region + P1OFF), 10 K steps x 3
template <int P1OFF, int ROT, int SPIN, int ACC = 0, int XC = 0, int CLW = 0, int STAMP = 0>
__global__ void __cluster_dims__(2, 1, 1) layer_bench(long long *out, int layers)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, empty[4], accb[4];
    __shared__ uint32_t tslot;
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
    {
        mbar_init(&full, 1);
        for (int k = 0; k < 4; k++)
        {
            mbar_init(&empty[k], 1);
            mbar_init(&accb[k], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0)
        tmem_alloc2<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (rank == 0 && warp == 0)
    {
        const uint32_t base = smem_u32(sm);
        long long t0 = clock64();
        int stage = 0;
        for (int m = 0; m < layers; m++)
        {
            const uint32_t dreg = tmem + (ROT ? (m % 3) * 160 : 0), areg = tmem + (ROT ? ((m + 2) % 3) * 160 : 320);
            for (int p = 0; p < 2; p++)
            {
                const uint32_t d = dreg + (p ? P1OFF : 0);
                const int np = p ? 64 : 96;
                const uint32_t idesc = make_idesc(1, 256, np);
                const uint32_t kb = np * 16, lbo = np / 2 / 8 * 128;
                if (XC && (m % 2 == 0))
                {
                    // xc products: A (128 x 48) from shared memory, 3 K steps x 3
                    tc_fence_after();
                    const uint32_t b = base + stage * 18432;
                    const uint32_t xa = base + 100 * 1024;
                    if (elect_one())
                    {
                        for (int kk = 0; kk < 3; kk++)
                        {
                            const uint32_t bk = b + kk * 2 * kb;
                            const uint64_t dbh = make_desc(bk, lbo, 128), dbl = make_desc(bk + kb, lbo, 128);
                            const uint64_t dah = make_desc(xa + 2 * kk * 2048, 2048, 128);
                            const uint64_t dal = make_desc(xa + 12288 + 2 * kk * 2048, 2048, 128);
                            mma2_f16(d, dah, dbh, idesc, kk > 0 ? 1u : 0u);
                            mma2_f16(d, dal, dbh, idesc, 1u);
                            mma2_f16(d, dah, dbl, idesc, 1u);
                        }
                        mma2_commit(&empty[stage & 3], 3);
                    }
                    __syncwarp();
                    stage = (stage + 1) % 5;
                }
                for (int kind = 1; kind <= 2; kind++)
                {
                    tc_fence_after();
                    if (STAMP && (threadIdx.x & 31) == 0)
                        out[1000 + (blockIdx.x * 8 + (m * 4 + p * 2 + kind) % 8)] = clock64();
                    const uint32_t b = base + stage * 18432;
                    if (elect_one())
                    {
                        const int nk = kind == 1 ? 6 : 4;
#pragma unroll 1
                        for (int kk = 0; kk < nk; kk++)
                        {
                            const uint32_t bk = b + kk * 2 * kb;
                            const uint64_t dbh = make_desc(bk, lbo, 128), dbl = make_desc(bk + kb, lbo, 128);
                            const uint32_t ahi = areg + 16 * ((kind == 1 ? 0 : 6) + kk);
                            mma2_f16_ts(d, ahi, dbh, idesc, (!XC || m % 2) && (kind == 1 && kk == 0) ? 0u : 1u);
                            mma2_f16_ts(d, ahi + 8, dbh, idesc, 1u);
                            mma2_f16_ts(d, ahi, dbl, idesc, 1u);
                        }
                        mma2_commit(&empty[stage & 3], 3);
                    }
                    __syncwarp();
                    stage = (stage + 1) % 5;
                }
                if (ACC)
                {
                    if (elect_one())
                        mma2_commit(&accb[(m & 1) * 2 + p], 3);
                    __syncwarp();
                }
            }
        }
        if (elect_one())
            mma2_commit(&full, 3);
        __syncwarp();
        mbar_wait(&full, 0);
        if (threadIdx.x == 0)
            out[blockIdx.x / 2] = clock64() - t0;
    }
    else if (!CLW)
        mbar_wait_cluster(&full, 0);
    tc_fence_before();
    cluster_sync();
    if (warp == 0)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

template <int P1OFF, int ROT, int SPIN = 3, int ACC = 0, int XC = 0, int CLW = 0, int STAMP = 0>
void run_layer(int pairs)
{
    long long *d, h[256];
    cudaMalloc(&d, sizeof(long long) * 4096);
    const int layers = 200;
    auto k = layer_bench<P1OFF, ROT, SPIN, ACC, XC, CLW, STAMP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    k<<<2 * pairs, 32 * (SPIN + 1), 150 * 1024>>>(d, layers);
    k<<<2 * pairs, 32 * (SPIN + 1), 150 * 1024>>>(d, layers);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * pairs, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < pairs; i++)
        avg += h[i];
    avg /= pairs;
    printf("layer pattern stamp=%d clw=%d xc=%d acc=%d spin=%d p1off=%d rot=%d: %7.1f cycles/layer (ideal 2400 / 2760 with xc) %s\n", STAMP, CLW, XC, ACC, SPIN, P1OFF, ROT, avg / layers,
           cudaGetErrorString(e));
    cudaFree(d);
}

// TMEM -> register bandwidth (tcgen05.ld 32x32b.x16 by LW warps), optionally while
// the leader runs TS UMMAs (M=256, N=96) in a loop
template <int LW, int WITH_MMA>
__global__ void __cluster_dims__(2, 1, 1) ldtm_bench(long long *out, float *sink, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, stop;
    __shared__ uint32_t tslot;
    __shared__ long long tl[32];
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0)
    {
        mbar_init(&full, 1);
        mbar_init(&stop, 1);
        fence_mbar_init();
    }
    if (warp == LW)
        tmem_alloc2<512>(&tslot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    volatile uint32_t *flag = reinterpret_cast<volatile uint32_t *>(sm + 200 * 1024 - 16);
    if (threadIdx.x == 0)
        *flag = 0;
    __syncthreads();
    if (warp == LW)
    {
        if (rank == 0 && WITH_MMA)
        {
            const uint32_t idesc = make_idesc(1, 256, 96);
            const uint64_t db = make_desc(smem_u32(sm), 768, 128);
            int j = 0;
            while (*flag == 0 && j < 100000)
            {
                if (elect_one())
                {
#pragma unroll
                    for (int k = 0; k < 12; k++)
                        mma2_f16_ts(tmem + 320 + 96 * (k & 1) * 0, tmem + 160 + 16 * (k % 8) + 8 * (k & 1), db, idesc, 1u);
                }
                __syncwarp();
                j++;
            }
            if (elect_one())
                mma2_commit(&full, 3);
            __syncwarp();
        }
        else if (WITH_MMA)
            ;
    }
    else if (warp < LW)
    {
        const uint32_t q = warp & 3;
        float acc = 0.f;
        long long t0 = clock64();
        for (int i = 0; i < iters; i++)
        {
            float v[16];
            tmem_ld16(tmem + ((q * 32) << 16) + 16 * ((warp >> 2) + 4 * (i & 1)) % 160, v);
            for (int c = 0; c < 16; c++)
                acc += v[c];
        }
        long long t1 = clock64();
        if (lane == 0)
            tl[warp] = t1 - t0;
        sink[blockIdx.x * 1024 + threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0)
    {
        *flag = 1;
        long long mx = 0;
        for (int w = 0; w < LW; w++)
            mx = tl[w] > mx ? tl[w] : mx;
        out[blockIdx.x] = mx;
    }
    __syncthreads();
    if (WITH_MMA && warp == LW)
    {
        if (rank == 0)
            mbar_wait(&full, 0);
        else
            mbar_wait_cluster(&full, 0);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == LW)
    {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
    }
}

template <int LW, int WITH_MMA>
void run_ldtm(int pairs)
{
    long long *d, h[512];
    float *sink;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&sink, 2 * pairs * 1024 * 4);
    const int iters = 256;
    auto k = ldtm_bench<LW, WITH_MMA>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<2 * pairs, 32 * (LW + 1), 200 * 1024>>>(d, sink, iters);
    k<<<2 * pairs, 32 * (LW + 1), 200 * 1024>>>(d, sink, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * 2 * pairs, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 2 * pairs; i++)
        avg += h[i];
    avg /= 2 * pairs;
    const double bytes = (double)LW * iters * 2048;
    printf("ldtm warps=%d mma=%d: %.1f B/cycle per SM %s\n", LW, WITH_MMA, bytes / avg, cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(sink);
}
static uint16_t bf(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7fff + ((u >> 16) & 1);
    return u >> 16;
}
static float fb(uint16_t h)
{
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

template <int NN, int BATCH, int NACC, int RANDOM = 0>
void run_bench(int pairs)
{
    long long *d, h[256];
    cudaMalloc(&d, sizeof(h));
    const int batches = 4000 / BATCH;
    auto k = pair_bench<NN, BATCH, NACC, RANDOM>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    k<<<2 * pairs, 128, 150 * 1024>>>(d, batches);
    k<<<2 * pairs, 128, 150 * 1024>>>(d, batches);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * pairs, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < pairs; i++)
        avg += h[i];
    avg /= pairs;
    printf("pair TS rnd=%d M=256 N=%3d nacc=%d batch=%2d: %6.1f cycles/MMA (ideal per-SM %5.1f) %s\n", RANDOM, NN, NACC, BATCH,
           avg / (batches * BATCH), 128.0 * NN / 256.0, cudaGetErrorString(e));
    cudaFree(d);
}

int main()
{
    std::vector<uint16_t> A(256 * 16), B(N * 16);
    srand(1);
    for (auto &x : A)
        x = bf((rand() % 2001 - 1000) / 1000.0f);
    for (auto &x : B)
        x = bf((rand() % 2001 - 1000) / 1000.0f);
    std::vector<float> ref(256 * N);
    for (int m = 0; m < 256; m++)
        for (int n = 0; n < N; n++)
        {
            double s = 0;
            for (int k = 0; k < 16; k++)
                s += (double)fb(A[m * 16 + k]) * fb(B[n * 16 + k]);
            ref[m * N + n] = (float)s;
        }
    uint16_t *dA, *dB;
    float *dD;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, ref.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    for (int ts = 0; ts < 2; ts++)
        for (int mode = 0; mode < 2; mode++)
        {
            cudaMemset(dD, 0, ref.size() * 4);
            if (ts)
                pair_test<1><<<2, 128>>>(dA, dB, dD, mode);
            else
                pair_test<0><<<2, 128>>>(dA, dB, dD, mode);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> out(ref.size());
            cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost);
            double err = 0;
            int bad = 0;
            for (size_t i = 0; i < out.size(); i++)
            {
                const double d = fabs(out[i] - ref[i]);
                err = fmax(err, d);
                bad += d > 1e-3;
            }
            printf("ts=%d mode=%d: max err %.3g bad %d (%s)\n", ts, mode, err, bad, cudaGetErrorString(e));
            if (e != cudaSuccess)
                return 1;
        }
    run_ldtm<4, 0>(74);
    run_ldtm<16, 0>(74);
    run_ldtm<16, 1>(74);
    run_ldtm<20, 1>(74);
    return 0;
}
