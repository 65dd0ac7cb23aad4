// Can a small kernel share SMs with a persistent 704-thread, ~191 KB-smem kernel?
#include <cstdio>
#include <cuda_runtime.h>
#include <unistd.h>
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int CL>
__global__ void big(unsigned long long *t, long long spin)
{
    extern __shared__ char sm[];
    if (threadIdx.x == 0 && blockIdx.x == 0)
        t[0] = gtime();
    long long t0 = clock64();
    while (clock64() - t0 < spin)
        ;
    sm[threadIdx.x] = 1;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        t[1] = gtime();
}
__global__ void __cluster_dims__(2, 1, 1) big_cl(unsigned long long *t, long long spin)
{
    extern __shared__ char sm[];
    if (threadIdx.x == 0 && blockIdx.x == 0)
        t[0] = gtime();
    long long t0 = clock64();
    while (clock64() - t0 < spin)
        ;
    sm[threadIdx.x] = 1;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        t[1] = gtime();
}
__global__ void small(unsigned long long *t)
{
    extern __shared__ char sm[];
    sm[threadIdx.x] = 1;
    if (threadIdx.x == 0)
        atomicMin(&t[2], gtime());
    if (threadIdx.x == 0)
        atomicMax(&t[3], gtime());
}
int main()
{
    unsigned long long *t, h[4];
    cudaMalloc(&t, 64);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    const int big_smem = 195784, small_smem = 14336;
    cudaFuncSetAttribute(big<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    cudaFuncSetAttribute(big_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    cudaFuncSetAttribute(small, cudaFuncAttributeMaxDynamicSharedMemorySize, small_smem);
    cudaFuncSetAttribute(small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (int mode = 0; mode < 5; mode++)
    {
        h[0] = h[1] = 0;
        h[2] = ~0ull;
        h[3] = 0;
        cudaMemcpy(t, h, 32, cudaMemcpyHostToDevice);
        const int threads = mode == 2 ? 512 : mode == 4 ? 128 : 704;
        const int smem = mode == 3 ? 150000 : mode == 4 ? 1024 : big_smem;
        if (mode == 1)
            big_cl<<<148, threads, smem, a>>>(t, 20000000);
        else
            big<0><<<148, threads, smem, a>>>(t, 20000000);
        usleep(2000);
        small<<<148 * 2, 128, small_smem, b>>>(t);
        cudaDeviceSynchronize();
        cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): big %.2f ms, small first start at %+.2f ms, last at %+.2f ms (relative to big start) %s\n",
               mode, mode == 1 ? "cluster" : mode == 2 ? "512 thr" : mode == 3 ? "150KB" : "plain",
               (h[1] - h[0]) / 1e6, ((long long)h[2] - (long long)h[0]) / 1e6, ((long long)h[3] - (long long)h[0]) / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
