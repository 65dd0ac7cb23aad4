#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin_a(long long cycles)
{
    extern __shared__ char sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles)
        ;
    if (threadIdx.x == 9999) sm[0] = 1;
}
__global__ void __cluster_dims__(2, 1, 1) spin_c(long long cycles)
{
    extern __shared__ char sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles)
        ;
    if (threadIdx.x == 9999) sm[0] = 1;
}
__global__ void spin_b(long long cycles)
{
    extern __shared__ char sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles)
        ;
    if (threadIdx.x == 9999) sm[0] = 1;
}
int main()
{
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case { int a_thr, a_smem, a_attr, b_thr, b_smem, b_carve; const char *name; int a_carve = -1; };
    Case cs[] = {
        {128, 0, 0, 128, 0, -1, "plain"},
        {128, 1024, 200000, 128, 1024, -1, "A attr 200KB (launch 1KB)"},
        {128, 1024, 200000, 128, 1024, 100, "A attr 200KB, B carveout 100"},
        {704, 195784, 200000, 128, 14336, 100, "A 704thr 191KB, B 14KB carve100"},
        {704, 195784, 200000, 128, 14336, -1, "A 704thr 191KB, B 14KB"},
        {704, 150000, 200000, 128, 14336, 100, "A 704thr 146KB, B 14KB carve100"},
        {512, 100000, 200000, 128, 14336, 100, "A 512thr 98KB, B 14KB carve100"},
        {704, 195784, 200000, 128, 14336, 100, "A 191KB carve100, B carve100", 100},
        {704, 195784, 200000, 128, 14336, -1, "A 191KB carve100, B default", 100},
        {704, 150000, 200000, 128, 14336, 100, "A 146KB carve100, B carve100", 100},
    };
    {
        // cluster kernel A (2-CTA clusters), 704 threads, 191 KB, carveout 100
        cudaFuncSetAttribute(spin_c, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(spin_c, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(spin_b, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
        cudaFuncSetAttribute(spin_b, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        cudaDeviceSynchronize();
        spin_c<<<148, 704, 195784, a>>>(10000000);
        spin_b<<<148, 128, 14336, b>>>(10000000);
        cudaDeviceSynchronize();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s: %.2f ms (%s) %s\n", "CLUSTER A 191KB carve100, B carve100", ms, ms < 7 ? "concurrent" : "serial",
               cudaGetErrorString(cudaGetLastError()));
    }
    for (auto &c : cs)
    {
        cudaFuncSetAttribute(spin_a, cudaFuncAttributeMaxDynamicSharedMemorySize, c.a_attr ? c.a_attr : 48 * 1024);
        cudaFuncSetAttribute(spin_b, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
        cudaFuncSetAttribute(spin_b, cudaFuncAttributePreferredSharedMemoryCarveout, c.b_carve);
        cudaFuncSetAttribute(spin_a, cudaFuncAttributePreferredSharedMemoryCarveout, c.a_carve);
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        cudaDeviceSynchronize();
        spin_a<<<148, c.a_thr, c.a_smem, a>>>(10000000);
        spin_b<<<148, c.b_thr, c.b_smem, b>>>(10000000);
        cudaDeviceSynchronize();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s: %.2f ms (%s) %s\n", c.name, ms, ms < 7 ? "concurrent" : "serial", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
