// Batched evaluation metrics: PSNR, SSIM, L1 of rendered spectra against
// targets (spectrum.cpp:145-250), the consumer of the render path in
// train::evaluate (training.cpp:380-406). All statistics in double like the
// reference ("float/double instantiations agree to roundoff", spectrum.cpp:176).
//
//   metrics_point_kernel  one CTA per spectrum pair: sum (a-b)^2 and |a-b| over
//                         the 2*H*W floats -> PSNR (clamped at 100 dB) and L1;
//                         counts non-finite inputs (the reference throws
//                         domain_error, spectrum.cpp:44-49)
//   ssim_h_kernel         one CTA per (pair, channel, row): the 11-tap horizontal
//                         correlation of x, y, x^2, y^2, xy (valid columns)
//   ssim_v_kernel         one CTA per (pair, channel, valid row): vertical taps,
//                         the per-window SSIM, a fixed-order block sum
//   ssim_final_kernel     mean over windows, average of the two channels
// Every reduction has a fixed order, so the results are deterministic.
#include "swr_internal.h"

#include <cmath>

namespace swr
{

namespace
{
constexpr int kWin = 11;
__constant__ double c_taps[kWin];

// fixed-order block sum of a double (blockDim.x multiple of 32, <= 1024)
__device__ double block_sum(double v, double *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0)
        sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < nw; k++)
            t += sh[k];
    __syncthreads();
    return t; // valid in thread 0
}

__global__ void __launch_bounds__(512) metrics_point_kernel(const float *__restrict__ a, const float *__restrict__ b, int64_t n, double peak,
                                     double *__restrict__ psnr, double *__restrict__ l1, int *__restrict__ bad)
{
    __shared__ double sh[32];
    const int64_t s = blockIdx.x;
    const float *x = a + s * n, *y = b + s * n;
    double sq = 0.0, ab = 0.0;
    int nf = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x)
    {
        const float xv = x[k], yv = y[k];
        if (!isfinite(xv) || !isfinite(yv))
            nf++;
        const double d = (double)xv - (double)yv;
        sq = __fma_rn(d, d, sq);
        ab += fabs(d);
    }
    nf = __syncthreads_count(nf > 0);
    sq = block_sum(sq, sh);
    ab = block_sum(ab, sh);
    if (threadIdx.x == 0)
    {
        if (nf)
            atomicAdd(bad, 1);
        const double mse = sq / (double)n;
        if (psnr)
            psnr[s] = mse <= 0.0 ? 100.0 : fmin(100.0, 10.0 * log10(peak * peak / mse));
        if (l1)
            l1[s] = ab / (double)n;
    }
}

// tmp layout: [pair][channel][5 quantities][H][vw]
__global__ void __launch_bounds__(256) ssim_h_kernel(const float *__restrict__ a, const float *__restrict__ b, int H, int W,
                              double *__restrict__ tmp)
{
    extern __shared__ double row[]; // [2][W]: x, y of this row and channel
    const int i = blockIdx.x, c = blockIdx.y;
    const int64_t s = blockIdx.z;
    const int vw = W - kWin + 1;
    const float *x = a + (s * H + i) * (int64_t)W * 2, *y = b + (s * H + i) * (int64_t)W * 2;
    for (int j = threadIdx.x; j < W; j += blockDim.x)
    {
        row[j] = (double)x[2 * j + c];
        row[W + j] = (double)y[2 * j + c];
    }
    __syncthreads();
    double *out = tmp + ((s * 2 + c) * 5) * (int64_t)H * vw + (int64_t)i * vw;
    const int64_t qs = (int64_t)H * vw;
    for (int j = threadIdx.x; j < vw; j += blockDim.x)
    {
        double mx = 0.0, my = 0.0, mxx = 0.0, myy = 0.0, mxy = 0.0;
#pragma unroll
        for (int t = 0; t < kWin; t++)
        {
            const double g = c_taps[t], xv = row[j + t], yv = row[W + j + t];
            mx = __fma_rn(g, xv, mx);
            my = __fma_rn(g, yv, my);
            mxx = __fma_rn(g, xv * xv, mxx);
            myy = __fma_rn(g, yv * yv, myy);
            mxy = __fma_rn(g, xv * yv, mxy);
        }
        out[j] = mx;
        out[qs + j] = my;
        out[2 * qs + j] = mxx;
        out[3 * qs + j] = myy;
        out[4 * qs + j] = mxy;
    }
}

__global__ void __launch_bounds__(256) ssim_v_kernel(const double *__restrict__ tmp, int H, int W, double peak, double *__restrict__ part)
{
    __shared__ double sh[32];
    const int i = blockIdx.x, c = blockIdx.y;
    const int64_t s = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int64_t qs = (int64_t)H * vw;
    const double *in = tmp + ((s * 2 + c) * 5) * qs;
    const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
    double acc = 0.0;
    for (int j = threadIdx.x; j < vw; j += blockDim.x)
    {
        double m[5];
#pragma unroll
        for (int q = 0; q < 5; q++)
        {
            double v = 0.0;
#pragma unroll
            for (int t = 0; t < kWin; t++)
                v = __fma_rn(c_taps[t], in[q * qs + (int64_t)(i + t) * vw + j], v);
            m[q] = v;
        }
        const double ux = m[0], uy = m[1];
        const double vx = m[2] - ux * ux, vy = m[3] - uy * uy, vxy = m[4] - ux * uy;
        const double a1 = 2.0 * ux * uy + c1, a2 = 2.0 * vxy + c2;
        const double b1 = ux * ux + uy * uy + c1, b2 = vx + vy + c2;
        acc += (a1 * a2) / (b1 * b2);
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0)
        part[(s * 2 + c) * vh + i] = acc;
}

__global__ void ssim_final_kernel(const double *__restrict__ part, int nb, int vh, int vw, double *__restrict__ ssim)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nb)
        return;
    double ch[2];
    for (int c = 0; c < 2; c++)
    {
        double t = 0.0;
        for (int i = 0; i < vh; i++)
            t += part[((int64_t)s * 2 + c) * vh + i];
        ch[c] = t / ((double)vh * vw);
    }
    ssim[s] = 0.5 * (ch[0] + ch[1]);
}
} // namespace

// host: the window taps exactly as spectrum.cpp:51-70 computes them
static void upload_taps()
{
    static bool done = false;
    if (done)
        return;
    double g[kWin], sum = 0.0;
    for (int i = 0; i < kWin; i++)
    {
        const double d = i - kWin / 2;
        g[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
        sum += g[i];
    }
    for (double &v : g)
        v /= sum;
    check_cuda(cudaMemcpyToSymbol(c_taps, g, sizeof(g)), "ssim taps");
    done = true;
}

size_t metrics_tmp_doubles(const Ctx &c, int nb)
{
    const int vw = std::max(c.g.W - kWin + 1, 0), vh = std::max(c.g.H - kWin + 1, 0); // no SSIM below 11x11
    return std::max<size_t>((size_t)nb * 2 * 5 * c.g.H * vw + (size_t)nb * 2 * vh, 1);
}

// d_out* may be null; d_tmp holds metrics_tmp_doubles(c, nb); d_bad counts
// spectra with a non-finite value (the caller raises domain_error)
void launch_metrics(Ctx &c, const float *d_pred, const float *d_target, int nb, double peak, double *d_psnr,
                    double *d_ssim, double *d_l1, double *d_tmp, int *d_bad, cudaStream_t st)
{
    upload_taps();
    const int H = c.g.H, W = c.g.W, vw = W - kWin + 1, vh = H - kWin + 1;
    const int64_t n = (int64_t)2 * H * W;
    metrics_point_kernel<<<nb, 512, 0, st>>>(d_pred, d_target, n, peak, d_psnr, d_l1, d_bad);
    c.launches++;
    if (!d_ssim)
        return;
    double *part = d_tmp + (size_t)nb * 2 * 5 * H * vw;
    const int threads = std::min(256, ((std::max(vw, 32) + 31) / 32) * 32);
    ssim_h_kernel<<<dim3(H, 2, nb), threads, 2 * W * sizeof(double), st>>>(d_pred, d_target, H, W, d_tmp);
    ssim_v_kernel<<<dim3(vh, 2, nb), threads, 0, st>>>(d_tmp, H, W, peak, part);
    ssim_final_kernel<<<(nb + 127) / 128, 128, 0, st>>>(part, nb, vh, vw, d_ssim);
    c.launches += 3;
    check_cuda(cudaGetLastError(), "metrics kernels");
}

} // namespace swr
