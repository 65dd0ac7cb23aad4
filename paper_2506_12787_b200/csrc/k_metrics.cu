// Batched evaluation metrics: PSNR, SSIM, L1 of rendered spectra against
// targets (spectrum.cpp:145-250), the consumer of the render path in
// train::evaluate (training.cpp:380-406). All statistics in double like the
// reference ("float/double instantiations agree to roundoff", spectrum.cpp:176).
//
//   metrics_part_kernel   one CTA per (pair, 1024-float chunk): sum (a-b)^2 and
//                         |a-b|; counts non-finite inputs (the reference throws
//                         domain_error, spectrum.cpp:44-49)
//   metrics_final_kernel  per pair, the chunk sums in order -> PSNR (clamped at
//                         100 dB) and L1
//   ssim_fused_kernel     one CTA per (pair, channel, 32 x 64 block of windows):
//                         the input block and its 11-tap horizontal correlations
//                         of x, y, x^2, y^2, xy stay in shared memory, then the
//                         vertical taps, the per-window SSIM, a fixed-order sum
//   ssim_fused_final      mean over windows, average of the two channels
//   ssim_h_kernel         (hybrid loss) one CTA per (pair, channel, row): the
//                         horizontal correlations into a global buffer the
//                         gradient's adjoint pass reads back
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

constexpr int kPtChunk = 1024; // floats per partial of the point metrics
inline int pt_chunks(int64_t n) { return (int)((n + kPtChunk - 1) / kPtChunk); }

// (sum (a-b)^2, sum |a-b|) of one chunk of one pair, fixed-order block sums
__global__ void __launch_bounds__(256) metrics_part_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                           int64_t n, int chunks, double2 *__restrict__ part,
                                                           int *__restrict__ bad)
{
    __shared__ double sh[32];
    const int64_t s = blockIdx.y;
    const int64_t lo = (int64_t)blockIdx.x * kPtChunk, hi = min(n, lo + kPtChunk);
    const float *x = a + s * n, *y = b + s * n;
    double sq = 0.0, ab = 0.0;
    int nf = 0;
    for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x)
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
        part[s * chunks + blockIdx.x] = make_double2(sq, ab);
    }
}

// per pair: chunk partials in ascending order -> PSNR (clamped at 100 dB) and L1
__global__ void metrics_final_kernel(const double2 *__restrict__ part, int chunks, int nb, int64_t n, double peak,
                                     double *__restrict__ psnr, double *__restrict__ l1)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nb)
        return;
    double sq = 0.0, ab = 0.0;
    for (int c = 0; c < chunks; c++)
    {
        const double2 v = part[(int64_t)s * chunks + c];
        sq += v.x;
        ab += v.y;
    }
    const double mse = sq / (double)n;
    if (psnr)
        psnr[s] = mse <= 0.0 ? 100.0 : fmin(100.0, 10.0 * log10(peak * peak / mse));
    if (l1)
        l1[s] = ab / (double)n;
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

// Fused SSIM of one (pair, channel, 32-row x 64-column block of windows): the
// input window block (42 x 74 cells, double) and its horizontal 11-tap
// correlations (5 quantities x 42 rows x 64 columns) stay in shared memory, so
// nothing round-trips through HBM. Per value the operation order is the same
// as the loss path's (horizontal then vertical taps, ascending, fma), so the
// window statistics are the same doubles; the block's sum is fixed-order.
constexpr int kFR = 32, kFC = 64;                       // windows per block (rows, columns)
constexpr int kFIR = kFR + kWin - 1, kFIC = kFC + kWin - 1; // input rows / columns per block
constexpr size_t kFusedSmem = sizeof(double) * (2 * kFIR * kFIC + 5 * kFIR * kFC + 32);

__global__ void __launch_bounds__(256) ssim_fused_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                         int H, int W, double peak, double *__restrict__ part)
{
    extern __shared__ double fsm[];
    double *xin = fsm, *yin = fsm + kFIR * kFIC; // [kFIR][kFIC]
    double *hq = yin + kFIR * kFIC;              // [5][kFIR][kFC]
    double *sh = hq + 5 * kFIR * kFC;            // [32]
    const int ct = blockIdx.x, rt = blockIdx.y;
    const int64_t sc = blockIdx.z; // pair * 2 + channel
    const int64_t s = sc >> 1;
    const int c = int(sc & 1);
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int i0 = rt * kFR, j0 = ct * kFC;
    const float *x = a + s * int64_t(H) * W * 2, *y = b + s * int64_t(H) * W * 2;
    for (int e = threadIdx.x; e < kFIR * kFIC; e += blockDim.x)
    {
        const int r = e / kFIC, cc = e % kFIC;
        const int gi = i0 + r, gj = j0 + cc;
        const bool ok = gi < H && gj < W;
        xin[e] = ok ? (double)x[(int64_t(gi) * W + gj) * 2 + c] : 0.0;
        yin[e] = ok ? (double)y[(int64_t(gi) * W + gj) * 2 + c] : 0.0;
    }
    __syncthreads();
    // horizontal correlations (ssim_h_kernel's order)
    for (int e = threadIdx.x; e < kFIR * kFC; e += blockDim.x)
    {
        const int r = e / kFC, jj = e % kFC;
        const double *xr = xin + r * kFIC + jj, *yr = yin + r * kFIC + jj;
        double mx = 0.0, my = 0.0, mxx = 0.0, myy = 0.0, mxy = 0.0;
#pragma unroll
        for (int t = 0; t < kWin; t++)
        {
            const double g = c_taps[t], xv = xr[t], yv = yr[t];
            mx = __fma_rn(g, xv, mx);
            my = __fma_rn(g, yv, my);
            mxx = __fma_rn(g, xv * xv, mxx);
            myy = __fma_rn(g, yv * yv, myy);
            mxy = __fma_rn(g, xv * yv, mxy);
        }
        hq[0 * kFIR * kFC + e] = mx;
        hq[1 * kFIR * kFC + e] = my;
        hq[2 * kFIR * kFC + e] = mxx;
        hq[3 * kFIR * kFC + e] = myy;
        hq[4 * kFIR * kFC + e] = mxy;
    }
    __syncthreads();
    // vertical taps + per-window SSIM
    const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
    double acc = 0.0;
    for (int e = threadIdx.x; e < kFR * kFC; e += blockDim.x)
    {
        const int ii = e / kFC, jj = e % kFC;
        if (i0 + ii >= vh || j0 + jj >= vw)
            continue;
        double m[5];
#pragma unroll
        for (int q = 0; q < 5; q++)
        {
            double v = 0.0;
#pragma unroll
            for (int t = 0; t < kWin; t++)
                v = __fma_rn(c_taps[t], hq[q * kFIR * kFC + (ii + t) * kFC + jj], v);
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
        part[(sc * gridDim.y + rt) * gridDim.x + ct] = acc;
}

// per pair: the blocks' sums in (channel, row block, column block) order -> mean SSIM
__global__ void ssim_fused_final_kernel(const double *__restrict__ part, int nb, int blocks, int64_t windows,
                                        double *__restrict__ ssim)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nb)
        return;
    double ch[2];
    for (int c = 0; c < 2; c++)
    {
        double t = 0.0;
        for (int k = 0; k < blocks; k++)
            t += part[((int64_t)s * 2 + c) * blocks + k];
        ch[c] = t / (double)windows;
    }
    ssim[s] = 0.5 * (ch[0] + ch[1]);
}


// ------------------------------------------------- hybrid loss + gradient
// training.cpp:62-106: loss = lambda1 * L1 + (1 - lambda1) * (1 - SSIM), and its
// gradient wrt the prediction; the SSIM gradient follows ssim_channel's
// f1/f2/f3 window terms scattered back with the adjoint correlation
// (spectrum.cpp:103-131, 209-235), all in double, rounded to float where the
// reference stores floats.

// per window: SSIM and the three gradient terms; F layout [pair][channel][3][vh][vw]
__global__ void __launch_bounds__(256) ssim_vgrad_kernel(const double *__restrict__ tmp, int H, int W,
                                                         double *__restrict__ part, double *__restrict__ F)
{
    __shared__ double sh[32];
    const int i = blockIdx.x, c = blockIdx.y;
    const int64_t s = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int64_t qs = (int64_t)H * vw, fs = (int64_t)vh * vw;
    const double *in = tmp + ((s * 2 + c) * 5) * qs;
    double *f = F + ((s * 2 + c) * 3) * fs + (int64_t)i * vw;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03; // peak 1 (training.cpp:79-80)
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
        const double sv = (a1 * a2) / (b1 * b2);
        acc += sv;
        f[j] = 2.0 * uy * (a2 - a1) / (b1 * b2) - 2.0 * sv * ux / b1 + 2.0 * sv * ux / b2;
        f[fs + j] = 2.0 * a1 / (b1 * b2);
        f[2 * fs + j] = -2.0 * sv / b2;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0)
        part[(s * 2 + c) * vh + i] = acc;
}

// adjoint correlation, horizontal: T[q][i][col] = sum_t g[t] F[q][i][col - t]
__global__ void __launch_bounds__(256) scatter_h_kernel(const double *__restrict__ F, int H, int W,
                                                        double *__restrict__ T)
{
    const int i = blockIdx.x, cq = blockIdx.y; // cq = channel * 3 + q
    const int64_t s = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const double *src = F + ((s * 6 + cq) * vh + i) * (int64_t)vw;
    double *dst = T + ((s * 6 + cq) * vh + i) * (int64_t)W;
    for (int col = threadIdx.x; col < W; col += blockDim.x)
    {
        double v = 0.0;
        for (int t = 0; t < kWin; t++) // scatter order: t ascending for a fixed column
        {
            const int j = col - t;
            if (j >= 0 && j < vw)
                v = __fma_rn(c_taps[t], src[j], v);
        }
        dst[col] = v;
    }
}

// adjoint, vertical, then the loss gradient per cell and channel
__global__ void __launch_bounds__(256) loss_grad_kernel(const double *__restrict__ T, const float *__restrict__ pred,
                                                        const float *__restrict__ target, int H, int W,
                                                        double lambda1, float *__restrict__ grad)
{
    const int r = blockIdx.x, c = blockIdx.y; // one CTA per (row, channel)
    const int64_t s = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const double inv_w = 1.0 / ((double)vh * vw);
    const double inv = lambda1 / (2.0 * H * W), sw = 0.5 * (1.0 - lambda1);
    for (int col = threadIdx.x; col < W; col += blockDim.x)
    {
        const int64_t k = ((s * H) + r) * (int64_t)W + col;
        double gq[3];
        for (int q = 0; q < 3; q++)
        {
            const double *src = T + ((s * 6 + c * 3 + q) * vh) * (int64_t)W;
            double v = 0.0;
            for (int t = kWin - 1; t >= 0; t--) // scatter order: source rows ascending
            {
                const int i = r - t;
                if (i >= 0 && i < vh)
                    v = __fma_rn(c_taps[t], src[(int64_t)i * W + col], v);
            }
            gq[q] = v;
        }
        const double x = (double)pred[2 * k + c], y = (double)target[2 * k + c];
        const float g_ssim = (float)((gq[0] + gq[1] * y + gq[2] * x) * inv_w); // ssim_channel's T grad
        const float d = pred[2 * k + c] - target[2 * k + c];
        const double sgn = d > 0.f ? 1.0 : (d < 0.f ? -1.0 : 0.0);
        grad[2 * k + c] = (float)(inv * sgn - sw * (double)g_ssim);
    }
}

__global__ void loss_final_kernel(const double *__restrict__ part, const double *__restrict__ l1v, int nb, int vh,
                                  int vw, double lambda1, double *__restrict__ terms)
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
    const double ssim = 0.5 * (ch[0] + ch[1]);
    const double l1t = lambda1 * l1v[s], st = (1.0 - lambda1) * (1.0 - ssim);
    terms[3 * s] = l1t + st;
    terms[3 * s + 1] = l1t;
    terms[3 * s + 2] = st;
}
} // namespace

// host: the window taps exactly as spectrum.cpp:51-70 computes them
static void upload_taps(int device)
{
    static DeviceOnce once;
    once.get(device, [] {
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
    return 1;
    });
}

size_t metrics_tmp_doubles(const Ctx &c, int nb)
{
    const int vw = std::max(c.g.W - kWin + 1, 0), vh = std::max(c.g.H - kWin + 1, 0); // no SSIM below 11x11
    const int chunks = pt_chunks((int64_t)2 * c.g.H * c.g.W);
    const size_t blocks = (size_t)((vw + kFC - 1) / kFC) * ((vh + kFR - 1) / kFR);
    return std::max<size_t>((size_t)nb * 2 * blocks + (size_t)nb * 2 * chunks, 1);
}

// d_out* may be null; d_tmp holds metrics_tmp_doubles(c, nb); d_bad counts
// spectra with a non-finite value (the caller raises domain_error)
void launch_metrics(Ctx &c, const float *d_pred, const float *d_target, int nb, double peak, double *d_psnr,
                    double *d_ssim, double *d_l1, double *d_tmp, int *d_bad, cudaStream_t st)
{
    upload_taps(c.device);
    const int H = c.g.H, W = c.g.W, vw = W - kWin + 1, vh = H - kWin + 1;
    const int64_t n = (int64_t)2 * H * W;
    const int chunks = pt_chunks(n);
    const int cbt = (std::max(vw, 0) + kFC - 1) / kFC, rbt = (std::max(vh, 0) + kFR - 1) / kFR;
    double *part = d_tmp;                                                       // [nb][2][rbt * cbt]
    double2 *pt = reinterpret_cast<double2 *>(d_tmp + (size_t)nb * 2 * cbt * rbt); // [nb][chunks]
    metrics_part_kernel<<<dim3(chunks, nb), 256, 0, st>>>(d_pred, d_target, n, chunks, pt, d_bad);
    metrics_final_kernel<<<(nb + 127) / 128, 128, 0, st>>>(pt, chunks, nb, n, peak, d_psnr, d_l1);
    c.launches += 2;
    if (!d_ssim)
        return;
    static DeviceOnce once;
    once.get(c.device, [] {
        check_cuda(cudaFuncSetAttribute(ssim_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kFusedSmem),
                   "ssim smem attribute");
        return 1;
    });
    ssim_fused_kernel<<<dim3(cbt, rbt, 2 * nb), 256, kFusedSmem, st>>>(d_pred, d_target, H, W, peak, part);
    ssim_fused_final_kernel<<<(nb + 127) / 128, 128, 0, st>>>(part, nb, cbt * rbt, (int64_t)vh * vw, d_ssim);
    c.launches += 2;
    check_cuda(cudaGetLastError(), "metrics kernels");
}

} // namespace swr

namespace swr
{
size_t loss_tmp_doubles(const Ctx &c, int nb)
{
    const int H = c.g.H, W = c.g.W, vw = std::max(W - kWin + 1, 0), vh = std::max(H - kWin + 1, 0);
    // h-correlations (5 q) | partial sums | F (3 q x windows) | adjoint rows (3 q x vh x W) | l1 per pair
    const int chunks = pt_chunks((int64_t)2 * H * W);
    return std::max<size_t>((size_t)nb * 2 * (5 * (size_t)H * vw + vh + 3 * (size_t)vh * vw + 3 * (size_t)vh * W) + nb + 1 +
                                (size_t)nb * 2 * chunks,
                            1);
}

// hybrid_loss (training.cpp:62-106) for nb pairs: terms [nb][3] = (loss, l1_term,
// ssim_term) in double, grad [nb][H][W][2] float (null: value only)
void launch_hybrid_loss(Ctx &c, const float *d_pred, const float *d_target, int nb, double lambda1, double *d_terms,
                        float *d_grad, double *d_tmp, int *d_bad, cudaStream_t st)
{
    upload_taps(c.device);
    const int H = c.g.H, W = c.g.W, vw = W - kWin + 1, vh = H - kWin + 1;
    const int64_t n = (int64_t)2 * H * W;
    double *hcor = d_tmp;
    double *part = hcor + (size_t)nb * 2 * 5 * H * vw;
    double *F = part + (size_t)nb * 2 * vh;
    double *T = F + (size_t)nb * 2 * 3 * vh * vw;
    double *l1v = T + (size_t)nb * 2 * 3 * vh * W;
    const int threads = std::min(256, ((std::max(std::max(vw, W), 32) + 31) / 32) * 32);
    const int chunks = pt_chunks(n);
    double2 *pt = reinterpret_cast<double2 *>(l1v + ((nb + 1) & ~1)); // 16-byte aligned
    metrics_part_kernel<<<dim3(chunks, nb), 256, 0, st>>>(d_pred, d_target, n, chunks, pt, d_bad);
    metrics_final_kernel<<<(nb + 127) / 128, 128, 0, st>>>(pt, chunks, nb, n, 1.0, nullptr, l1v);
    ssim_h_kernel<<<dim3(H, 2, nb), threads, 2 * W * sizeof(double), st>>>(d_pred, d_target, H, W, hcor);
    ssim_vgrad_kernel<<<dim3(vh, 2, nb), threads, 0, st>>>(hcor, H, W, part, F);
    loss_final_kernel<<<(nb + 127) / 128, 128, 0, st>>>(part, l1v, nb, vh, vw, lambda1, d_terms);
    c.launches += 5;
    if (d_grad)
    {
        scatter_h_kernel<<<dim3(vh, 6, nb), threads, 0, st>>>(F, H, W, T);
        loss_grad_kernel<<<dim3(H, 2, nb), threads, 0, st>>>(T, d_pred, d_target, H, W, lambda1, d_grad);
        c.launches += 2;
    }
    check_cuda(cudaGetLastError(), "hybrid loss kernels");
}
} // namespace swr
