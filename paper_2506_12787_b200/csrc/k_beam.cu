// Beam scan: the synthetic-data generator's
// dense step — for every sample the K-element phase-only channel is steered
// over every grid cell,
//   A(cell) = (1/K) sum_k w_k(cell) u_k,  w = e^{-j phase_shift}, u = h/|h|
// (sim::beam_scan, wavesim.cpp:213-252), batched over samples, plus
// generate_dataset's target post-processing (dataset.cpp:86-124): magnitude,
// one global normalization, float targets with a zero imaginary channel.
//
//   steering table  built once per (array, grid) on the host exactly like
//                   build_steering_table (wavesim.cpp:183-211: glibc cos/sin of
//                   the wrapped phase), uploaded as [cells][K] (wr, wi)
//   beam_scan_kernel  CTA = 128 cells x 8 samples; a thread keeps its cell's K
//                   weights in registers and walks the samples' unit channels
//                   (shared memory); double arithmetic in the reference's order
//                   (products, difference, running sum, then * 1/K), explicit
//                   _rn intrinsics so no FMA is contracted: bit-identical to the
//                   reference compiled without contraction
//   mag_max_kernel  |A| per cell (double, hypot) + a fixed-order per-CTA max;
//                   max_reduce_kernel -> the dataset normalization
//   target_kernel   float(|A| / normalization), imaginary 0
// The phase-only channel u = h/|h| (16 hypot per sample) is formed on the host
// with the reference's own formula, so the device sees identical inputs.
#include "swr.h"
#include "swr_internal.h"

#include <cmath>
#include <memory>
#include <stdexcept>
#include <vector>

namespace swr
{

namespace
{
constexpr int kMaxK = 64;        // elements per array supported by the kernel (8 x 8)
constexpr int kCells = 128;      // cells per CTA (one per thread)
constexpr int kSamples = 8;      // samples per CTA

template <int K>
__global__ void __launch_bounds__(kCells) beam_scan_kernel(const double *__restrict__ wr, const double *__restrict__ wi,
                                                           const double2 *__restrict__ u, int cells, int64_t B,
                                                           double inv_k, double2 *__restrict__ out)
{
    __shared__ double2 su[kSamples][K];
    const int cell = blockIdx.x * kCells + threadIdx.x;
    const int64_t s0 = (int64_t)blockIdx.y * kSamples;
    for (int i = threadIdx.x; i < kSamples * K; i += kCells)
    {
        const int64_t s = s0 + i / K;
        su[i / K][i % K] = s < B ? u[s * K + i % K] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (cell >= cells)
        return;
    double r[K], m[K];
#pragma unroll
    for (int e = 0; e < K; e++)
    {
        r[e] = wr[(int64_t)cell * K + e];
        m[e] = wi[(int64_t)cell * K + e];
    }
    for (int j = 0; j < kSamples; j++)
    {
        const int64_t s = s0 + j;
        if (s >= B)
            break;
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int e = 0; e < K; e++)
        {
            const double2 v = su[j][e];
            // ar += wr*ur - wi*ui; ai += wr*ui + wi*ur (wavesim.cpp:243-246)
            ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(r[e], v.x), __dmul_rn(m[e], v.y)));
            ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(r[e], v.y), __dmul_rn(m[e], v.x)));
        }
        out[s * cells + cell] = make_double2(__dmul_rn(ar, inv_k), __dmul_rn(ai, inv_k));
    }
}

// |A| per cell and the max over a CTA's cells
__global__ void __launch_bounds__(256) mag_max_kernel(const double2 *__restrict__ a, int64_t total,
                                                      double *__restrict__ mag, double *__restrict__ part)
{
    __shared__ double sm[256];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double m = 0.0;
    if (i < total)
    {
        const double2 v = a[i];
        m = hypot(v.x, v.y);
        mag[i] = m;
    }
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1)
    {
        if ((int)threadIdx.x < o)
            sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        part[blockIdx.x] = sm[0];
}

__global__ void max_reduce_kernel(const double *__restrict__ part, int64_t n, double *__restrict__ out)
{
    __shared__ double sm[1024];
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        m = fmax(m, part[i]);
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1)
    {
        if ((int)threadIdx.x < o)
            sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[0] = sm[0] > 0.0 ? sm[0] : 1.0; // dataset.cpp:97: 1 when every magnitude is 0
}

__global__ void target_kernel(const double *__restrict__ mag, int64_t total, const double *__restrict__ norm,
                              float2 *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total)
        out[i] = make_float2((float)__ddiv_rn(mag[i], norm[0]), 0.0f);
}

inline int64_t blocks64(int64_t n, int t) { return (n + t - 1) / t; }
} // namespace

// element_layout (wavesim.cpp:22-35) + phase_shift (wavesim.cpp:37-44)
static void steering_host(int k, double spacing, double wavelength, int H, int W, std::vector<double> &wr,
                          std::vector<double> &wi)
{
    if (k < 1)
        throw std::invalid_argument("k_elements must be >= 1");
    const int side = int(std::lround(std::sqrt(double(k))));
    if (side * side != k)
        throw std::invalid_argument("k_elements must be a perfect square");
    if (H < 1 || W < 1)
        throw std::invalid_argument("empty angular grid");
    std::vector<double> er, eb;
    for (int m = 1; m <= side; m++)
        for (int n = 1; n <= side; n++)
        {
            er.push_back(spacing * std::sqrt(double((m - 1) * (m - 1) + (n - 1) * (n - 1))));
            eb.push_back(std::atan2(double(m - 1), double(n - 1)));
        }
    const double cel = (kPi / 2.0) / H, caz = (2.0 * kPi) / W; // spectrum.cpp:29-32
    wr.resize(size_t(H) * W * k);
    wi.resize(wr.size());
    for (int i = 0; i < H; i++)
    {
        const double el = (i + 0.5) * cel;
        for (int j = 0; j < W; j++)
        {
            const double az = (j + 0.5) * caz;
            const size_t base = (size_t(i) * W + j) * k;
            for (int e = 0; e < k; e++)
            {
                const double raw = -2.0 * kPi * er[e] * std::cos(az - eb[e]) * std::cos(el) / wavelength;
                double a = std::fmod(raw, 2.0 * kPi);
                if (a < 0.0)
                    a += 2.0 * kPi;
                wr[base + e] = std::cos(a);
                wi[base + e] = -std::sin(a); // w = e^{-j a}
            }
        }
    }
}

} // namespace swr

using namespace swr;

struct swr_steering
{
    int device = 0, k = 0, H = 0, W = 0;
    cudaStream_t stream = nullptr;
    double *wr = nullptr, *wi = nullptr;
    ~swr_steering()
    {
        cudaSetDevice(device);
        cudaFree(wr);
        cudaFree(wi);
        if (stream)
            cudaStreamDestroy(stream);
    }
};

namespace
{
// u = h/|h| per element, 1 for a zero entry (wavesim.cpp:222-236)
std::vector<double> unit_channels(const double *channel, int64_t B, int k)
{
    std::vector<double> u(size_t(B) * k * 2);
    for (int64_t i = 0; i < B * k; i++)
    {
        const double re = channel[2 * i], im = channel[2 * i + 1];
        const double mag = std::hypot(re, im); // std::abs(std::complex<double>)
        if (mag == 0.0)
        {
            u[2 * i] = 1.0;
            u[2 * i + 1] = 0.0;
        }
        else
        {
            u[2 * i] = re / mag;
            u[2 * i + 1] = im / mag;
        }
    }
    return u;
}

template <class T>
T *dmalloc(size_t n)
{
    void *p = nullptr;
    check_cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    return static_cast<T *>(p);
}

void launch_scan(swr_steering *st, const double2 *d_u, int64_t B, double2 *d_out)
{
    const int cells = st->H * st->W;
    dim3 grid(unsigned((cells + kCells - 1) / kCells), unsigned((B + kSamples - 1) / kSamples));
    const double inv_k = 1.0 / double(st->k);
    switch (st->k)
    {
    case 1: beam_scan_kernel<1><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 4: beam_scan_kernel<4><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 9: beam_scan_kernel<9><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 16: beam_scan_kernel<16><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 25: beam_scan_kernel<25><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 36: beam_scan_kernel<36><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 49: beam_scan_kernel<49><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    case 64: beam_scan_kernel<64><<<grid, kCells, 0, st->stream>>>(st->wr, st->wi, d_u, cells, B, inv_k, d_out); break;
    default: throw std::invalid_argument("beam scan supports square arrays up to 8 x 8 elements");
    }
    check_cuda(cudaGetLastError(), "beam scan launch");
}
} // namespace

extern "C" {

int swr_steering_create(int32_t k_elements, double spacing, double wavelength, int32_t H, int32_t W, int device,
                        swr_steering **out)
{
    return swr_guarded([&] {
        if (!out)
            throw std::invalid_argument("null argument");
        if (k_elements > kMaxK)
            throw std::invalid_argument("beam scan supports square arrays up to 8 x 8 elements");
        std::vector<double> wr, wi;
        steering_host(k_elements, spacing, wavelength, H, W, wr, wi);
        auto st = std::make_unique<swr_steering>();
        if (device < 0)
            check_cuda(cudaGetDevice(&device), "cudaGetDevice");
        st->device = device;
        check_cuda(cudaSetDevice(device), "cudaSetDevice");
        check_cuda(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking), "stream");
        st->k = k_elements;
        st->H = H;
        st->W = W;
        st->wr = dmalloc<double>(wr.size());
        st->wi = dmalloc<double>(wi.size());
        check_cuda(cudaMemcpy(st->wr, wr.data(), sizeof(double) * wr.size(), cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(st->wi, wi.data(), sizeof(double) * wi.size(), cudaMemcpyHostToDevice), "H2D");
        *out = st.release();
    });
}

void swr_steering_destroy(swr_steering *st) { delete st; }

int swr_steering_table(swr_steering *st, double *wr, double *wi)
{
    return swr_guarded([&] {
        check_cuda(cudaSetDevice(st->device), "cudaSetDevice");
        const size_t n = size_t(st->H) * st->W * st->k;
        if (wr)
            check_cuda(cudaMemcpy(wr, st->wr, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
        if (wi)
            check_cuda(cudaMemcpy(wi, st->wi, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

int swr_beam_scan_device(swr_steering *st, const double *d_unit, int64_t B, double *d_spectra, void *stream)
{
    return swr_guarded([&] {
        if (B < 0)
            throw std::invalid_argument("negative batch");
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(st->device), "cudaSetDevice");
        cudaStream_t keep = st->stream;
        if (stream)
            st->stream = static_cast<cudaStream_t>(stream);
        try
        {
            launch_scan(st, reinterpret_cast<const double2 *>(d_unit), B, reinterpret_cast<double2 *>(d_spectra));
        }
        catch (...)
        {
            st->stream = keep;
            throw;
        }
        st->stream = keep;
    });
}

int swr_beam_scan(swr_steering *st, const double *channel, int64_t B, double *spectra)
{
    return swr_guarded([&] {
        if (B < 0)
            throw std::invalid_argument("negative batch");
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(st->device), "cudaSetDevice");
        const std::vector<double> u = unit_channels(channel, B, st->k);
        const size_t cells = size_t(st->H) * st->W;
        // batches of samples bounded to ~1 GB of output per pass
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, (int64_t(1) << 30) / int64_t(16 * cells)));
        double *d_u = dmalloc<double>(size_t(chunk) * st->k * 2);
        double *d_out = dmalloc<double>(size_t(chunk) * cells * 2);
        try
        {
            for (int64_t b0 = 0; b0 < B; b0 += chunk)
            {
                const int64_t nb = std::min(chunk, B - b0);
                check_cuda(cudaMemcpyAsync(d_u, u.data() + size_t(b0) * st->k * 2, sizeof(double) * nb * st->k * 2,
                                           cudaMemcpyHostToDevice, st->stream),
                           "H2D channels");
                launch_scan(st, reinterpret_cast<const double2 *>(d_u), nb, reinterpret_cast<double2 *>(d_out));
                check_cuda(cudaMemcpyAsync(spectra + size_t(b0) * cells * 2, d_out, sizeof(double) * nb * cells * 2,
                                           cudaMemcpyDeviceToHost, st->stream),
                           "D2H spectra");
            }
            check_cuda(cudaStreamSynchronize(st->stream), "beam scan");
        }
        catch (...)
        {
            cudaFree(d_u);
            cudaFree(d_out);
            throw;
        }
        cudaFree(d_u);
        cudaFree(d_out);
    });
}

int swr_beam_scan_targets(swr_steering *st, const double *channel, int64_t B, float *targets, double *normalization)
{
    return swr_guarded([&] {
        if (B < 1)
            throw std::invalid_argument("no samples to scan");
        check_cuda(cudaSetDevice(st->device), "cudaSetDevice");
        const std::vector<double> u = unit_channels(channel, B, st->k);
        const int64_t cells = int64_t(st->H) * st->W, total = cells * B;
        const int64_t nblk = blocks64(total, 256);
        double *d_u = nullptr, *d_m = nullptr, *d_part = nullptr;
        double2 *d_a = nullptr;
        float2 *d_t = nullptr;
        auto release = [&] {
            for (void *p : {(void *)d_u, (void *)d_a, (void *)d_m, (void *)d_part, (void *)d_t})
                cudaFree(p);
        };
        try
        {
            d_u = dmalloc<double>(u.size());
            d_a = dmalloc<double2>(size_t(total));
            d_m = dmalloc<double>(size_t(total));
            d_part = dmalloc<double>(size_t(nblk) + 1);
            d_t = dmalloc<float2>(size_t(total));
            check_cuda(cudaMemcpyAsync(d_u, u.data(), sizeof(double) * u.size(), cudaMemcpyHostToDevice, st->stream),
                       "H2D");
            launch_scan(st, reinterpret_cast<const double2 *>(d_u), B, d_a);
            mag_max_kernel<<<unsigned(nblk), 256, 0, st->stream>>>(d_a, total, d_m, d_part);
            max_reduce_kernel<<<1, 1024, 0, st->stream>>>(d_part, nblk, d_part + nblk);
            target_kernel<<<unsigned(nblk), 256, 0, st->stream>>>(d_m, total, d_part + nblk, d_t);
            check_cuda(cudaGetLastError(), "targets");
            check_cuda(cudaMemcpyAsync(targets, d_t, sizeof(float2) * total, cudaMemcpyDeviceToHost, st->stream), "D2H");
            if (normalization)
                check_cuda(cudaMemcpyAsync(normalization, d_part + nblk, sizeof(double), cudaMemcpyDeviceToHost,
                                           st->stream),
                           "D2H");
            check_cuda(cudaStreamSynchronize(st->stream), "targets");
        }
        catch (...)
        {
            release();
            throw;
        }
        release();
    });
}

} // extern "C"
