// Training kernels: the optimizer, the device
// refresh of the render scene after each step, and the deformation network's
// forward-with-activations / backward for one TX position over all primitives
// (train::train, training.cpp:198-376; deform_backward, deform.cpp:264-326).
//
//   gauss_adam_kernel  one thread per primitive: Adam on center_raw (coarse only),
//                      cholesky (+ the width floors of training.cpp:276-284),
//                      atten_logit and response (training.cpp:39-57), then
//                      re-materialises the primitive's SceneDev entries (the
//                      setup/raster/backward inputs built on the host by
//                      build_scene) with device tanhf/expf; centre-derived
//                      entries only while the centres train (coarse stage)
//   adam_flat_kernel   Adam over the network's flat parameter vector (all 22
//                      tensors share lr, betas and step count, training.cpp:366-373)
//   gemm_rows_kernel   Out[m][j] = epi(sum_k A(m,k) B(k,j)) over the n primitive
//                      rows: the trunk's forward (A = [h | x] segments, B = W^T,
//                      +bias, ReLU), the heads (+bias, written into the residual
//                      planes) and dIN = dZ W fused with the previous layer's ReLU
//                      mask (deform.cpp:305-324). (16 RPT) x (32 NT) tile, BK 16, FP32,
//                      3-stage cp.async ring; RPT picked so the busiest SM has the fewest rows
//   gemm_dw_kernel     dW = dZ^T [IN | 1] per row chunk (split-K sized for ~2 CTAs/SM; the appended
//                      ones column gives db), partials summed in ascending chunk
//                      order by dw_reduce_kernel: deterministic, no atomics
//   heads_bwd_kernel   dZ7 = (dR Wh) * (h7 > 0) in the reference's branch order
//                      (centre, response, attenuation; deform.cpp:283-293)
// All FP32 like the reference (T = float); summation orders differ from Eigen's.
#include "swr_internal.h"

namespace swr
{

// ------------------------------------------------------------------ optimizer

__device__ __forceinline__ void adam1(float &p, float g, float &m, float &v, const AdamHp &hp, double bc1,
                                      double bc2)
{
    const float b1 = float(hp.beta1), b2 = float(hp.beta2);
    m = b1 * m + (1.0f - b1) * g;
    v = b2 * v + (1.0f - b2) * g * g;
    const double mhat = double(m) / bc1, vhat = double(v) / bc2;
    p -= float(hp.lr * mhat / (sqrt(vhat) + hp.eps));
}

namespace
{

__global__ void gauss_adam_kernel(Grid g, SceneDev sd, GaussDev gp, AdamHp hp, TrainSched sc, int step_center,
                                  int step_rest, float floor_el, float floor_az)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= g.n)
        return;
    const double *bc = sc.bc + 6 * *sc.it; // (center bc1, bc2, rest bc1, bc2, net bc1, bc2)
    const double bc1_c = bc[0], bc2_c = bc[1], bc1 = bc[2], bc2 = bc[3];
    float cr[2] = {gp.center[2 * p], gp.center[2 * p + 1]};
    float ch[3] = {gp.chol[3 * p], gp.chol[3 * p + 1], gp.chol[3 * p + 2]};
    float at = gp.atten[p];
    float rs[2] = {gp.resp[2 * p], gp.resp[2 * p + 1]};
    if (step_center)
        for (int k = 0; k < 2; k++)
            adam1(cr[k], gp.g_center[2 * p + k], gp.m_center[2 * p + k], gp.v_center[2 * p + k], hp, bc1_c, bc2_c);
    if (step_rest)
    {
        // training.cpp:318-328 / 355-362: cholesky, project_widths, atten, response
        for (int k = 0; k < 3; k++)
            adam1(ch[k], gp.g_chol[3 * p + k], gp.m_chol[3 * p + k], gp.v_chol[3 * p + k], hp, bc1, bc2);
        ch[0] = fmaxf(ch[0], floor_el);
        ch[2] = fmaxf(ch[2], floor_az);
        adam1(at, gp.g_atten[p], gp.m_atten[p], gp.v_atten[p], hp, bc1, bc2);
        for (int k = 0; k < 2; k++)
            adam1(rs[k], gp.g_resp[2 * p + k], gp.m_resp[2 * p + k], gp.v_resp[2 * p + k], hp, bc1, bc2);
    }
    gp.center[2 * p] = cr[0];
    gp.center[2 * p + 1] = cr[1];
    for (int k = 0; k < 3; k++)
        gp.chol[3 * p + k] = ch[k];
    gp.atten[p] = at;
    gp.resp[2 * p] = rs[0];
    gp.resp[2 * p + 1] = rs[1];

    // the scene entries build_scene derives on the host (capi.cpp), same formulas
    // centres (and their chain-rule factors) only change in the coarse stage; the
    // fine stage keeps the host-derived (glibc tanhf) values set at its entry
    float4 bw = sd.bwd[p];
    if (step_center)
    {
        const float th_el = tanhf(cr[0]), th_az = tanhf(cr[1]);
        sd.el0[p] = float(kPi / 4) * (th_el + 1.0f);
        sd.az0[p] = float(kPi) * (th_az + 1.0f);
        bw.x = 1.0f - th_el * th_el;
        bw.y = 1.0f - th_az * th_az;
    }
    sd.delta0[p] = 1.0f / (1.0f + expf(-at));
    sd.re0[p] = rs[0];
    sd.im0[p] = rs[1];
    const float c1 = ch[0], l2 = ch[1], c3 = ch[2];
    const float l1 = c1 < 1e-4f ? 1e-4f : c1;
    const float l3 = c3 < 1e-4f ? 1e-4f : c3;
    const float det = l1 * l1 * l3 * l3;
    sd.shape[p] = make_float4((l2 * l2 + l3 * l3) / det, -l2 / (l1 * l3 * l3), 1.0f / (l3 * l3), 1.0f / l1);
    sd.inv_l3[p] = 1.0f / l3;
    sd.l2[p] = l2;
    sd.half[p] = make_double2(double(g.radius) * double(l1), double(g.radius) * sqrt(double(l2) * l2 + double(l3) * l3));
    sd.bwd[p] = make_float4(bw.x, bw.y, c1 >= 1e-4f ? 1.0f : 0.0f, c3 >= 1e-4f ? 1.0f : 0.0f);
}

__global__ void adam_flat_kernel(float *__restrict__ p, const float *__restrict__ gr, float *__restrict__ m,
                                 float *__restrict__ v, int64_t count, AdamHp hp, TrainSched sc)
{
    const double bc1 = sc.bc[6 * *sc.it + 4], bc2 = sc.bc[6 * *sc.it + 5];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    {
        float x = p[i], mm = m[i], vv = v[i];
        adam1(x, gr[i], mm, vv, hp, bc1, bc2);
        p[i] = x;
        m[i] = mm;
        v[i] = vv;
    }
}

// ------------------------------------------------------------- network GEMMs

constexpr int BK = 16, GT = 256;
__device__ const float c_one = 1.0f; // the dW kernel's appended ones column

// A(m, k): k < ka from a1 (row stride ld1), else from a2 (row stride ld2) up to kb
struct ASrc
{
    const float *a1, *a2;
    int ld1, ld2, ka, K;
};

__device__ __forceinline__ const float *a_ptr(const ASrc &a, int m, int k)
{
    return k < a.ka ? a.a1 + int64_t(m) * a.ld1 + k : a.a2 + int64_t(m) * a.ld2 + (k - a.ka);
}

// 4-byte cp.async, zero-filled when !pred (src must still be a valid address)
__device__ __forceinline__ void cp4(float *dst, const float *src, bool pred)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait()
{
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int STAGES = 3;

// mode 0: +bias, ReLU -> out[m][j]; 1: * (mask[m][j] > 0) -> out[m][j];
// 2: +bias -> planes out[j * plane + m]
// Tile 16 RPT rows x 32 NT columns, k-tiles of 16 through a 3-stage cp.async ring
// (two tiles in flight while one is consumed); thread = RPT rows x 2 NT columns.
template <int NT, bool KCONTIG_B, int MODE, int RPT>
__global__ void __launch_bounds__(GT) gemm_rows_kernel(ASrc a, const float *__restrict__ B, int sbk, int sbn, int M,
                                                       int N, const float *__restrict__ bias,
                                                       const float *__restrict__ mask, int ldm, float *__restrict__ out,
                                                       int64_t ldo)
{
    constexpr int BM = 16 * RPT, BN = 32 * NT, AS = BM + 4, BS = BN + 4;
    __shared__ __align__(16) float As[STAGES][BK][AS];
    __shared__ __align__(16) float Bs[STAGES][BK][BS];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int m0 = blockIdx.x * BM;
    float acc[RPT][2 * NT];
#pragma unroll
    for (int i = 0; i < RPT; i++)
#pragma unroll
        for (int j = 0; j < 2 * NT; j++)
            acc[i][j] = 0.0f;
    constexpr int AL = BM * BK / GT, BL = BK * BN / GT;
    auto issue = [&](int k0, int stg) {
#pragma unroll
        for (int i = 0; i < AL; i++)
        {
            const int e = t + GT * i, mm = e / BK, kk = e % BK;
            const int m = m0 + mm, k = k0 + kk;
            const bool ok = m < M && k < a.K;
            cp4(&As[stg][kk][mm], ok ? a_ptr(a, m, k) : a.a1, ok);
        }
#pragma unroll
        for (int i = 0; i < BL; i++)
        {
            const int e = t + GT * i;
            const int kk = KCONTIG_B ? e % BK : e / BN, jj = KCONTIG_B ? e / BK : e % BN;
            const int k = k0 + kk;
            const bool ok = k < a.K && jj < N;
            cp4(&Bs[stg][kk][jj], ok ? B + int64_t(k) * sbk + int64_t(jj) * sbn : B, ok);
        }
    };
    const int nt = (a.K + BK - 1) / BK;
#pragma unroll
    for (int sidx = 0; sidx < STAGES - 1; sidx++)
    {
        if (sidx < nt)
            issue(sidx * BK, sidx);
        cp_commit();
    }
    for (int kt = 0; kt < nt; kt++)
    {
        cp_wait<STAGES - 2>();
        __syncthreads(); // tile kt landed for every thread; stage (kt-1) % STAGES is free
        if (kt + STAGES - 1 < nt)
            issue((kt + STAGES - 1) * BK, (kt + STAGES - 1) % STAGES);
        cp_commit();
        const int stg = kt % STAGES;
#pragma unroll
        for (int kk = 0; kk < BK; kk++)
        {
            float ar[RPT];
#pragma unroll
            for (int i = 0; i < RPT; i++)
                ar[i] = As[stg][kk][ty * RPT + i];
#pragma unroll
            for (int jj = 0; jj < NT; jj++)
            {
                const float2 bv = *reinterpret_cast<const float2 *>(&Bs[stg][kk][tx * 2 + 32 * jj]);
#pragma unroll
                for (int i = 0; i < RPT; i++)
                {
                    acc[i][2 * jj] = fmaf(ar[i], bv.x, acc[i][2 * jj]);
                    acc[i][2 * jj + 1] = fmaf(ar[i], bv.y, acc[i][2 * jj + 1]);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; i++)
    {
        const int m = m0 + ty * RPT + i;
        if (m >= M)
            continue;
#pragma unroll
        for (int jj = 0; jj < NT; jj++)
#pragma unroll
            for (int h = 0; h < 2; h++)
            {
                const int j = tx * 2 + 32 * jj + h;
                if (j >= N)
                    continue;
                float v = acc[i][2 * jj + h];
                if (MODE == 0)
                {
                    v += bias[j];
                    out[int64_t(m) * ldo + j] = v > 0.0f ? v : 0.0f;
                }
                else if (MODE == 1)
                    out[int64_t(m) * ldo + j] = mask[int64_t(m) * ldm + j] > 0.0f ? v : 0.0f;
                else
                    out[int64_t(j) * ldo + m] = v + bias[j];
            }
    }
}

constexpr int DW_C = 64, DW_CHUNK_MIN = 64;

// P[chunk][r][c] = sum_{m in chunk} dZ[m][r] * IN(m, c), IN(m, K) = 1 (db).
// Tile: all R rows (<= 32 NTR) x 64 columns; thread = 2 NTR rows x 4 columns;
// k-tiles of 16 chunk rows through the same 3-stage cp.async ring.
template <int NTR>
__global__ void __launch_bounds__(GT) gemm_dw_kernel(const float *__restrict__ dz, int ldz, int R, ASrc in, int M,
                                                     int chunk, const float *__restrict__ ones, float *__restrict__ part)
{
    constexpr int RT = 32 * NTR;
    __shared__ __align__(16) float As[STAGES][BK][RT + 4];
    __shared__ __align__(16) float Bs[STAGES][BK][DW_C + 4];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int c0 = blockIdx.x * DW_C, ch = blockIdx.y;
    const int C = in.K + 1;
    const int mb = ch * chunk, me = min(M, mb + chunk);
    constexpr int AL = RT * BK / GT, BL = DW_C * BK / GT;
    float acc[2 * NTR][4];
#pragma unroll
    for (int i = 0; i < 2 * NTR; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
            acc[i][j] = 0.0f;
    auto issue = [&](int k0, int stg) {
#pragma unroll
        for (int i = 0; i < AL; i++)
        {
            const int e = t + GT * i, kk = e / RT, x = e % RT;
            const int m = k0 + kk;
            const bool ok = m < me && x < R;
            cp4(&As[stg][kk][x], ok ? dz + int64_t(m) * ldz + x : dz, ok);
        }
#pragma unroll
        for (int i = 0; i < BL; i++)
        {
            const int e = t + GT * i, kk = e / DW_C, x = e % DW_C;
            const int m = k0 + kk, c = c0 + x;
            const bool ok = m < me && c < C;
            cp4(&Bs[stg][kk][x], ok ? (c == in.K ? ones : a_ptr(in, m, c)) : ones, ok);
        }
    };
    const int nt = (me - mb + BK - 1) / BK;
#pragma unroll
    for (int sidx = 0; sidx < STAGES - 1; sidx++)
    {
        if (sidx < nt)
            issue(mb + sidx * BK, sidx);
        cp_commit();
    }
    for (int kt = 0; kt < nt; kt++)
    {
        cp_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < nt)
            issue(mb + (kt + STAGES - 1) * BK, (kt + STAGES - 1) % STAGES);
        cp_commit();
        const int stg = kt % STAGES;
#pragma unroll
        for (int kk = 0; kk < BK; kk++)
        {
            const float4 bv = *reinterpret_cast<const float4 *>(&Bs[stg][kk][tx * 4]);
            const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int i = 0; i < NTR; i++)
            {
                const float2 av = *reinterpret_cast<const float2 *>(&As[stg][kk][ty * 2 + 32 * i]);
#pragma unroll
                for (int j = 0; j < 4; j++)
                {
                    acc[2 * i][j] = fmaf(av.x, br[j], acc[2 * i][j]);
                    acc[2 * i + 1][j] = fmaf(av.y, br[j], acc[2 * i + 1][j]);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NTR; i++)
#pragma unroll
        for (int h = 0; h < 2; h++)
        {
            const int r = ty * 2 + 32 * i + h;
            if (r >= R)
                continue;
            const int c = c0 + tx * 4;
            float *dst = part + (int64_t(ch) * R + r) * C;
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (c + j < C)
                    dst[c + j] = acc[2 * i + h][j];
        }
}

// dW[r][c] (c < C-1) and db[r] (c == C-1) = sum over chunks in ascending order
__global__ void dw_reduce_kernel(const float *__restrict__ part, int chunks, int R, int C, float *__restrict__ dw,
                                 float *__restrict__ db)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= R * C)
        return;
    float s = 0.0f;
    for (int ch = 0; ch < chunks; ch++)
        s += part[int64_t(ch) * R * C + e];
    const int r = e / C, c = e % C;
    if (c == C - 1)
        db[r] = s;
    else
        dw[int64_t(r) * (C - 1) + c] = s;
}

// dZ7[m][k] = ((dc0 w0 + dc1 w1) + (dr0 w2 + dr1 w3) + da w4)[k] * (h7[m][k] > 0)
__global__ void heads_bwd_kernel(const float *__restrict__ d_center, const float *__restrict__ d_response,
                                 const float *__restrict__ d_atten, const float *__restrict__ wh_c,
                                 const float *__restrict__ wh_r, const float *__restrict__ wh_a,
                                 const float *__restrict__ h7, int n, int width, float *__restrict__ dz)
{
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e >= int64_t(n) * width)
        return;
    const int m = int(e / width), k = int(e % width);
    const float c = d_center[2 * m] * wh_c[k] + d_center[2 * m + 1] * wh_c[width + k];
    const float r = d_response[2 * m] * wh_r[k] + d_response[2 * m + 1] * wh_r[width + k];
    const float a = d_atten[m] * wh_a[k];
    const float v = (c + r) + a;
    dz[e] = h7[e] > 0.0f ? v : 0.0f;
}

// dR [n][5] view of the merge outputs for the heads' dW (centre 2, response 2, atten 1)
__global__ void pack_dr_kernel(const float *__restrict__ d_center, const float *__restrict__ d_response,
                               const float *__restrict__ d_atten, int n, float *__restrict__ dr)
{
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n)
        return;
    dr[5 * m + 0] = d_center[2 * m];
    dr[5 * m + 1] = d_center[2 * m + 1];
    dr[5 * m + 2] = d_response[2 * m];
    dr[5 * m + 3] = d_response[2 * m + 1];
    dr[5 * m + 4] = d_atten[m];
}

// input rows x[m] = [encode(centre_m) (static), encode(position)] (deform.cpp:157-168)
__global__ void penc_kernel(float *__restrict__ x, int n, int d, int dc, TrainSched sc, int dp)
{
    const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (e >= int64_t(n) * dp)
        return;
    const int m = int(e / dp), k = int(e % dp);
    x[int64_t(m) * d + dc + k] = sc.penc[*sc.it * dp + k];
}

// this iteration's training target (the drawn sample's spectrum) into a fixed buffer
__global__ void gather_target_kernel(const float4 *__restrict__ spectra, int64_t per4, TrainSched sc,
                                     float4 *__restrict__ out)
{
    const float4 *src = spectra + per4 * sc.idx[*sc.it];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per4; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = src[i];
}

// the loss-log row of this iteration, then advance the schedule cursor
__global__ void log_advance_kernel(const double *__restrict__ terms, double *__restrict__ log, TrainSched sc)
{
    const int64_t it = *sc.it;
    log[3 * it + 0] = terms[0];
    log[3 * it + 1] = terms[1];
    log[3 * it + 2] = terms[2];
    *sc.it = it + 1;
}

inline int blocks(int64_t n, int t) { return int((n + t - 1) / t); }

// rows per thread of gemm_rows_kernel: one CTA per SM in flight (128 regs x 256
// threads), so pick the tile height that minimises the rows of the busiest SM
inline int pick_rpt(int n)
{
    int best = 5, best_rows = 1 << 30;
    for (int r = 5; r >= 3; r--)
    {
        const int ctas = (n + 16 * r - 1) / (16 * r);
        const int rows = ((ctas + 147) / 148) * 16 * r;
        if (rows < best_rows)
        {
            best_rows = rows;
            best = r;
        }
    }
    return best;
}

template <int NT, bool KC, int MODE>
void launch_rows(int rpt, int n, const ASrc &a, const float *B, int sbk, int sbn, int N, const float *bias,
                 const float *mask, int ldm, float *out, int64_t ldo, cudaStream_t st)
{
    switch (rpt)
    {
    case 3:
        gemm_rows_kernel<NT, KC, MODE, 3><<<blocks(n, 48), GT, 0, st>>>(a, B, sbk, sbn, n, N, bias, mask, ldm, out, ldo);
        break;
    case 4:
        gemm_rows_kernel<NT, KC, MODE, 4><<<blocks(n, 64), GT, 0, st>>>(a, B, sbk, sbn, n, N, bias, mask, ldm, out, ldo);
        break;
    default:
        gemm_rows_kernel<NT, KC, MODE, 5><<<blocks(n, 80), GT, 0, st>>>(a, B, sbk, sbn, n, N, bias, mask, ldm, out, ldo);
        break;
    }
}

} // namespace

void launch_gauss_adam(Ctx &c, const GaussDev &gp, const AdamHp &hp, const TrainSched &sc, bool step_center,
                       bool step_rest, float floor_el, float floor_az, cudaStream_t st)
{
    if (c.g.n == 0)
        return;
    gauss_adam_kernel<<<blocks(c.g.n, 256), 256, 0, st>>>(c.g, c.s, gp, hp, sc, step_center, step_rest, floor_el,
                                                           floor_az);
    c.launches++;
}

void launch_adam_flat(Ctx &c, float *p, const float *g, float *m, float *v, int64_t count, const AdamHp &hp,
                      const TrainSched &sc, cudaStream_t st)
{
    if (count == 0)
        return;
    adam_flat_kernel<<<std::min<int64_t>(blocks(count, 256), 148 * 8), 256, 0, st>>>(p, g, m, v, count, hp, sc);
    c.launches++;
}

void launch_position_encoding(Ctx &c, float *x, int d, int dc, const TrainSched &sc, int dp, cudaStream_t st)
{
    penc_kernel<<<blocks(int64_t(c.g.n) * dp, 256), 256, 0, st>>>(x, c.g.n, d, dc, sc, dp);
    c.launches++;
}

void launch_gather_target(Ctx &c, const float *spectra, const TrainSched &sc, float *out, cudaStream_t st)
{
    const int64_t per4 = int64_t(c.g.H) * c.g.W / 2; // 2 H W floats
    gather_target_kernel<<<std::min<int64_t>(blocks(per4, 256), 148 * 2), 256, 0, st>>>(
        reinterpret_cast<const float4 *>(spectra), per4, sc, reinterpret_cast<float4 *>(out));
    c.launches++;
}

void launch_log_advance(Ctx &c, const double *terms, double *log, const TrainSched &sc, cudaStream_t st)
{
    log_advance_kernel<<<1, 1, 0, st>>>(terms, log, sc);
    c.launches++;
}

// one trunk layer forward: h = relu([a1 | a2] W^T + b), W [width][K] row-major
void launch_dense_fwd(Ctx &c, const float *a1, int ld1, int ka, const float *a2, int ld2, int K, const float *W,
                      const float *b, int width, float *h, cudaStream_t st)
{
    const int n = c.g.n;
    ASrc a{a1, a2, ld1, ld2, ka, K};
    if (width > 160)
        throw std::invalid_argument("training supports deform-net widths up to 160");
    launch_rows<5, true, 0>(pick_rpt(n), n, a, W, 1, K, width, b, nullptr, 0, h, width, st);
    c.launches++;
}

// heads forward into the residual planes [5][plane] (dEl, dAz, dRe, dIm, dDelta)
void launch_heads_fwd(Ctx &c, const float *h7, int width, const float *Wh, const float *bh, float *planes,
                      int64_t plane, cudaStream_t st)
{
    const int n = c.g.n;
    ASrc a{h7, nullptr, width, 0, width, width};
    launch_rows<1, true, 2>(4, n, a, Wh, 1, width, 5, bh, nullptr, 0, planes, plane, st);
    c.launches++;
}

// dZ_prev = (dZ W[:, :width]) * (h_prev > 0), W [width][cols]
void launch_dense_bwd_input(Ctx &c, const float *dz, int width, const float *W, int cols, const float *h_prev,
                            float *dz_prev, cudaStream_t st)
{
    const int n = c.g.n;
    ASrc a{dz, nullptr, width, 0, width, width};
    launch_rows<5, false, 1>(pick_rpt(n), n, a, W, cols, 1, width, nullptr, h_prev, width, dz_prev, width, st);
    c.launches++;
}

size_t dw_partial_floats(int n, int R, int C) { return size_t((n + DW_CHUNK_MIN - 1) / DW_CHUNK_MIN) * R * (C + 1); }

// rows per split-K chunk: about two CTAs per SM over the whole grid (a multiple
// of 16 rows, at least DW_CHUNK_MIN)
static int dw_chunk(int n, int coltiles)
{
    const int target = std::max(1, 2 * 148 / coltiles);
    const int rows = (n + target - 1) / target;
    return std::max(DW_CHUNK_MIN, (rows + 15) / 16 * 16);
}

// dW [R][K] = dZ^T [a1 | a2], db [R] = column sums of dZ
void launch_dense_bwd_weights(Ctx &c, const float *dz, int R, const float *a1, int ld1, int ka, const float *a2,
                              int ld2, int K, float *part, float *dW, float *db, cudaStream_t st)
{
    const int n = c.g.n;
    const int coltiles = blocks(K + 1, DW_C);
    const int chunk = dw_chunk(n, coltiles);
    const int chunks = std::max(1, (n + chunk - 1) / chunk);
    ASrc in{a1, a2, ld1, ld2, ka, K};
    dim3 grid(coltiles, chunks);
    const float *one = nullptr;
    check_cuda(cudaGetSymbolAddress((void **)&one, c_one), "ones symbol");
    if (R <= 32)
        gemm_dw_kernel<1><<<grid, GT, 0, st>>>(dz, R, R, in, n, chunk, one, part);
    else if (R <= 160)
        gemm_dw_kernel<5><<<grid, GT, 0, st>>>(dz, R, R, in, n, chunk, one, part);
    else
        throw std::invalid_argument("training supports deform-net widths up to 160");
    dw_reduce_kernel<<<blocks(int64_t(R) * (K + 1), 256), 256, 0, st>>>(part, chunks, R, K + 1, dW, db);
    c.launches += 2;
}

void launch_heads_bwd(Ctx &c, const float *d_center, const float *d_response, const float *d_atten,
                      const float *Wc, const float *Wr, const float *Wa, const float *h7, int width, float *dz7,
                      float *dr5, cudaStream_t st)
{
    const int n = c.g.n;
    heads_bwd_kernel<<<blocks(int64_t(n) * width, 256), 256, 0, st>>>(d_center, d_response, d_atten, Wc, Wr, Wa, h7,
                                                                      n, width, dz7);
    pack_dr_kernel<<<blocks(n, 256), 256, 0, st>>>(d_center, d_response, d_atten, n, dr5);
    c.launches += 2;
}

} // namespace swr
