// C ABI of libswr.so (include/swr.h): scene load, host-side per-scene
// precompute, the chunked render pipeline and the per-stage parity hooks.
//
// Host precompute (once per scene) uses this host's glibc exactly as the
// reference does, so every per-scene constant that reaches a bin is the
// reference's bit pattern: materialised centres (tanhf, splat.cpp:60-65),
// delta0 = 1/(1+expf(-a)) (splat.cpp:105-106), the centre encoding
// (sinf/cosf, deform.cpp:54-70), Sigma^-1 entries (splat.cpp:200-211) and the
// FP64 bbox half widths (splat.cpp:223-225). This TU is compiled with
// -ffp-contract=off.
#include "swr.h"
#include "swr_internal.h"

#include <json.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>
#include <thread>
#include <chrono>

namespace swr
{

struct cuda_error : std::runtime_error
{
    using std::runtime_error::runtime_error;
};

void check_cuda(cudaError_t e, const char *what)
{
    if (e != cudaSuccess)
        throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Calls on one context are ordered on the device even when they use different
// streams: every entry point that touches the context's buffers first waits for
// the previous call's last work (an event), then records its own.
struct StreamOrder
{
    // Orders this call after the previous C-ABI call on the context (the two may run
    // on different streams and share the context's work buffers). Under CUDA-graph
    // capture of `st` (swr_render_device only) the cross-call event is neither waited
    // on nor recorded -- an event of uncaptured work cannot enter a graph -- and
    // ordering the graph's replays against other calls on the context is the
    // caller's (as for any graph); allocation and host syncs are refused meanwhile.
    Ctx &c;
    cudaStream_t st;
    bool captured = false;
    StreamOrder(Ctx &cx, cudaStream_t s, bool allow_capture = false) : c(cx), st(s)
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        check_cuda(cudaStreamIsCapturing(st, &cs), "capture status");
        if (cs != cudaStreamCaptureStatusNone)
        {
            if (!allow_capture)
                throw std::invalid_argument("this call synchronises with the host and cannot be captured into a "
                                            "CUDA graph (swr_render_device can)");
            captured = true;
            c.capturing = true;
            return;
        }
        if (!c.order_ev)
            check_cuda(cudaEventCreateWithFlags(&c.order_ev, cudaEventDisableTiming), "order event");
        else if (c.order_pending)
            check_cuda(cudaStreamWaitEvent(st, c.order_ev, 0), "order wait");
    }
    ~StreamOrder()
    {
        if (captured)
        {
            c.capturing = false;
            return;
        }
        if (cudaEventRecord(c.order_ev, st) == cudaSuccess)
            c.order_pending = true;
    }
};

static thread_local std::string g_err;

template <class F>
static int guarded(F &&f)
{
    try
    {
        f();
        return SWR_OK;
    }
    catch (const std::invalid_argument &e)
    {
        g_err = e.what();
        return SWR_EINVAL;
    }
    catch (const std::domain_error &e)
    {
        g_err = e.what();
        return SWR_EDOMAIN;
    }
    catch (const cuda_error &e)
    {
        g_err = e.what();
        return SWR_ECUDA;
    }
    catch (const std::runtime_error &e)
    {
        g_err = e.what();
        return SWR_ERUNTIME;
    }
    catch (const std::exception &e)
    {
        g_err = e.what();
        return SWR_ERUNTIME;
    }
}

int swr_guarded(const std::function<void()> &f) { return guarded(f); }

// ------------------------------------------------------------- scene build

// Per-primitive render inputs from the raw fields, on the host (glibc tanhf /
// expf like the reference's prepare(), splat.cpp:159-249)
SceneFields scene_fields(const Grid &g, int n, const float *center_raw, const float *cholesky, const float *atten,
                         const float *response)
{
    const int np = g.np;
    SceneFields f;
    f.el0.assign(np, 0.f);
    f.az0.assign(np, 0.f);
    f.d0.assign(np, 0.f);
    f.re0.assign(np, 0.f);
    f.im0.assign(np, 0.f);
    f.il3.assign(np, 0.f);
    f.l2v.assign(np, 0.f);
    f.shape.assign(np, make_float4(0, 0, 0, 0));
    f.bwd.assign(np, make_float4(0, 0, 0, 0));
    f.half.assign(np, make_double2(0, 0));
    for (int p = 0; p < n; p++)
    {
        const float rel = center_raw[2 * size_t(p)], raz = center_raw[2 * size_t(p) + 1];
        f.el0[p] = float(kPi / 4) * (std::tanh(rel) + 1.0f); // float overloads: glibc tanhf
        f.az0[p] = float(kPi) * (std::tanh(raz) + 1.0f);
        const float a = atten[p];
        f.d0[p] = 1.0f / (1.0f + std::exp(-a));
        f.re0[p] = response[2 * size_t(p)];
        f.im0[p] = response[2 * size_t(p) + 1];
        const float c1 = cholesky[3 * size_t(p)], l2 = cholesky[3 * size_t(p) + 1], c3 = cholesky[3 * size_t(p) + 2];
        const float l1 = c1 < 1e-4f ? 1e-4f : c1; // std::max(l, chol_floor)
        const float l3 = c3 < 1e-4f ? 1e-4f : c3;
        const float det = l1 * l1 * l3 * l3;
        f.shape[p] = make_float4((l2 * l2 + l3 * l3) / det, -l2 / (l1 * l3 * l3), 1.0f / (l3 * l3), 1.0f / l1);
        f.il3[p] = 1.0f / l3;
        f.l2v[p] = l2;
        f.half[p] = make_double2(double(g.radius) * double(l1),
                                 double(g.radius) * std::sqrt(double(l2) * l2 + double(l3) * l3));
        const float th_el = std::tanh(rel), th_az = std::tanh(raz);
        f.bwd[p] = make_float4(1.0f - th_el * th_el, 1.0f - th_az * th_az, c1 >= 1e-4f ? 1.0f : 0.0f,
                               c3 >= 1e-4f ? 1.0f : 0.0f);
    }
    return f;
}

// overwrite the device scene entries of c with host-derived ones (same arrays)
void refresh_scene_host(Ctx &c, const float *center_raw, const float *cholesky, const float *atten,
                        const float *response)
{
    const SceneFields f = scene_fields(c.g, c.g.n, center_raw, cholesky, atten, response);
    auto put = [&](void *dst, const void *src, size_t bytes) {
        check_cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "refresh scene");
    };
    const size_t np = size_t(c.g.np);
    put(c.s.el0, f.el0.data(), 4 * np);
    put(c.s.az0, f.az0.data(), 4 * np);
    put(c.s.delta0, f.d0.data(), 4 * np);
    put(c.s.re0, f.re0.data(), 4 * np);
    put(c.s.im0, f.im0.data(), 4 * np);
    put(c.s.shape, f.shape.data(), 16 * np);
    put(c.s.inv_l3, f.il3.data(), 4 * np);
    put(c.s.l2, f.l2v.data(), 4 * np);
    put(c.s.half, f.half.data(), 16 * np);
    put(c.s.bwd, f.bwd.data(), 16 * np);
}

// Upper bound on the (tile, primitive) pairs of one position for ANY residuals:
// residuals move centres and attenuation but never the covariance, so each
// primitive's box extent is fixed by its static half widths (splat.cpp:222-248):
// rows <= floor(2 h_el / cell) + 3, columns <= floor(2 h_az / cell) + 3 (or the
// full circle), and a span of m cells crosses at most ceil((m - 1) / T) + 1 tiles
// (+1 column tile for a split wrapped span).
int64_t pair_bound(const Grid &g, const std::vector<double2> &half, int n)
{
    if (!g.cut)
        return int64_t(n) * g.tiles;
    auto span_tiles = [&](int64_t m) { return (m - 1 + g.tile - 1) / g.tile + 1; };
    int64_t total = 0;
    for (int p = 0; p < n; p++)
    {
        const double rows_d = std::floor(2.0 * half[p].x / g.cell_el) + 3.0;
        const int64_t rows = rows_d >= double(g.H) ? g.H : std::max<int64_t>(1, int64_t(rows_d));
        const int64_t tr = std::min<int64_t>(g.th, span_tiles(rows));
        int64_t tc = g.tw;
        if (2.0 * half[p].y < double(g.W) * g.cell_az)
        {
            const double cols_d = std::floor(2.0 * half[p].y / g.cell_az) + 3.0;
            const int64_t cols = cols_d >= double(g.W) ? g.W : std::max<int64_t>(1, int64_t(cols_d));
            tc = std::min<int64_t>(g.tw, span_tiles(cols) + 1);
        }
        total += tr * tc;
    }
    return std::max<int64_t>(total, 1);
}

void build_scene(Ctx &c, const HostScene &hs, int device)
{
    c.host = std::make_shared<const HostScene>(hs);
    if (hs.H < 1 || hs.W < 1)
        throw std::invalid_argument("gaussian set has an empty grid");
    if (hs.n < 0)
        throw std::invalid_argument("negative primitive count");
    int ndev = 0;
    check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0)
        check_cuda(cudaGetDevice(&device), "cudaGetDevice");
    if (device >= ndev)
        throw cuda_error("no such CUDA device");
    cudaDeviceProp prop;
    check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        throw cuda_error("libswr requires an sm_100 (B200) device; found sm_" + std::to_string(prop.major) +
                         std::to_string(prop.minor));
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    c.device = device;
    {
        size_t free_b = 0, total_b = 0;
        check_cuda(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        c.mem_total = total_b;
    }
    check_cuda(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "cudaStreamCreate");

    const int tile = hs.tile < 1 ? 16 : hs.tile; // splat.cpp:166
    if (tile > 32)
        throw std::invalid_argument("tile edge above 32 cells is not supported by the device rasteriser");
    Grid &g = c.g;
    g.H = hs.H;
    g.W = hs.W;
    g.n = hs.n;
    g.np = std::max(16, (hs.n + 15) / 16 * 16);
    g.tile = tile;
    g.th = (hs.H + tile - 1) / tile;
    g.tw = (hs.W + tile - 1) / tile;
    g.tiles = g.th * g.tw;
    if (g.tiles > 1024)
        throw std::invalid_argument("more than 1024 tiles per spectrum is not supported");
    g.cut = hs.cutoff > 0.0f;
    g.radius = g.cut ? hs.cutoff : 0.0f;
    g.cut2 = g.cut ? hs.cutoff * hs.cutoff : INFINITY;
    g.cell_el = (kPi / 2.0) / hs.H; // spectrum.cpp:29-32
    g.cell_az = (2.0 * kPi) / hs.W;
    c.cutoff = hs.cutoff;
    c.tile = hs.tile;
    // default chunk: ~12.8M (Gaussian, position) rows per chunk, 256..1024 positions
    // (measured: 256 is fastest at 50k Gaussians, 1024 at 10k; option "chunk" overrides)

    std::memcpy(c.bbox_min, hs.bmin, sizeof(hs.bmin));
    c.manifest_hash = hs.manifest_hash;
    std::memcpy(c.bbox_max, hs.bmax, sizeof(hs.bmax));
    c.rssi_calibrated = hs.has_rssi;
    c.rssi_slope = hs.rssi_slope;
    c.rssi_intercept = hs.rssi_intercept;

    const int n = hs.n, np = g.np;
    SceneFields f = scene_fields(g, n, hs.center_raw.data(), hs.cholesky.data(), hs.atten.data(), hs.response.data());
    // positions per chunk: ~12.8M (Gaussian, position) rows, 256..1024 (measured: 256
    // is fastest at 50k Gaussians, 1024 at 10k; option "chunk" overrides), and never
    // more than keeps a chunk's pair list within 32-bit offsets for any residuals
    c.pairs_per_pos_max = pair_bound(g, f.half, n);
    c.chunk_cap = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(1) << 30, (int64_t(INT32_MAX) - 1) / c.pairs_per_pos_max)));
    c.chunk = int(std::min<int64_t>(c.chunk_cap, std::min<int64_t>(1024, std::max<int64_t>(256, (int64_t(12800000) / std::max(1, hs.n)) / 64 * 64))));
    const std::vector<float> &el0 = f.el0, &az0 = f.az0;
    std::vector<float> elc(hs.H), azc(hs.W);
    for (int r = 0; r < hs.H; r++)
        elc[r] = float((r + 0.5) * g.cell_el);
    for (int j = 0; j < hs.W; j++)
        azc[j] = float((j + 0.5) * g.cell_az);
    SceneDev &s = c.s;
    s.el0 = upload(c, f.el0);
    s.az0 = upload(c, f.az0);
    s.delta0 = upload(c, f.d0);
    s.re0 = upload(c, f.re0);
    s.im0 = upload(c, f.im0);
    s.shape = upload(c, f.shape);
    s.inv_l3 = upload(c, f.il3);
    s.l2 = upload(c, f.l2v);
    s.half = upload(c, f.half);
    s.bwd = upload(c, f.bwd);
    s.el_c = upload(c, elc);
    s.az_c = upload(c, azc);

    // --------------------------------------------------------------- network
    c.has_net = !hs.lw.empty();
    if (!c.has_net)
        return;
    NetDev &nt = c.net;
    nt.width = hs.width;
    if (hs.width < 1 || hs.width > 512)
        throw std::invalid_argument("deform-net width must be in [1, 512]");
    nt.wp = hs.width <= 160 ? 160 : 512;
    nt.bands_c = hs.bands_c;
    nt.bands_p = hs.bands_p;
    nt.dc = 2 * (2 * hs.bands_c + 1);
    nt.dp = 3 * (2 * hs.bands_p + 1);
    nt.d = nt.dc + nt.dp;
    if (nt.dp > 64 || hs.bands_p > 20 || hs.bands_c > 40)
        throw std::invalid_argument("encoding bands out of the supported range");
    const int Wd = hs.width, WP = nt.wp, D = nt.d, Dc = nt.dc, Dp = nt.dp;
    // shape checks against deform.cpp:72-102
    for (int i = 0; i < 8; i++)
    {
        const size_t cols = i == 0 ? D : ((i == 2 || i == 4 || i == 6) ? Wd + D : Wd);
        if (hs.lw[i].size() != size_t(Wd) * cols || hs.lb[i].size() != size_t(Wd))
            throw std::invalid_argument("deform layer shape does not match width/encoding");
    }
    const int hr[3] = {2, 2, 1};
    for (int i = 0; i < 3; i++)
        if (hs.lw[8 + i].size() != size_t(hr[i]) * Wd || hs.lb[8 + i].size() != size_t(hr[i]))
            throw std::invalid_argument("deform head shape does not match width");

    std::vector<float> whT(size_t(7) * WP * WP, 0.f), bias(size_t(8) * WP, 0.f), wpos(size_t(4) * WP * Dp, 0.f),
        wcen(size_t(4) * WP * Dc, 0.f), heads(size_t(5) * WP, 0.f), hbias(5, 0.f);
    for (int l = 0; l < 8; l++)
    {
        const size_t cols = l == 0 ? D : ((l == 2 || l == 4 || l == 6) ? Wd + D : Wd);
        const float *Wl = hs.lw[l].data();
        for (int r = 0; r < Wd; r++)
            bias[size_t(l) * WP + r] = hs.lb[l][r];
        if (l >= 1)
            for (int r = 0; r < Wd; r++)
                for (int k = 0; k < Wd; k++)
                    whT[(size_t(l - 1) * WP + k) * WP + r] = Wl[r * cols + k];
        if (l % 2 == 0)
        {
            const int j = l / 2;
            const size_t off = l == 0 ? 0 : Wd; // encoding columns follow the hidden block
            for (int r = 0; r < Wd; r++)
            {
                for (int k = 0; k < Dc; k++)
                    wcen[(size_t(j) * WP + r) * Dc + k] = Wl[r * cols + off + k];
                for (int k = 0; k < Dp; k++)
                    wpos[(size_t(j) * WP + r) * Dp + k] = Wl[r * cols + off + Dc + k];
            }
        }
    }
    int h = 0;
    for (int i = 0; i < 3; i++)
        for (int r = 0; r < hr[i]; r++, h++)
        {
            for (int k = 0; k < Wd; k++)
                heads[size_t(h) * WP + k] = hs.lw[8 + i][size_t(r) * Wd + k];
            hbias[h] = hs.lb[8 + i][r];
        }
    nt.whT = upload(c, whT);
    nt.bias = upload(c, bias);
    nt.wpos = upload(c, wpos);
    nt.wcen = upload(c, wcen);
    nt.heads = upload(c, heads);
    nt.hbias = upload(c, hbias);
    nt.cg = dalloc<float>(c, size_t(np) * 4 * WP);

    // centre encoding per Gaussian (host glibc sinf/cosf, deform.cpp:54-70)
    std::vector<float> cenc(size_t(np) * Dc, 0.f);
    for (int p = 0; p < n; p++)
    {
        float *row = cenc.data() + size_t(p) * Dc;
        const float v[2] = {el0[p], az0[p]};
        row[0] = v[0];
        row[1] = v[1];
        float *blk = row + 2;
        for (int k = 0; k < hs.bands_c; k++)
        {
            const float f = float(std::ldexp(kPi, k));
            blk[0] = std::sin(f * v[0]);
            blk[1] = std::sin(f * v[1]);
            blk[2] = std::cos(f * v[0]);
            blk[3] = std::cos(f * v[1]);
            blk += 4;
        }
    }
    float *d_cenc = upload(c, cenc);
    launch_center_terms(c, d_cenc, c.stream);
    check_cuda(cudaStreamSynchronize(c.stream), "centre terms");
    dfree(c, d_cenc);
    if (mlp_tc_available() && (WP == 160 || WP == 512) && n > 0)
    {
        // activation scale of the tensor-core MLP: the largest ReLU output over all
        // Gaussians x 16 probe positions (bbox corners + interior points), FP32 kernel
        constexpr int kProbe = 16;
        ensure_work(c, kProbe);
        std::vector<float> probe(3 * kProbe);
        for (int p = 0; p < kProbe; p++)
            for (int a = 0; a < 3; a++)
            {
                const double t = p < 8 ? double((p >> a) & 1) : 0.125 + 0.75 * ((p * 0.618034 * (a + 1)) - std::floor(p * 0.618034 * (a + 1)));
                probe[3 * p + a] = float(t);
            }
        float *d_probe = upload(c, probe);
        launch_pos_prep(c, d_probe, kProbe, true, c.stream); // mlp_precision 0 here: unscaled
        float amax[8];
        probe_activations(c, kProbe, amax, c.stream);
        dfree(c, d_probe);
        // per layer: 2^k_l amax_l <= 65504 / 64 (headroom for positions the probe did
        // not see; an overflow anyway re-runs the chunk in FP32), k_l in [-20, 10]
        for (int l = 0; l < 8; l++)
        {
            const float m = amax[l];
            c.net.tc_amax[l] = m;
            int k = 10;
            if (m > 0.0f && std::isfinite(m))
                k = std::min(10, std::max(-20, int(std::floor(std::log2(65504.0 / 64.0 / double(m))))));
            c.net.tc_ascale[l] = k;
        }
        if (WP == 160)
            prepare_tc2_weights(c, whT, heads, bias);
        else
            prepare_wide_weights(c, whT, heads, bias);
        c.mlp_precision = 1; // FP32-grade tensor-core MLP by default (SWR_MLP_FP32 remains an option)
    }
}

// ------------------------------------------------------------- work buffers

void ensure_work(Ctx &c, int64_t nb)
{
    Work &w = c.w;
    if (w.cap_b >= nb)
        return;
    for (void *p : {(void *)w.pos01, (void *)w.pterm, (void *)w.res, (void *)w.dyn, (void *)w.rng, (void *)w.cnt,
                    (void *)w.seg, (void *)w.poff, (void *)w.tile_off, (void *)w.tile_part, (void *)w.tile_sum})
        dfree(c, p);
    const int np = c.g.np, tiles = c.g.tiles;
    const int wp = c.has_net ? c.net.wp : 32;
    w.cap_b = nb;
    w.pos01 = dalloc<float>(c, size_t(nb) * 4);
    w.pterm = dalloc<float>(c, size_t(nb) * 4 * wp);
    w.res = dalloc<float>(c, size_t(5) * nb * np);
    w.dyn = dalloc<float4>(c, size_t(nb) * np);
    w.rng = dalloc<int4>(c, size_t(nb) * np);
    w.cnt = dalloc<int>(c, size_t(nb) * np);
    w.seg = dalloc<int64_t>(c, size_t(nb) + 1);
    w.poff = dalloc<int>(c, size_t(nb) * np);
    w.tile_off = dalloc<int>(c, size_t(nb) * (tiles + 1));
    w.tile_part = dalloc<float4>(c, size_t(nb) * tiles);
    w.tile_sum = dalloc<double>(c, size_t(nb) * tiles);
    if (!w.stats)
        w.stats = dalloc<int64_t>(c, 3);
    if (!w.reruns)
    {
        w.reruns = dalloc<unsigned long long>(c, 1);
        check_cuda(cudaMemset(w.reruns, 0, sizeof(unsigned long long)), "rerun counter");
    }
    if (!w.host_pairs)
        check_cuda(cudaHostAlloc((void **)&w.host_pairs, 4 * sizeof(int64_t), cudaHostAllocDefault), "host alloc");
    w.max_chunks = 0; // chunk histogram re-sized on demand
    dfree(c, w.chunk_hist);
    w.chunk_hist = nullptr;
}

void ensure_pairs(Ctx &c, int64_t pairs, int nb, int64_t max_seg)
{
    Work &w = c.w;
    if (pairs > w.cap_pairs)
    {
        dfree(c, w.keys);
        dfree(c, w.vals);
        dfree(c, w.sorted);
        dfree(c, w.perm);
        w.perm = nullptr;
        const int64_t cap = std::max<int64_t>(pairs + pairs / 8, 1024);
        w.keys = dalloc<uint16_t>(c, cap);
        w.vals = dalloc<int>(c, cap);
        w.sorted = dalloc<int>(c, cap);
        w.cap_pairs = cap;
    }
    if (w.want_perm && !w.perm)
        w.perm = dalloc<int>(c, w.cap_pairs);
    const int need = int(std::max<int64_t>(1, (max_seg + kSort - 1) / kSort));
    if (need > w.max_chunks || !w.chunk_hist)
    {
        dfree(c, w.chunk_hist);
        w.max_chunks = std::max(need + need / 4, 1);
        w.chunk_hist = dalloc<int>(c, size_t(w.cap_b) * w.max_chunks * c.g.tiles);
    }
    (void)nb;
}

// --------------------------------------------------------------- pipeline

struct Timer
{
    Ctx &c;
    cudaStream_t st;
    cudaEvent_t ev[7];
    int k = 0;
    bool on;
    Timer(Ctx &cx, cudaStream_t s) : c(cx), st(s), on(cx.stage_timing && !cx.capturing)
    {
        if (on)
            for (auto &e : ev)
                cudaEventCreate(&e);
    }
    void mark()
    {
        if (on)
            cudaEventRecord(ev[k++], st);
    }
    // events are read lazily (resolve_stage_times) so timing adds no host sync
    void finish()
    {
        if (!on)
            return;
        std::array<cudaEvent_t, 7> a;
        for (int i = 0; i < 7; i++)
            a[i] = ev[i];
        c.stage_pending.push_back(a);
    }
};

// fold the recorded per-chunk stage intervals into c.stage_ms (or drop them)
static void resolve_stage_times(Ctx &c, bool keep)
{
    for (auto &a : c.stage_pending)
    {
        cudaEventSynchronize(a[6]);
        if (keep)
            for (int i = 0; i < 6; i++)
            {
                float ms = 0;
                cudaEventElapsedTime(&ms, a[i], a[i + 1]);
                c.stage_ms[i] += ms;
            }
        for (auto &e : a)
            cudaEventDestroy(e);
    }
    c.stage_pending.clear();
}

// Render one chunk of nb positions whose (device) coordinates are d_pos.
// Residuals come from the MLP (use_mlp), the caller (already in w.res) or are
// zero. d_spec may be null (heads only).
// slices (non-empty): the raster runs in launches of these many positions (summing to
// nb) and after_raster(first, count) is called after each (the host-buffer path
// queues that slice's D2H there, so the copies overlap the following slices)
static void run_chunk(Ctx &c, const float *d_pos, int nb, bool normalized, bool use_mlp, bool with_res,
                      float *d_spec, bool heads, uint32_t flags, double *d_pooled, double *d_rssi, int32_t *d_aoa_rc,
                      double *d_aoa_ang, cudaStream_t st, const std::vector<int> &slices = {},
                      const std::function<void(int, int)> &after_raster = {}, bool host_pairs = false)
{
    Timer tm(c, st);
    tm.mark();
    if (use_mlp)
    {
        launch_pos_prep(c, d_pos, nb, normalized, st);
        tm.mark();
        launch_mlp(c, nb, st);
        tm.mark();
    }
    else
    {
        tm.mark();
        tm.mark();
    }
    check_cuda(cudaMemsetAsync(c.w.stats + 2, 0, sizeof(int64_t), st), "reset flag");
    launch_setup(c, nb, use_mlp || with_res, st);
    tm.mark();
    launch_bin_count(c, nb, st);
    // Pair buffers sized to the scene's bound (pair_bound: any residuals) when that
    // fits the budget: then nothing in the chunk waits for the host -- the sort grid
    // covers the bound (CTAs past a segment exit), and an fp16 overflow of the
    // tensor-core MLP (a non-finite residual flagged by setup) re-runs the chunk's
    // MLP in FP32 through kernels gated on that device flag. Otherwise (huge
    // scenes) the pair count is read back and the buffers sized to it.
    const int64_t bound = int64_t(nb) * c.pairs_per_pos_max;
    const int64_t budget =
        c.async_pair_budget >= 0 ? c.async_pair_budget : std::min<int64_t>(int64_t(24) << 30, int64_t(c.mem_total / 4));
    const bool async = !host_pairs && bound * (c.w.want_perm ? 14 : 10) <= budget;
    if (async)
    {
        if (use_mlp && mlp_uses_tc(c))
        {
            const int keep = c.mlp_precision;
            c.gate = c.w.stats + 2;
            c.mlp_precision = 0;
            try
            {
                launch_pos_prep(c, d_pos, nb, normalized, st); // unscaled position terms
                launch_mlp(c, nb, st);
                launch_setup(c, nb, true, st);
                launch_bin_count(c, nb, st);
            }
            catch (...)
            {
                c.gate = nullptr;
                c.mlp_precision = keep;
                throw;
            }
            c.gate = nullptr;
            c.mlp_precision = keep;
        }
        ensure_pairs(c, bound, nb, c.pairs_per_pos_max);
        c.pairs_on_host = false;
        // sort grid for ~45% of the bound (measured segments: ~40% of it)
        launch_bin_sort(c, nb, -1, int(std::min<int64_t>(c.pairs_per_pos_max * 9 / 20 + 1, INT32_MAX)), st);
    }
    else
    {
        if (c.capturing)
            throw std::invalid_argument("swr_render_device under CUDA-graph capture: this batch's pair bound exceeds "
                                        "async_pair_budget, so the chunk would read its pair count on the host; "
                                        "capture smaller batches or raise the budget");
        check_cuda(cudaMemcpyAsync(c.w.host_pairs, c.w.stats, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                   "D2H pair count");
        check_cuda(cudaStreamSynchronize(st), "pair count");
        if (use_mlp && c.mlp_precision != 0 && c.w.host_pairs[2] != 0)
        {
            // a non-finite residual from the fp16 tensor-core MLP (an activation above
            // 65504): redo this chunk's MLP on the FP32 CUDA-core kernel
            c.mlp_reruns++;
            const int keep = c.mlp_precision;
            c.mlp_precision = 0;
            launch_pos_prep(c, d_pos, nb, normalized, st); // unscaled position terms
            launch_mlp(c, nb, st);
            c.mlp_precision = keep;
            launch_setup(c, nb, true, st);
            launch_bin_count(c, nb, st);
            check_cuda(cudaMemcpyAsync(c.w.host_pairs, c.w.stats, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                       "D2H pair count");
            check_cuda(cudaStreamSynchronize(st), "pair count");
        }
        const int64_t pairs = c.w.host_pairs[0], max_seg = c.w.host_pairs[1];
        if (pairs > INT32_MAX) // cannot happen within chunk_cap (pair_bound); the sort's offsets are 32-bit
            throw std::runtime_error("pair list of a chunk exceeds 2^31 entries");
        c.pairs_last = pairs;
        c.pairs_on_host = true;
        ensure_pairs(c, pairs, nb, max_seg);
        launch_bin_sort(c, nb, pairs, int(max_seg), st);
    }
    tm.mark();
    if (slices.empty())
    {
        launch_raster(c, nb, d_spec, heads, st, 0, 0);
        if (after_raster)
            after_raster(0, nb);
    }
    else
        for (int s0 = 0, i = 0; s0 < nb; s0 += slices[size_t(i)], i++)
        {
            const int n = std::min(slices[size_t(i)], nb - s0);
            launch_raster(c, n, d_spec, heads, st, 0, s0);
            if (after_raster)
                after_raster(s0, n);
        }
    tm.mark();
    if (heads)
        launch_heads(c, nb, flags, d_pooled, d_rssi, d_aoa_rc, d_aoa_ang, st);
    tm.mark();
    check_cuda(cudaGetLastError(), "kernel launch");
    tm.finish();
}

// positions per raster launch + D2H slice in swr_render: option "copy_chunk" (Ctx::copy_chunk, default 256)

// Raster launches of a chunk in swr_render, each slice's spectra copied out right
// behind it: 256-position slices, except that the call's LAST chunk ends in halving
// slices (.., 128, 64, 32, 32), so only ~32 spectra's copy is left exposed after
// the last raster (a uniform small slice costs launch tails on every slice).
static std::vector<int> copy_slices(int nb, bool last, int kCopySlice)
{
    std::vector<int> v;
    int r = nb;
    while (r > 0)
    {
        int n = std::min(r, kCopySlice);
        if (last && r <= kCopySlice && r > 64)
            n = std::max(32, r / 2);
        v.push_back(n);
        r -= n;
    }
    return v;
}

static bool is_pinned(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess)
    {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

static void device_render(Ctx &c, const float *d_pos, int64_t B, uint32_t flags, float *d_spec, double *d_pooled,
                          double *d_rssi, int32_t *d_aoa_rc, double *d_aoa_ang, cudaStream_t st)
{
    const bool use_mlp = c.has_net && !(flags & SWR_NO_RESIDUALS);
    if (use_mlp && c.g.n < 1)
        throw std::invalid_argument("empty gaussian set"); // predict_residuals (deform.cpp:147-148) via render_at
    const bool heads = flags & (SWR_OUT_POOLED | SWR_OUT_RSSI | SWR_OUT_AOA);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
    ensure_work(c, chunk);
    const size_t per = size_t(2) * c.g.H * c.g.W;
    for (int64_t b0 = 0; b0 < B; b0 += chunk)
    {
        const int nb = int(std::min<int64_t>(chunk, B - b0));
        run_chunk(c, d_pos + 3 * b0, nb, false, use_mlp, false,
                  (flags & SWR_OUT_SPECTRA) && d_spec ? d_spec + per * b0 : nullptr, heads, flags,
                  (flags & SWR_OUT_POOLED) && d_pooled ? d_pooled + b0 : nullptr,
                  (flags & SWR_OUT_RSSI) && d_rssi ? d_rssi + b0 : nullptr,
                  (flags & SWR_OUT_AOA) && d_aoa_rc ? d_aoa_rc + 2 * b0 : nullptr,
                  (flags & SWR_OUT_AOA) && d_aoa_ang ? d_aoa_ang + 2 * b0 : nullptr, st);
    }
}

struct Stage
{
    int64_t cap_b = 0;
    size_t cap_spec = 0;
    float *pos = nullptr;
    float *spec[2] = {nullptr, nullptr};
    double *pooled = nullptr, *rssi = nullptr, *ang = nullptr;
    int32_t *rc = nullptr;
    cudaStream_t copy = nullptr;
    cudaEvent_t done[2]{}, freed[2]{};
};

static Stage &stage_for(Ctx &c, int64_t B, int64_t chunk, size_t spec_elems)
{
    static_assert(sizeof(void *) == 8, "64-bit only");
    if (!c.host_stage)
        c.host_stage = new Stage();
    Stage &S = *static_cast<Stage *>(c.host_stage);
    if (!S.copy)
    {
        check_cuda(cudaStreamCreateWithFlags(&S.copy, cudaStreamNonBlocking), "copy stream");
        for (int i = 0; i < 2; i++)
        {
            check_cuda(cudaEventCreateWithFlags(&S.done[i], cudaEventDisableTiming), "event");
            check_cuda(cudaEventCreateWithFlags(&S.freed[i], cudaEventDisableTiming), "event");
        }
    }
    if (B > S.cap_b)
    {
        for (void *p : {(void *)S.pos, (void *)S.pooled, (void *)S.rssi, (void *)S.ang, (void *)S.rc})
            dfree(c, p);
        S.pos = dalloc<float>(c, size_t(3) * B);
        S.pooled = dalloc<double>(c, B);
        S.rssi = dalloc<double>(c, B);
        S.ang = dalloc<double>(c, 2 * B);
        S.rc = dalloc<int32_t>(c, 2 * B);
        S.cap_b = B;
    }
    if (spec_elems > S.cap_spec)
    {
        for (auto &p : S.spec)
        {
            dfree(c, p);
            p = dalloc<float>(c, spec_elems);
        }
        S.cap_spec = spec_elems;
    }
    (void)chunk;
    return S;
}

static void free_stage(Ctx &c)
{
    if (!c.host_stage)
        return;
    Stage *S = static_cast<Stage *>(c.host_stage);
    if (S->copy)
    {
        cudaStreamDestroy(S->copy);
        for (int i = 0; i < 2; i++)
        {
            cudaEventDestroy(S->done[i]);
            cudaEventDestroy(S->freed[i]);
        }
    }
    delete S;
    c.host_stage = nullptr;
}

static void upload_residuals(Ctx &c, const float *dc, const float *dr, const float *da, int64_t b0, int nb)
{
    // reference layouts [B][n][2], [B][n][2], [B][n] -> planes [5][cap_b][np]
    const int n = c.g.n, np = c.g.np;
    std::vector<float> planes(size_t(5) * c.w.cap_b * np, 0.f);
    const size_t plane = size_t(c.w.cap_b) * np;
    for (int s = 0; s < nb; s++)
        for (int g = 0; g < n; g++)
        {
            const size_t src = (size_t(b0 + s) * n + g);
            const size_t dst = size_t(s) * np + g;
            planes[0 * plane + dst] = dc[2 * src];
            planes[1 * plane + dst] = dc[2 * src + 1];
            planes[2 * plane + dst] = dr[2 * src];
            planes[3 * plane + dst] = dr[2 * src + 1];
            planes[4 * plane + dst] = da[src];
        }
    check_cuda(cudaMemcpy(c.w.res, planes.data(), planes.size() * sizeof(float), cudaMemcpyHostToDevice),
               "upload residuals");
}

HostScene parse_wrfc(const char *path)
{
    std::ifstream is(path, std::ios::binary);
    if (!is)
        throw std::runtime_error(std::string("cannot open ") + path);
    std::vector<char> buf((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    size_t at = 0;
    auto need = [&](size_t k) {
        if (at + k > buf.size())
            throw std::runtime_error("unexpected end of file");
    };
    auto u32 = [&]() {
        need(4);
        uint32_t v;
        std::memcpy(&v, buf.data() + at, 4);
        at += 4;
        return v;
    };
    auto u64 = [&]() {
        need(8);
        uint64_t v;
        std::memcpy(&v, buf.data() + at, 8);
        at += 8;
        return v;
    };
    auto magic = [&](const char *m, const char *what) {
        need(4);
        if (std::memcmp(buf.data() + at, m, 4) != 0)
            throw std::runtime_error(std::string("bad magic, not a ") + what);
        at += 4;
    };
    auto f32s = [&](std::vector<float> &v, size_t cnt) {
        need(4 * cnt);
        v.resize(cnt);
        std::memcpy(v.data(), buf.data() + at, 4 * cnt);
        at += 4 * cnt;
    };
    // checkpoint.cpp:100-141
    magic("WRFC", "checkpoint");
    if (u32() != 1)
        throw std::runtime_error("unsupported checkpoint version");
    if (u32() != 3)
        throw std::runtime_error("unexpected checkpoint section count");
    u32();
    uint64_t off[3], size[3];
    for (int i = 0; i < 3; i++)
    {
        off[i] = u64();
        size[i] = u64();
    }
    HostScene hs;
    // splat.cpp:723-736
    at = off[0];
    magic("WRF2", "gaussian section");
    if (u32() != 1)
        throw std::runtime_error("unsupported gaussian section version");
    const uint32_t n = u32();
    u32();
    hs.n = int(n);
    f32s(hs.center_raw, size_t(n) * 2);
    f32s(hs.cholesky, size_t(n) * 3);
    f32s(hs.atten, n);
    f32s(hs.response, size_t(n) * 2);
    // deform.cpp:354-384
    at = off[1];
    magic("WRFD", "deform section");
    if (u32() != 1)
        throw std::runtime_error("unsupported deform section version");
    if (u32() != 11)
        throw std::runtime_error("unexpected deform layer count");
    hs.width = int(u32());
    hs.bands_c = int(u32());
    hs.bands_p = int(u32());
    std::vector<std::pair<uint32_t, uint32_t>> shp(11);
    for (auto &s : shp)
    {
        s.first = u32();
        s.second = u32();
    }
    hs.lw.resize(11);
    hs.lb.resize(11);
    for (int i = 0; i < 11; i++)
    {
        f32s(hs.lw[i], size_t(shp[i].first) * shp[i].second);
        f32s(hs.lb[i], shp[i].first);
    }
    need(0);
    if (off[2] + size[2] > buf.size())
        throw std::runtime_error("unexpected end of file");
    const auto j = nlohmann::json::parse(std::string(buf.data() + off[2], size[2]));
    hs.H = j.at("grid").at("n_elevation").get<int>();
    hs.W = j.at("grid").at("n_azimuth").get<int>();
    const auto &cfg = j.at("config");
    if (cfg.contains("cutoff_radius"))
        hs.cutoff = cfg.at("cutoff_radius").get<float>();
    if (cfg.contains("tile"))
        hs.tile = cfg.at("tile").get<int>();
    const auto bmin = j.at("bbox_min").get<std::vector<double>>();
    const auto bmax = j.at("bbox_max").get<std::vector<double>>();
    for (int a = 0; a < 3; a++)
    {
        hs.bmin[a] = bmin.at(a);
        hs.bmax[a] = bmax.at(a);
    }
    if (j.contains("manifest_hash"))
        hs.manifest_hash = std::stoull(j.at("manifest_hash").get<std::string>(), nullptr, 16);
    hs.config_json = cfg.dump();
    if (j.contains("iteration"))
        hs.iteration = j.at("iteration").get<int64_t>();
    // an RSSI model (load_rssi_model, tasks.cpp:139-150): the affine calibration
    if (j.contains("rssi_slope") && j.contains("rssi_intercept"))
    {
        hs.has_rssi = true;
        hs.rssi_slope = j.at("rssi_slope").get<double>();
        hs.rssi_intercept = j.at("rssi_intercept").get<double>();
    }
    return hs;
}

} // namespace swr

using namespace swr;

struct swr_ctx
{
    Ctx c;
};

static void destroy(swr_ctx *h)
{
    if (!h)
        return;
    cudaSetDevice(h->c.device);
    if (h->c.order_ev) // the last call's device work (possibly on a caller's stream) ends first
    {
        cudaEventSynchronize(h->c.order_ev);
        cudaEventDestroy(h->c.order_ev);
    }
    resolve_stage_times(h->c, false);
    for (void *p : h->c.allocs)
        cudaFree(p);
    if (h->c.w.host_pairs)
        cudaFreeHost(h->c.w.host_pairs);
    free_stage(h->c);
    if (h->c.stream)
        cudaStreamDestroy(h->c.stream);
    delete h;
}

extern "C" {

const char *swr_last_error(void) { return g_err.c_str(); }
int swr_version(void) { return 100; }

int swr_scene_create_wrfc(const char *path, int device, swr_ctx **out)
{
    *out = nullptr;
    auto *h = new swr_ctx();
    const int rc = guarded([&] {
        const HostScene hs = parse_wrfc(path);
        build_scene(h->c, hs, device);
    });
    if (rc)
    {
        destroy(h);
        return rc;
    }
    *out = h;
    return SWR_OK;
}

int swr_wrfc_peek(const char *path, swr_scene_info *info, double *rssi_cal, int *has_rssi)
{
    return guarded([&] {
        const HostScene hs = parse_wrfc(path);
        if (info)
        {
            std::memset(info, 0, sizeof(*info));
            info->n_elevation = hs.H;
            info->n_azimuth = hs.W;
            info->n = hs.n;
            info->width = hs.width;
            info->bands_center = hs.bands_c;
            info->bands_position = hs.bands_p;
            info->cutoff_radius = hs.cutoff;
            info->tile = hs.tile;
            for (int a = 0; a < 3; a++)
            {
                info->bbox_min[a] = hs.bmin[a];
                info->bbox_max[a] = hs.bmax[a];
            }
        }
        if (has_rssi)
            *has_rssi = hs.has_rssi ? 1 : 0;
        if (rssi_cal)
        {
            rssi_cal[0] = hs.rssi_slope;
            rssi_cal[1] = hs.rssi_intercept;
        }
    });
}

int swr_scene_create(int H, int W, int n, const float *center_raw, const float *cholesky, const float *atten_logit,
                     const float *response, int width, int bands_c, int bands_p, const float *const *layer_w,
                     const float *const *layer_b, float cutoff, int tile, const double *bmin, const double *bmax,
                     int device, swr_ctx **out)
{
    *out = nullptr;
    auto *h = new swr_ctx();
    const int rc = guarded([&] {
        HostScene hs;
        hs.H = H;
        hs.W = W;
        hs.n = n;
        hs.center_raw.assign(center_raw, center_raw + size_t(2) * n);
        hs.cholesky.assign(cholesky, cholesky + size_t(3) * n);
        hs.atten.assign(atten_logit, atten_logit + size_t(n));
        hs.response.assign(response, response + size_t(2) * n);
        hs.width = width;
        hs.bands_c = bands_c;
        hs.bands_p = bands_p;
        hs.cutoff = cutoff;
        hs.tile = tile;
        for (int a = 0; a < 3; a++)
        {
            hs.bmin[a] = bmin ? bmin[a] : 0.0;
            hs.bmax[a] = bmax ? bmax[a] : 1.0;
        }
        if (layer_w)
        {
            const int D = 2 * (2 * bands_c + 1) + 3 * (2 * bands_p + 1);
            hs.lw.resize(11);
            hs.lb.resize(11);
            for (int i = 0; i < 11; i++)
            {
                const size_t rows = i < 8 ? width : (i == 10 ? 1 : 2);
                const size_t cols = i == 0 ? D : (i < 8 ? ((i == 2 || i == 4 || i == 6) ? width + D : width) : width);
                hs.lw[i].assign(layer_w[i], layer_w[i] + rows * cols);
                hs.lb[i].assign(layer_b[i], layer_b[i] + rows);
            }
        }
        build_scene(h->c, hs, device);
    });
    if (rc)
    {
        destroy(h);
        return rc;
    }
    *out = h;
    return SWR_OK;
}

void swr_scene_destroy(swr_ctx *ctx) { destroy(ctx); }

int swr_scene_get_arrays(swr_ctx *ctx, float *center_raw, float *cholesky, float *atten_logit, float *response)
{
    return guarded([&] {
        const HostScene &h = *ctx->c.host;
        auto put = [](float *dst, const std::vector<float> &v) {
            if (dst && !v.empty())
                std::memcpy(dst, v.data(), v.size() * sizeof(float));
        };
        put(center_raw, h.center_raw);
        put(cholesky, h.cholesky);
        put(atten_logit, h.atten);
        put(response, h.response);
    });
}

int swr_scene_get_layer(swr_ctx *ctx, int layer, int *rows, int *cols, float *w, float *b)
{
    return guarded([&] {
        const HostScene &h = *ctx->c.host;
        if (h.lw.empty())
            throw std::invalid_argument("scene has no deform net");
        if (layer < 0 || layer >= int(h.lw.size()))
            throw std::invalid_argument("layer index out of range");
        const int r = int(h.lb[layer].size());
        const int cl = r > 0 ? int(h.lw[layer].size() / size_t(r)) : 0;
        if (rows)
            *rows = r;
        if (cols)
            *cols = cl;
        if (w)
            std::memcpy(w, h.lw[layer].data(), h.lw[layer].size() * sizeof(float));
        if (b)
            std::memcpy(b, h.lb[layer].data(), h.lb[layer].size() * sizeof(float));
    });
}

int swr_scene_get_meta(swr_ctx *ctx, int64_t *iteration, uint64_t *manifest_hash)
{
    return guarded([&] {
        if (iteration)
            *iteration = ctx->c.host->iteration;
        if (manifest_hash)
            *manifest_hash = ctx->c.manifest_hash;
    });
}

int swr_scene_get_info(swr_ctx *ctx, swr_scene_info *info)
{
    return guarded([&] {
    Ctx &c = ctx->c;
    info->n_elevation = c.g.H;
    info->n_azimuth = c.g.W;
    info->n = c.g.n;
    info->width = c.has_net ? c.net.width : 0;
    info->bands_center = c.has_net ? c.net.bands_c : 0;
    info->bands_position = c.has_net ? c.net.bands_p : 0;
    info->cutoff_radius = c.cutoff;
    info->tile = c.tile;
    for (int a = 0; a < 3; a++)
    {
        info->bbox_min[a] = c.bbox_min[a];
        info->bbox_max[a] = c.bbox_max[a];
    }
    if (!c.pairs_on_host && c.w.stats)
    {
        // the async chunk path leaves the count on the device (ordered after the last call)
        int64_t p = 0;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        check_cuda(cudaStreamSynchronize(c.stream), "pair count");
        if (c.order_pending)
            check_cuda(cudaEventSynchronize(c.order_ev), "pair count");
        check_cuda(cudaMemcpy(&p, c.w.stats, sizeof(p), cudaMemcpyDeviceToHost), "pair count");
        c.pairs_last = p;
        c.pairs_on_host = true;
    }
    info->pairs_last = c.pairs_last;
    });
}

int swr_set_option(swr_ctx *ctx, const char *key, double value)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        const std::string k(key);
        if (k == "mlp_precision")
        {
            const int v = int(value);
            if (v < 0 || v > 2)
                throw std::invalid_argument("mlp_precision must be 0 (fp32), 1 (fp16x3) or 2 (fp16)");
            if (v != 0 && !(mlp_tc_available() && c.has_net && (c.net.wp == 160 || c.net.wp == 512)))
                throw std::invalid_argument("tensor-core MLP unavailable for this scene");
            if (v == 2 && c.net.wp == 512)
                throw std::invalid_argument("the single-pass fp16 tier exists for widths <= 160 only");
            c.mlp_precision = v;
        }
        else if (k == "chunk")
        {
            if (value < 1)
                throw std::invalid_argument("chunk must be >= 1");
            c.chunk = int(std::min<double>(value, c.chunk_cap)); // pair offsets stay 32-bit
        }
        else if (k == "mlp_max_clusters")
            c.mlp_max_clusters = int(value);
        else if (k == "mlp_smem_pad")
            c.mlp_smem_pad = int(value);
        else if (k == "copy_chunk")
        {
            if (value < 32)
                throw std::invalid_argument("copy_chunk must be >= 32");
            c.copy_chunk = int(std::min<double>(value, c.chunk_cap));
        }
        else if (k == "rssi_slope")
        {
            c.rssi_slope = value;
            c.rssi_calibrated = true;
        }
        else if (k == "rssi_intercept")
        {
            c.rssi_intercept = value;
            c.rssi_calibrated = true;
        }
        else if (k == "stage_timing")
            c.stage_timing = value != 0.0;
        else if (k == "async_pair_budget") // bytes; < 0: the default min(24 GiB, memory / 4); 0 forces the sync path
            c.async_pair_budget = int64_t(value);
        else if (k == "wide_block_rows")
        {
            if (value < 256)
                throw std::invalid_argument("wide_block_rows must be >= 256");
            c.wide_block_rows = int64_t(value);
        }
        else if (k == "stage_reset")
        {
            resolve_stage_times(c, false);
            std::fill(c.stage_ms, c.stage_ms + 6, 0.0);
        }
        else
            throw std::invalid_argument("unknown option " + k);
    });
}

int swr_get_option(swr_ctx *ctx, const char *key, double *value)
{
    return guarded([&] {
        const Ctx &c = ctx->c;
        const std::string k(key);
        if (k == "mlp_precision")
            *value = c.mlp_precision;
        else if (k == "chunk")
            *value = c.chunk;
        else if (k == "copy_chunk")
            *value = c.copy_chunk;
        else if (k == "rssi_slope")
            *value = c.rssi_slope;
        else if (k == "rssi_intercept")
            *value = c.rssi_intercept;
        else if (k == "stage_timing")
            *value = c.stage_timing ? 1.0 : 0.0;
        else if (k == "mlp_reruns")
        {
            unsigned long long d = 0;
            if (c.w.reruns)
            {
                check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
                check_cuda(cudaDeviceSynchronize(), "rerun count");
                check_cuda(cudaMemcpy(&d, c.w.reruns, sizeof(d), cudaMemcpyDeviceToHost), "rerun count");
            }
            *value = double(c.mlp_reruns + int64_t(d));
        }
        else if (k == "chunk_cap")
            *value = c.chunk_cap;
        else if (k == "device")
            *value = c.device;
        else if (k == "wide_block_rows")
            *value = double(c.wide_block_rows);
        else if (k == "pairs_per_position_max")
            *value = double(c.pairs_per_pos_max);
        else if (k == "rssi_calibrated")
            *value = c.rssi_calibrated ? 1.0 : 0.0;
        else if (k == "mlp_act_scale_exp") // smallest of the per-layer exponents
            *value = *std::min_element(c.net.tc_ascale, c.net.tc_ascale + 8);
        else if (k == "mlp_probe_amax")
            *value = *std::max_element(c.net.tc_amax, c.net.tc_amax + 8);
        else
            throw std::invalid_argument("unknown option " + k);
    });
}

// RSSI needs the affine calibration of an RSSI model (load_rssi_model throws the
// same way on a checkpoint without it, tasks.cpp:146-147)
static void check_rssi(const Ctx &c, uint32_t flags)
{
    if ((flags & SWR_OUT_RSSI) && !c.rssi_calibrated)
        throw std::runtime_error("scene is not an RSSI model (no calibration in trailer); set the rssi_slope / "
                                 "rssi_intercept options");
}

int swr_render_device(swr_ctx *ctx, const float *d_pos, int64_t B, uint32_t flags, float *d_spec, double *d_pooled,
                      double *d_rssi, int32_t *d_aoa_rc, double *d_aoa_ang, void *stream)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_rssi(c, flags);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        cudaStream_t st = stream ? (cudaStream_t)stream : c.stream;
        StreamOrder order(c, st, true);
        device_render(c, d_pos, B, flags, d_spec, d_pooled, d_rssi, d_aoa_rc, d_aoa_ang, st);
    });
}

int swr_render(swr_ctx *ctx, const float *pos_m, int64_t B, uint32_t flags, float *spectra, double *pooled,
               double *rssi, int32_t *aoa_rc, double *aoa_ang)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_rssi(c, flags);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        cudaStream_t st = c.stream;
        StreamOrder order(c, st);
        // host buffers: chunks of at most 256 positions once the batch exceeds that, so
        // every chunk's spectra copy out while the next chunk's MLP runs (the copy of a
        // 1,024-position batch takes ~4.7 ms at ~56 GB/s -- longer than the raster alone
        // at 10k Gaussians, 4.3 ms -- so copies left to the end would stay exposed)
        int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        if ((flags & SWR_OUT_SPECTRA) && spectra && chunk > c.copy_chunk)
            chunk = c.copy_chunk;
        ensure_work(c, chunk);
        const size_t per = size_t(2) * c.g.H * c.g.W;
        // device staging (kept in the context across calls): positions, two
        // spectrum chunk buffers (compute of chunk i+1 overlaps the D2H of chunk i),
        // head outputs; a copy stream and its events
        const bool want_spec = (flags & SWR_OUT_SPECTRA) && spectra;
        Stage &S = stage_for(c, B, chunk, want_spec ? per * chunk : 0);
        float *d_pos = S.pos;
        float *d_spec[2] = {S.spec[0], S.spec[1]};
        double *d_pooled = S.pooled, *d_rssi = S.rssi, *d_ang = S.ang;
        int32_t *d_rc = S.rc;
        cudaStream_t copy_st = S.copy;
        cudaEvent_t *done = S.done, *freed = S.freed;
        const bool use_mlp = c.has_net && !(flags & SWR_NO_RESIDUALS);
        if (use_mlp && c.g.n < 1)
            throw std::invalid_argument("empty gaussian set"); // predict_residuals (deform.cpp:147-148) via render_at
        check_cuda(cudaMemcpyAsync(d_pos, pos_m, sizeof(float) * 3 * B, cudaMemcpyHostToDevice, st), "H2D positions");
        const bool heads = flags & (SWR_OUT_POOLED | SWR_OUT_RSSI | SWR_OUT_AOA);
        int k = 0;
        // chunk sizes: `chunk` each; with spectra going to the host, the last one is halved,
        // so the copy backlog it leaves behind the last raster slice is shorter (at 10k
        // Gaussians PCIe moves ~216k spectra/s, the raster ~250k/s)
        std::vector<int64_t> sizes;
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
            sizes.push_back(std::min<int64_t>(chunk, B - b0));
        if (want_spec && sizes.size() > 1 && sizes.back() >= 2 * 64)
        {
            const int64_t last = sizes.back();
            sizes.back() = last - last / 2;
            sizes.push_back(last / 2);
        }
        int64_t b0 = 0;
        for (size_t ci = 0; ci < sizes.size(); b0 += sizes[ci], ci++, k ^= 1)
        {
            const int nb = int(sizes[ci]);
            if (want_spec && ci >= 2)
                check_cuda(cudaStreamWaitEvent(st, freed[k], 0), "wait copy");
            // the raster of a chunk above 256 positions runs in 256-position slices, each
            // slice's spectra copied out right behind it (smaller slices lengthen the
            // raster's launch tails more than they shorten the exposed copy)
            auto copy_slice = [&](int s0, int n) {
                check_cuda(cudaEventRecord(done[k], st), "record");
                check_cuda(cudaStreamWaitEvent(copy_st, done[k], 0), "wait compute");
                check_cuda(cudaMemcpyAsync(spectra + per * (b0 + s0), d_spec[k] + per * s0, sizeof(float) * per * n,
                                           cudaMemcpyDeviceToHost, copy_st),
                           "D2H spectra");
            };
            run_chunk(c, d_pos + 3 * b0, nb, false, use_mlp, false, want_spec ? d_spec[k] : nullptr, heads, flags,
                      d_pooled + b0, d_rssi + b0, d_rc + 2 * b0, d_ang + 2 * b0, st,
                      want_spec ? copy_slices(nb, ci + 1 == sizes.size(), c.copy_chunk) : std::vector<int>(),
                      want_spec ? std::function<void(int, int)>(copy_slice) : std::function<void(int, int)>());
            if (want_spec)
                check_cuda(cudaEventRecord(freed[k], copy_st), "record");
        }
        if (pooled && (flags & SWR_OUT_POOLED))
            check_cuda(cudaMemcpyAsync(pooled, d_pooled, sizeof(double) * B, cudaMemcpyDeviceToHost, st), "D2H");
        if (rssi && (flags & SWR_OUT_RSSI))
            check_cuda(cudaMemcpyAsync(rssi, d_rssi, sizeof(double) * B, cudaMemcpyDeviceToHost, st), "D2H");
        if (aoa_rc && (flags & SWR_OUT_AOA))
            check_cuda(cudaMemcpyAsync(aoa_rc, d_rc, sizeof(int32_t) * 2 * B, cudaMemcpyDeviceToHost, st), "D2H");
        if (aoa_ang && (flags & SWR_OUT_AOA))
            check_cuda(cudaMemcpyAsync(aoa_ang, d_ang, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "render");
        check_cuda(cudaStreamSynchronize(copy_st), "render copies");
        (void)is_pinned;
    });
}

int swr_normalize_positions(swr_ctx *ctx, const float *pos_m, int64_t B, float *pos01)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        for (int64_t b = 0; b < B; b++)
            for (int a = 0; a < 3; a++)
            {
                const double range = c.bbox_max[a] - c.bbox_min[a];
                pos01[3 * b + a] = range > 0.0 ? float((double(pos_m[3 * b + a]) - c.bbox_min[a]) / range) : 0.5f;
            }
    });
}

int swr_predict_residuals(swr_ctx *ctx, const float *pos01, int64_t B, float *dc, float *dr, float *da)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (!c.has_net)
            throw std::invalid_argument("deform net is not initialized");
        if (c.g.n < 1)
            throw std::invalid_argument("empty gaussian set");
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        ensure_work(c, chunk);
        float *d_pos = dalloc<float>(c, size_t(3) * std::max<int64_t>(B, 1));
        check_cuda(cudaMemcpy(d_pos, pos01, sizeof(float) * 3 * B, cudaMemcpyHostToDevice), "H2D");
        const int n = c.g.n, np = c.g.np;
        std::vector<float> planes(size_t(5) * c.w.cap_b * np);
        const size_t plane = size_t(c.w.cap_b) * np;
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            launch_pos_prep(c, d_pos + 3 * b0, nb, true, c.stream);
            launch_mlp(c, nb, c.stream);
            check_cuda(cudaGetLastError(), "launch");
            auto fetch = [&] {
                check_cuda(cudaMemcpyAsync(planes.data(), c.w.res, planes.size() * sizeof(float),
                                           cudaMemcpyDeviceToHost, c.stream),
                           "D2H residuals");
                check_cuda(cudaStreamSynchronize(c.stream), "predict");
            };
            fetch();
            if (c.mlp_precision != 0)
            {
                bool bad = false;
                for (int q = 0; q < 5 && !bad; q++)
                    for (int s = 0; s < nb && !bad; s++)
                        for (int g = 0; g < n; g++)
                            if (!std::isfinite(planes[q * plane + size_t(s) * np + g]))
                            {
                                bad = true;
                                break;
                            }
                if (bad) // fp16 overflow in the tensor-core MLP: this chunk again in FP32 (see run_chunk)
                {
                    c.mlp_reruns++;
                    const int keep = c.mlp_precision;
                    c.mlp_precision = 0;
                    launch_pos_prep(c, d_pos + 3 * b0, nb, true, c.stream);
                    launch_mlp(c, nb, c.stream);
                    c.mlp_precision = keep;
                    fetch();
                }
            }
            for (int s = 0; s < nb; s++)
                for (int g = 0; g < n; g++)
                {
                    const size_t src = size_t(s) * np + g, dst = size_t(b0 + s) * n + g;
                    dc[2 * dst] = planes[0 * plane + src];
                    dc[2 * dst + 1] = planes[1 * plane + src];
                    dr[2 * dst] = planes[2 * plane + src];
                    dr[2 * dst + 1] = planes[3 * plane + src];
                    da[dst] = planes[4 * plane + src];
                }
        }
        dfree(c, d_pos);
    });
}

int swr_setup(swr_ctx *ctx, const float *dc, const float *dr, const float *da, int64_t B, float *state, int32_t *rows,
              int32_t *cols, int32_t *tile_count)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        ensure_work(c, chunk);
        const int n = c.g.n, np = c.g.np;
        const bool with_res = dc != nullptr;
        float *d_state = dalloc<float>(c, size_t(chunk) * n * kStateStride);
        std::vector<int4> rng(size_t(chunk) * np);
        std::vector<int> cnt(size_t(chunk) * np);
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            if (with_res)
                upload_residuals(c, dc, dr, da, b0, nb);
            launch_setup(c, nb, with_res, c.stream);
            launch_state_out(c, nb, with_res, d_state, c.stream);
            check_cuda(cudaGetLastError(), "launch");
            if (state)
                check_cuda(cudaMemcpyAsync(state + size_t(b0) * n * kStateStride, d_state,
                                           sizeof(float) * nb * n * kStateStride, cudaMemcpyDeviceToHost, c.stream),
                           "D2H state");
            check_cuda(cudaMemcpyAsync(rng.data(), c.w.rng, sizeof(int4) * nb * np, cudaMemcpyDeviceToHost, c.stream),
                       "D2H ranges");
            check_cuda(cudaMemcpyAsync(cnt.data(), c.w.cnt, sizeof(int) * nb * np, cudaMemcpyDeviceToHost, c.stream),
                       "D2H counts");
            check_cuda(cudaStreamSynchronize(c.stream), "setup");
            for (int s = 0; s < nb; s++)
                for (int g = 0; g < n; g++)
                {
                    const int4 b = rng[size_t(s) * np + g];
                    const size_t d = size_t(b0 + s) * n + g;
                    if (rows)
                    {
                        rows[2 * d] = b.x;
                        rows[2 * d + 1] = b.y;
                    }
                    if (cols)
                    {
                        cols[2 * d] = b.z;
                        cols[2 * d + 1] = b.w;
                    }
                    if (tile_count)
                        tile_count[d] = cnt[size_t(s) * np + g];
                }
        }
        dfree(c, d_state);
    });
}

static void bins_for(Ctx &c, const float *dc, const float *dr, const float *da, int64_t B, int32_t *tile_offset,
                     int32_t *tile_prims, int64_t cap, int64_t *n_pairs, float *spectra)
{
    check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
    StreamOrder order(c, c.stream);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
    ensure_work(c, chunk);
    const bool with_res = dc != nullptr;
    const int tiles = c.g.tiles;
    const size_t per = size_t(2) * c.g.H * c.g.W;
    float *d_spec = spectra ? dalloc<float>(c, per * chunk) : nullptr;
    int64_t written = 0;
    std::vector<int64_t> seg(chunk + 1);
    for (int64_t b0 = 0; b0 < B; b0 += chunk)
    {
        const int nb = int(std::min<int64_t>(chunk, B - b0));
        if (with_res)
            upload_residuals(c, dc, dr, da, b0, nb);
        run_chunk(c, nullptr, nb, true, false, with_res, d_spec, false, 0, nullptr, nullptr, nullptr, nullptr,
                  c.stream, {}, {}, true);
        const int64_t pairs = c.pairs_last;
        if (tile_offset)
            check_cuda(cudaMemcpyAsync(tile_offset + size_t(b0) * (tiles + 1), c.w.tile_off,
                                       sizeof(int) * nb * (tiles + 1), cudaMemcpyDeviceToHost, c.stream),
                       "D2H offsets");
        if (tile_prims && written < cap)
            check_cuda(cudaMemcpyAsync(tile_prims + written, c.w.sorted,
                                       sizeof(int) * std::min<int64_t>(pairs, cap - written), cudaMemcpyDeviceToHost,
                                       c.stream),
                       "D2H prims");
        if (spectra)
            check_cuda(cudaMemcpyAsync(spectra + per * b0, d_spec, sizeof(float) * per * nb, cudaMemcpyDeviceToHost,
                                       c.stream),
                       "D2H spectra");
        check_cuda(cudaStreamSynchronize(c.stream), "bins");
        written += pairs;
    }
    if (n_pairs)
        *n_pairs = written;
    if (d_spec)
        dfree(c, d_spec);
}

int swr_bin(swr_ctx *ctx, const float *dc, const float *dr, const float *da, int64_t B, int32_t *tile_offset,
            int32_t *tile_prims, int64_t cap, int64_t *n_pairs)
{
    return guarded([&] { bins_for(ctx->c, dc, dr, da, B, tile_offset, tile_prims, cap, n_pairs, nullptr); });
}

int swr_rasterize(swr_ctx *ctx, const float *dc, const float *dr, const float *da, int64_t B, float *spectra)
{
    return guarded([&] { bins_for(ctx->c, dc, dr, da, B, nullptr, nullptr, 0, nullptr, spectra); });
}

int swr_heads(swr_ctx *ctx, const float *spectra, int64_t B, double *pooled, int32_t *aoa_rc, double *aoa_ang)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        ensure_work(c, chunk);
        const size_t per = size_t(2) * c.g.H * c.g.W;
        float *d_spec = dalloc<float>(c, per * chunk);
        double *d_pooled = dalloc<double>(c, chunk), *d_ang = dalloc<double>(c, 2 * chunk);
        int32_t *d_rc = dalloc<int32_t>(c, 2 * chunk);
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            check_cuda(cudaMemcpyAsync(d_spec, spectra + per * b0, sizeof(float) * per * nb, cudaMemcpyHostToDevice,
                                       c.stream),
                       "H2D spectra");
            launch_heads_from_spectra(c, nb, d_spec, c.stream);
            launch_heads(c, nb, SWR_OUT_POOLED | SWR_OUT_AOA, d_pooled, nullptr, d_rc, d_ang, c.stream);
            check_cuda(cudaGetLastError(), "launch");
            if (pooled)
                check_cuda(cudaMemcpyAsync(pooled + b0, d_pooled, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream),
                           "D2H");
            if (aoa_rc)
                check_cuda(cudaMemcpyAsync(aoa_rc + 2 * b0, d_rc, sizeof(int32_t) * 2 * nb, cudaMemcpyDeviceToHost,
                                           c.stream),
                           "D2H");
            if (aoa_ang)
                check_cuda(cudaMemcpyAsync(aoa_ang + 2 * b0, d_ang, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost,
                                           c.stream),
                           "D2H");
            check_cuda(cudaStreamSynchronize(c.stream), "heads");
        }
        for (void *p : {(void *)d_spec, (void *)d_pooled, (void *)d_ang, (void *)d_rc})
            dfree(c, p);
    });
}

int64_t swr_launch_count(swr_ctx *ctx) { return ctx->c.launches; }

// ------------------------------------------------------------- metrics

static void metrics_workspace(Ctx &c, int nb)
{
    Work &w = c.w;
    if (nb <= w.met_cap)
        return;
    for (void *p : {(void *)w.met_tmp, (void *)w.met_bad, (void *)w.met_out, (void *)w.met_pred, (void *)w.met_target})
        dfree(c, p);
    const size_t per = size_t(2) * c.g.H * c.g.W;
    w.met_tmp = dalloc<double>(c, metrics_tmp_doubles(c, nb));
    w.met_bad = dalloc<int>(c, 1);
    w.met_out = dalloc<double>(c, size_t(3) * nb);
    w.met_pred = dalloc<float>(c, per * nb);
    w.met_target = dalloc<float>(c, per * nb);
    w.met_cap = nb;
}

static void check_metric_args(const Ctx &c, bool want_ssim)
{
    if (want_ssim && (c.g.H < 11 || c.g.W < 11))
        throw std::invalid_argument("grid too small for the 11x11 SSIM window");
}

static void raise_if_nonfinite(Ctx &c, cudaStream_t st)
{
    int bad = 0;
    check_cuda(cudaMemcpyAsync(&bad, c.w.met_bad, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H metric flag");
    check_cuda(cudaStreamSynchronize(st), "metrics");
    if (bad)
        throw std::domain_error("spectrum contains a non-finite value");
}

int swr_metrics_device(swr_ctx *ctx, const float *d_pred, const float *d_target, int64_t B, double peak,
                       double *d_psnr, double *d_ssim, double *d_l1, void *stream)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_metric_args(c, d_ssim != nullptr);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c.stream;
        StreamOrder order(c, st);
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        metrics_workspace(c, int(chunk));
        check_cuda(cudaMemsetAsync(c.w.met_bad, 0, sizeof(int), st), "memset");
        const size_t per = size_t(2) * c.g.H * c.g.W;
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            launch_metrics(c, d_pred + per * b0, d_target + per * b0, nb, peak, d_psnr ? d_psnr + b0 : nullptr,
                           d_ssim ? d_ssim + b0 : nullptr, d_l1 ? d_l1 + b0 : nullptr, c.w.met_tmp, c.w.met_bad, st);
        }
        check_cuda(cudaGetLastError(), "metrics launch");
        raise_if_nonfinite(c, st);
    });
}

// host buffers: per chunk H2D of both spectra, metrics on device, D2H of 3 doubles per pair
int swr_metrics(swr_ctx *ctx, const float *pred, const float *target, int64_t B, double peak, double *psnr,
                double *ssim, double *l1)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_metric_args(c, ssim != nullptr);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        cudaStream_t st = c.stream;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        metrics_workspace(c, int(chunk));
        check_cuda(cudaMemsetAsync(c.w.met_bad, 0, sizeof(int), st), "memset");
        const size_t per = size_t(2) * c.g.H * c.g.W;
        double *o = c.w.met_out;
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            check_cuda(cudaMemcpyAsync(c.w.met_pred, pred + per * b0, sizeof(float) * per * nb, cudaMemcpyHostToDevice,
                                       st),
                       "H2D prediction");
            check_cuda(cudaMemcpyAsync(c.w.met_target, target + per * b0, sizeof(float) * per * nb,
                                       cudaMemcpyHostToDevice, st),
                       "H2D target");
            launch_metrics(c, c.w.met_pred, c.w.met_target, nb, peak, o, ssim ? o + chunk : nullptr, o + 2 * chunk,
                           c.w.met_tmp, c.w.met_bad, st);
            for (int k = 0; k < 3; k++)
            {
                double *dst = k == 0 ? psnr : (k == 1 ? ssim : l1);
                if (dst)
                    check_cuda(cudaMemcpyAsync(dst + b0, o + k * chunk, sizeof(double) * nb, cudaMemcpyDeviceToHost, st),
                               "D2H metrics");
            }
            check_cuda(cudaStreamSynchronize(st), "metrics chunk");
        }
        raise_if_nonfinite(c, st);
    });
}

// train::evaluate (training.cpp:380-406) batched: render every position and
// compare with its target spectrum on the device; only the 3 metrics per
// sample come back (the spectra never leave the GPU)
int swr_evaluate(swr_ctx *ctx, const float *pos_m, const float *target, int64_t B, double peak, double *psnr,
                 double *ssim, double *l1)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_metric_args(c, ssim != nullptr);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        cudaStream_t st = c.stream;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        ensure_work(c, chunk);
        metrics_workspace(c, int(chunk));
        check_cuda(cudaMemsetAsync(c.w.met_bad, 0, sizeof(int), st), "memset");
        const size_t per = size_t(2) * c.g.H * c.g.W;
        float *d_pos = dalloc<float>(c, size_t(3) * B);
        check_cuda(cudaMemcpyAsync(d_pos, pos_m, sizeof(float) * 3 * B, cudaMemcpyHostToDevice, st), "H2D positions");
        const bool use_mlp = c.has_net;
        double *o = c.w.met_out;
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            check_cuda(cudaMemcpyAsync(c.w.met_target, target + per * b0, sizeof(float) * per * nb,
                                       cudaMemcpyHostToDevice, st),
                       "H2D target");
            run_chunk(c, d_pos + 3 * b0, nb, false, use_mlp, false, c.w.met_pred, false, 0, nullptr, nullptr, nullptr,
                      nullptr, st);
            launch_metrics(c, c.w.met_pred, c.w.met_target, nb, peak, o, ssim ? o + chunk : nullptr, o + 2 * chunk,
                           c.w.met_tmp, c.w.met_bad, st);
            for (int k = 0; k < 3; k++)
            {
                double *dst = k == 0 ? psnr : (k == 1 ? ssim : l1);
                if (dst)
                    check_cuda(cudaMemcpyAsync(dst + b0, o + k * chunk, sizeof(double) * nb, cudaMemcpyDeviceToHost, st),
                               "D2H metrics");
            }
            check_cuda(cudaStreamSynchronize(st), "evaluate chunk");
        }
        dfree(c, d_pos);
        raise_if_nonfinite(c, st);
    });
}

// train::evaluate (training.cpp:380-406) over a dataset split, streamed from
// spectra.bin chunk by chunk (positions + targets of c.chunk samples at a time)
int swr_evaluate_dataset(swr_ctx *ctx, swr_dataset *ds, int split, int32_t *sample_ids, double *psnr, double *ssim,
                         double *l1)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        const DatasetFile &d = ds->d;
        if (c.manifest_hash != d.hash)
            throw std::runtime_error("checkpoint was trained on a different dataset"); // train::hash_mismatch
        if (d.H != c.g.H || d.W != c.g.W)
            throw std::invalid_argument("spectrum shape mismatch");
        if (split < 0 || split > 2)
            throw std::invalid_argument("split must be 0 (train), 1 (test) or 2 (all)");
        const std::vector<int> idx = d.split(split);
        const int64_t B = int64_t(idx.size());
        if (sample_ids)
            std::memcpy(sample_ids, idx.data(), sizeof(int32_t) * idx.size());
        if (B == 0)
            return;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        const size_t per = size_t(2) * c.g.H * c.g.W;
        std::vector<float> pos(size_t(3) * chunk), tgt(per * chunk);
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int64_t nb = std::min<int64_t>(chunk, B - b0);
            d.read(idx.data() + b0, nb, pos.data(), tgt.data());
            const int rc = swr_evaluate(ctx, pos.data(), tgt.data(), nb, 1.0, psnr ? psnr + b0 : nullptr,
                                        ssim ? ssim + b0 : nullptr, l1 ? l1 + b0 : nullptr);
            if (rc == SWR_EDOMAIN)
                throw std::domain_error(g_err);
            if (rc != SWR_OK)
                throw std::runtime_error(g_err);
        }
    });
}

// ------------------------------------------------------------ backward

// splat::rasterize_backward (splat.cpp:494-669) per position: residuals as
// swr_rasterize (nullable), upstream [B][H][W][2]; outputs [B][n][...] in the
// reference's RenderGrads layout (splat.hpp:77-89), any may be NULL
int swr_rasterize_backward(swr_ctx *ctx, const float *dc, const float *dr, const float *da, int64_t B,
                           const float *upstream, float *g_center_raw, float *g_cholesky, float *g_atten_logit,
                           float *g_response, float *g_d_center, float *g_d_response, float *g_d_atten)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        cudaStream_t st = c.stream;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        ensure_work(c, chunk);
        const bool with_res = dc != nullptr;
        const int n = c.g.n;
        const size_t per = size_t(2) * c.g.H * c.g.W;
        float *d_state = dalloc<float>(c, size_t(chunk) * std::max(n, 1) * 11);
        float *d_up = dalloc<float>(c, per * chunk);
        const int widths[7] = {2, 3, 1, 2, 2, 2, 1};
        float *host_out[7] = {g_center_raw, g_cholesky, g_atten_logit, g_response, g_d_center, g_d_response, g_d_atten};
        float *d_out[7];
        for (int k = 0; k < 7; k++)
            d_out[k] = dalloc<float>(c, size_t(chunk) * std::max(n, 1) * widths[k]);
        float *d_slots = nullptr;
        int64_t slots_cap = 0;
        c.w.want_perm = true;
        try
        {
            for (int64_t b0 = 0; b0 < B; b0 += chunk)
            {
                const int nb = int(std::min<int64_t>(chunk, B - b0));
                if (with_res)
                    upload_residuals(c, dc, dr, da, b0, nb);
                check_cuda(cudaMemcpyAsync(d_up, upstream + per * b0, sizeof(float) * per * nb, cudaMemcpyHostToDevice,
                                           st),
                           "H2D upstream");
                // the forward's setup + bins (state, boxes, CSR lists) with the sort permutation
                launch_setup(c, nb, with_res, st);
                launch_bin_count(c, nb, st);
                check_cuda(cudaMemcpyAsync(c.w.host_pairs, c.w.stats, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                           "D2H pair count");
                check_cuda(cudaStreamSynchronize(st), "pair count");
                const int64_t pairs = c.w.host_pairs[0], max_seg = c.w.host_pairs[1];
                ensure_pairs(c, pairs, nb, max_seg);
                launch_bin_sort(c, nb, pairs, int(max_seg), st);
                launch_state_out(c, nb, with_res, d_state, st);
                if (pairs > slots_cap)
                {
                    dfree(c, d_slots);
                    slots_cap = std::max<int64_t>(pairs, 1);
                    d_slots = dalloc<float>(c, size_t(slots_cap) * 8);
                }
                launch_raster_backward(c, nb, d_state, d_up, d_slots, st);
                launch_bwd_merge(c, nb, with_res, d_slots, d_out, st);
                check_cuda(cudaGetLastError(), "backward launch");
                for (int k = 0; k < 7; k++)
                    if (host_out[k])
                        check_cuda(cudaMemcpyAsync(host_out[k] + size_t(b0) * n * widths[k], d_out[k],
                                                   sizeof(float) * size_t(nb) * n * widths[k], cudaMemcpyDeviceToHost,
                                                   st),
                                   "D2H grads");
                check_cuda(cudaStreamSynchronize(st), "backward");
            }
        }
        catch (...)
        {
            c.w.want_perm = false;
            throw;
        }
        c.w.want_perm = false;
        for (void *p : {(void *)d_state, (void *)d_up, (void *)d_slots})
            dfree(c, p);
        for (float *p : d_out)
            dfree(c, p);
    });
}

// hybrid_loss (training.cpp:62-106) for B (prediction, target) pairs: terms
// [B][3] = (loss, l1_term, ssim_term); grad [B][H][W][2] (NULL: value only)
int swr_hybrid_loss(swr_ctx *ctx, const float *pred, const float *target, int64_t B, double lambda1, double *terms,
                    float *grad)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        if (B < 0)
            throw std::invalid_argument("negative batch");
        check_metric_args(c, true);
        if (B == 0)
            return;
        check_cuda(cudaSetDevice(c.device), "cudaSetDevice");
        StreamOrder order(c, c.stream);
        cudaStream_t st = c.stream;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, c.chunk));
        metrics_workspace(c, int(chunk));
        const size_t per = size_t(2) * c.g.H * c.g.W;
        double *d_tmp = dalloc<double>(c, loss_tmp_doubles(c, int(chunk)));
        double *d_terms = dalloc<double>(c, size_t(3) * chunk);
        float *d_grad = grad ? dalloc<float>(c, per * chunk) : nullptr;
        check_cuda(cudaMemsetAsync(c.w.met_bad, 0, sizeof(int), st), "memset");
        for (int64_t b0 = 0; b0 < B; b0 += chunk)
        {
            const int nb = int(std::min<int64_t>(chunk, B - b0));
            check_cuda(cudaMemcpyAsync(c.w.met_pred, pred + per * b0, sizeof(float) * per * nb, cudaMemcpyHostToDevice,
                                       st),
                       "H2D prediction");
            check_cuda(cudaMemcpyAsync(c.w.met_target, target + per * b0, sizeof(float) * per * nb,
                                       cudaMemcpyHostToDevice, st),
                       "H2D target");
            launch_hybrid_loss(c, c.w.met_pred, c.w.met_target, nb, lambda1, d_terms, d_grad, d_tmp, c.w.met_bad, st);
            if (terms)
                check_cuda(cudaMemcpyAsync(terms + 3 * b0, d_terms, sizeof(double) * 3 * nb, cudaMemcpyDeviceToHost, st),
                           "D2H loss");
            if (grad)
                check_cuda(cudaMemcpyAsync(grad + per * b0, d_grad, sizeof(float) * per * nb, cudaMemcpyDeviceToHost, st),
                           "D2H loss gradient");
            check_cuda(cudaStreamSynchronize(st), "loss");
        }
        for (void *p : {(void *)d_tmp, (void *)d_terms, (void *)d_grad})
            dfree(c, p);
        raise_if_nonfinite(c, st);
    });
}

int swr_scene_set_manifest_hash(swr_ctx *ctx, uint64_t hash)
{
    ctx->c.manifest_hash = hash;
    return SWR_OK;
}

int swr_debug_mlp_trace2(long long *out)
{
    return swr::mlp_tc2_trace(out);
}

// debug: after a render, time (ms) the MLP alone, the raster (8 / 4 warps) alone
// and the MLP concurrent with the raster on a second stream: out[0..5] =
// mlp, r8, r4, mlp||r4 (both done), mlp||r8, nb
int swr_debug_overlap(swr_ctx *ctx, double *out)
{
    return guarded([&] {
        Ctx &c = ctx->c;
        const int nb = (int)c.w.cap_b;
        cudaStream_t a = c.stream, b;
        check_cuda(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "stream");
        cudaEvent_t e0, e1, e2;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        auto timed = [&](auto &&f) {
            cudaStreamSynchronize(a);
            cudaStreamSynchronize(b);
            cudaEventRecord(e0, a);
            cudaStreamWaitEvent(b, e0, 0);
            f();
            cudaEventRecord(e2, b);
            cudaStreamWaitEvent(a, e2, 0);
            cudaEventRecord(e1, a);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            return (double)ms;
        };
        out[0] = timed([&] { launch_mlp(c, nb, a); });
        out[1] = timed([&] { launch_raster(c, nb, nullptr, false, b, 2); });
        out[2] = timed([&] { launch_raster(c, nb, nullptr, false, b, 4); });
        out[3] = timed([&] {
            launch_mlp(c, nb, a);
            std::this_thread::sleep_for(std::chrono::microseconds(2000)); // MLP CTAs resident first
            launch_raster(c, nb, nullptr, false, b, 2);
        });
        out[4] = timed([&] {
            launch_mlp(c, nb, a);
            std::this_thread::sleep_for(std::chrono::microseconds(2000));
            launch_raster(c, nb, nullptr, false, b, 4);
        });
        out[5] = nb;
        check_cuda(cudaStreamSynchronize(a), "overlap");
        cudaStreamDestroy(b);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    });
}

int swr_stage_times(swr_ctx *ctx, double *ms6)
{
    resolve_stage_times(ctx->c, true);
    for (int i = 0; i < 6; i++)
        ms6[i] = ctx->c.stage_ms[i];
    return SWR_OK;
}

} // extern "C"
