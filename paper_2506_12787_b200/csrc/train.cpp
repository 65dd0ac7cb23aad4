// Device training loop: train::train
// (training.cpp:198-376) with every per-iteration step on the GPU.
//
// The reference draws everything random from one Rng (mt19937_64) whose stream
// does not depend on the training state: the initial Gaussians and network
// (init_random, splat.cpp:681-709; DeformNet::init, deform.cpp:73-102), then per
// iteration one sample index and, in the fine stage while the schedule is
// active, three normals of coordinate noise (training.cpp:116-128). The host
// replays that stream exactly; the device does the work:
//
//   coarse  setup -> bins -> raster -> hybrid loss + dL/dA -> state -> raster
//           backward -> merge -> Adam on all four Gaussian fields (+ width floors)
//   fine    position encoding -> 8 trunk layers (activations kept) -> heads into
//           the residual planes -> the same render / loss / backward with
//           residuals -> heads + trunk backward (dW split-K, dIN fused with the
//           ReLU mask) -> Adam on the network and on cholesky/atten/response
//
// The Gaussians' render inputs (SceneDev) are re-derived on the device by the
// Adam kernel after every step, so nothing returns to the host inside an
// iteration except the pair count the bin sort is sized by.
#include "swr.h"
#include "swr_internal.h"

#include <json.hpp>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace swr
{

namespace
{

// common.hpp:42-72 (uniform = top 53 bits; Box-Muller on two fresh uniforms)
struct RefRng
{
    std::mt19937_64 gen;
    explicit RefRng(uint64_t seed) : gen(seed) {}
    double uniform() { return double(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t index(uint64_t n) { return uint64_t(uniform() * double(n)) % n; }
    double normal()
    {
        const double u1 = double((gen() >> 11) + 1) * 0x1.0p-53;
        const double u2 = double(gen() >> 11) * 0x1.0p-53;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    }
};

// deform.cpp:54-70 on the host (float, glibc sinf/cosf like the reference)
void encode_host(const float *v, int count, int bands, float *out)
{
    for (int i = 0; i < count; i++)
        out[i] = v[i];
    float *blk = out + count;
    for (int k = 0; k < bands; k++)
    {
        const float f = float(std::ldexp(kPi, k));
        for (int i = 0; i < count; i++)
            blk[i] = std::sin(f * v[i]);
        for (int i = 0; i < count; i++)
            blk[count + i] = std::cos(f * v[i]);
        blk += 2 * count;
    }
}

nlohmann::json config_json(const swr_train_config &c)
{
    // config.cpp:84-102 keys
    nlohmann::json j;
    j["primitives"] = c.primitives;
    j["bands_center"] = c.bands_center;
    j["bands_position"] = c.bands_position;
    j["width"] = c.width;
    j["cutoff_radius"] = c.cutoff_radius;
    j["tile"] = c.tile;
    j["lr_gaussian"] = c.lr_gaussian;
    j["lr_mlp"] = c.lr_mlp;
    j["lambda1"] = c.lambda1;
    j["coarse_iters"] = c.coarse_iters;
    j["fine_iters"] = c.fine_iters;
    j["anneal_scale"] = c.anneal_scale;
    j["anneal_threshold"] = c.anneal_threshold;
    j["seed"] = c.seed;
    return j;
}

swr_train_config config_from_json(const std::string &text)
{
    const auto j = nlohmann::json::parse(text);
    swr_train_config c;
    swr_train_config_default(&c);
    auto get = [&](const char *k, auto &v) {
        if (j.contains(k))
            v = j.at(k).get<std::remove_reference_t<decltype(v)>>();
    };
    get("primitives", c.primitives);
    get("bands_center", c.bands_center);
    get("bands_position", c.bands_position);
    get("width", c.width);
    get("cutoff_radius", c.cutoff_radius);
    get("tile", c.tile);
    get("lr_gaussian", c.lr_gaussian);
    get("lr_mlp", c.lr_mlp);
    get("lambda1", c.lambda1);
    get("coarse_iters", c.coarse_iters);
    get("fine_iters", c.fine_iters);
    get("anneal_scale", c.anneal_scale);
    get("anneal_threshold", c.anneal_threshold);
    get("seed", c.seed);
    return c;
}

bool same_config(const swr_train_config &a, const swr_train_config &b)
{
    return a.primitives == b.primitives && a.bands_center == b.bands_center && a.bands_position == b.bands_position &&
           a.width == b.width && a.cutoff_radius == b.cutoff_radius && a.tile == b.tile &&
           a.lr_gaussian == b.lr_gaussian && a.lr_mlp == b.lr_mlp && a.lambda1 == b.lambda1 &&
           a.coarse_iters == b.coarse_iters && a.fine_iters == b.fine_iters && a.anneal_scale == b.anneal_scale &&
           a.anneal_threshold == b.anneal_threshold && a.seed == b.seed;
}

constexpr int kTrunkLayers = 8;
inline bool skip_layer(int i) { return i == 2 || i == 4 || i == 6; }

} // namespace

struct Trainer
{
    Ctx c;
    swr_train_config cfg{};
    RefRng rng{0};
    // dataset (on the device: every sample's spectrum, sample order)
    int H = 0, W = 0;
    int64_t samples = 0;
    std::vector<int> train_idx;
    std::vector<float> positions; // [samples][3]
    double bbox_min[3]{}, bbox_max[3]{};   // the checkpoint's (saved)
    double ds_min[3]{}, ds_max[3]{};       // the dataset's (normalizes training positions)
    uint64_t manifest_hash = 0;
    float *d_spectra = nullptr;
    // schedule
    int64_t iteration = 0, total = 0;
    bool in_fine = false, cenc_ready = false;
    // Gaussians
    int n = 0;
    GaussDev gp{};
    int64_t t_center = 0, t_rest = 0;
    // network: flat parameters [W0 b0 .. W7 b7 | Wh (head_center, head_response, head_atten rows) | bh]
    int width = 0, D = 0, Dc = 0, Dp = 0;
    int cols[kTrunkLayers]{};
    int64_t off_w[kTrunkLayers + 1]{}, off_b[kTrunkLayers + 1]{}, P = 0;
    float *net_p = nullptr, *net_g = nullptr, *net_m = nullptr, *net_v = nullptr;
    int64_t t_net = 0;
    float *x0 = nullptr, *h[kTrunkLayers]{}, *dz_a = nullptr, *dz_b = nullptr, *dr5 = nullptr, *part = nullptr;
    // per-iteration plan (device tables indexed by iteration - it_base) + cursor
    int64_t it_base = 0;
    int *d_sidx = nullptr;
    float *d_spenc = nullptr;
    double *d_sbc = nullptr, *d_log = nullptr;
    TrainSched sched{};
    int *g_sidx = nullptr; // one-entry plan of gradients()
    float *g_spenc = nullptr;
    double *g_sbc = nullptr;
    int64_t *g_it = nullptr;
    bool use_graphs = true;
    cudaGraphExec_t graph[2]{};
    int64_t graph_launches[2]{};
    // render / loss scratch (worst-case sized)
    int64_t pair_cap = 0;
    float *d_pred = nullptr, *d_lgrad = nullptr, *d_target = nullptr, *d_state = nullptr, *d_slots = nullptr;
    float *grads[7]{};
    double *d_tmp = nullptr, *d_terms = nullptr;
    int *d_bad = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    ~Trainer()
    {
        cudaSetDevice(c.device);
        if (ev0)
            cudaEventDestroy(ev0);
        if (ev1)
            cudaEventDestroy(ev1);
        for (void *p : c.allocs)
            cudaFree(p);
        if (c.w.host_pairs)
            cudaFreeHost(c.w.host_pairs);
        for (auto &gx : graph)
            if (gx)
                cudaGraphExecDestroy(gx);
        if (c.stream)
            cudaStreamDestroy(c.stream);
    }

    void reset_opt()
    {
        // training.cpp:257-268: fresh moments (the step counters restart in run()'s plan)
        cudaStream_t st = c.stream;
        for (float *p : {gp.m_center, gp.v_center})
            check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * 2 * std::max(n, 1), st), "memset");
        for (float *p : {gp.m_chol, gp.v_chol})
            check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * 3 * std::max(n, 1), st), "memset");
        for (float *p : {gp.m_atten, gp.v_atten})
            check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * std::max(n, 1), st), "memset");
        for (float *p : {gp.m_resp, gp.v_resp})
            check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * 2 * std::max(n, 1), st), "memset");
        for (float *p : {net_m, net_v})
            check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * P, st), "memset");
    }

    void setup_net_layout()
    {
        width = cfg.width;
        Dc = 2 * (2 * cfg.bands_center + 1);
        Dp = 3 * (2 * cfg.bands_position + 1);
        D = Dc + Dp;
        int64_t at = 0;
        for (int i = 0; i < kTrunkLayers; i++)
        {
            cols[i] = i == 0 ? D : (skip_layer(i) ? width + D : width);
            off_w[i] = at;
            at += int64_t(width) * cols[i];
            off_b[i] = at;
            at += width;
        }
        off_w[kTrunkLayers] = at;
        at += int64_t(5) * width;
        off_b[kTrunkLayers] = at;
        at += 5;
        P = at;
    }

    // params in the reference layer order -> flat device buffer
    void upload_net(const std::vector<std::vector<float>> &lw, const std::vector<std::vector<float>> &lb)
    {
        std::vector<float> flat(static_cast<size_t>(P), 0.f);
        for (int i = 0; i < kTrunkLayers; i++)
        {
            if (lw[i].size() != size_t(width) * cols[i] || lb[i].size() != size_t(width))
                throw std::invalid_argument("deform layer shape does not match width/encoding");
            std::memcpy(&flat[size_t(off_w[i])], lw[i].data(), sizeof(float) * lw[i].size());
            std::memcpy(&flat[size_t(off_b[i])], lb[i].data(), sizeof(float) * lb[i].size());
        }
        const int hr[3] = {2, 2, 1};
        int row = 0;
        for (int k = 0; k < 3; k++)
        {
            if (lw[8 + k].size() != size_t(hr[k]) * width || lb[8 + k].size() != size_t(hr[k]))
                throw std::invalid_argument("deform head shape does not match width");
            std::memcpy(&flat[size_t(off_w[kTrunkLayers] + int64_t(row) * width)], lw[8 + k].data(),
                        sizeof(float) * lw[8 + k].size());
            std::memcpy(&flat[size_t(off_b[kTrunkLayers] + row)], lb[8 + k].data(), sizeof(float) * lb[8 + k].size());
            row += hr[k];
        }
        check_cuda(cudaMemcpy(net_p, flat.data(), sizeof(float) * P, cudaMemcpyHostToDevice), "upload net");
    }

    void download_net(std::vector<std::vector<float>> &lw, std::vector<std::vector<float>> &lb)
    {
        std::vector<float> flat(static_cast<size_t>(P));
        check_cuda(cudaMemcpy(flat.data(), net_p, sizeof(float) * P, cudaMemcpyDeviceToHost), "download net");
        lw.assign(11, {});
        lb.assign(11, {});
        for (int i = 0; i < kTrunkLayers; i++)
        {
            lw[i].assign(flat.begin() + off_w[i], flat.begin() + off_w[i] + int64_t(width) * cols[i]);
            lb[i].assign(flat.begin() + off_b[i], flat.begin() + off_b[i] + width);
        }
        const int hr[3] = {2, 2, 1};
        int row = 0;
        for (int k = 0; k < 3; k++)
        {
            const int64_t w0 = off_w[kTrunkLayers] + int64_t(row) * width, b0 = off_b[kTrunkLayers] + row;
            lw[8 + k].assign(flat.begin() + w0, flat.begin() + w0 + int64_t(hr[k]) * width);
            lb[8 + k].assign(flat.begin() + b0, flat.begin() + b0 + hr[k]);
            row += hr[k];
        }
    }

    void alloc_buffers()
    {
        const size_t nn = size_t(std::max(n, 1));
        gp.center = dalloc<float>(c, 2 * nn);
        gp.chol = dalloc<float>(c, 3 * nn);
        gp.atten = dalloc<float>(c, nn);
        gp.resp = dalloc<float>(c, 2 * nn);
        gp.m_center = dalloc<float>(c, 2 * nn);
        gp.v_center = dalloc<float>(c, 2 * nn);
        gp.m_chol = dalloc<float>(c, 3 * nn);
        gp.v_chol = dalloc<float>(c, 3 * nn);
        gp.m_atten = dalloc<float>(c, nn);
        gp.v_atten = dalloc<float>(c, nn);
        gp.m_resp = dalloc<float>(c, 2 * nn);
        gp.v_resp = dalloc<float>(c, 2 * nn);
        const int widths[7] = {2, 3, 1, 2, 2, 2, 1};
        for (int k = 0; k < 7; k++)
            grads[k] = dalloc<float>(c, nn * widths[k]);
        gp.g_center = grads[0];
        gp.g_chol = grads[1];
        gp.g_atten = grads[2];
        gp.g_resp = grads[3];
        net_p = dalloc<float>(c, size_t(P));
        net_g = dalloc<float>(c, size_t(P));
        net_m = dalloc<float>(c, size_t(P));
        net_v = dalloc<float>(c, size_t(P));
        x0 = dalloc<float>(c, nn * D);
        for (int i = 0; i < kTrunkLayers; i++)
            h[i] = dalloc<float>(c, nn * width);
        dz_a = dalloc<float>(c, nn * width);
        dz_b = dalloc<float>(c, nn * width);
        dr5 = dalloc<float>(c, nn * 5);
        part = dalloc<float>(c, dw_partial_floats(n, width, width + D + 1));
        const size_t per = size_t(2) * H * W;
        d_pred = dalloc<float>(c, per);
        d_lgrad = dalloc<float>(c, per);
        d_target = dalloc<float>(c, per);
        d_state = dalloc<float>(c, nn * 11);
        d_tmp = dalloc<double>(c, loss_tmp_doubles(c, 1));
        d_terms = dalloc<double>(c, 3);
        d_bad = dalloc<int>(c, 1);
        // every (tile, primitive) pair of one position at most: no pair-count sync
        pair_cap = std::max<int64_t>(int64_t(n) * c.g.tiles, 1024);
        ensure_pairs(c, pair_cap, 1, pair_cap);
        d_slots = dalloc<float>(c, size_t(pair_cap) * 8);
        const int64_t cap = std::max<int64_t>(total - iteration, 1);
        it_base = iteration;
        d_sidx = dalloc<int>(c, size_t(cap));
        d_spenc = dalloc<float>(c, size_t(cap) * Dp);
        d_sbc = dalloc<double>(c, size_t(cap) * 6);
        d_log = dalloc<double>(c, size_t(cap) * 3);
        sched = TrainSched{d_sidx, d_spenc, d_sbc, dalloc<int64_t>(c, 1)};
        g_sidx = dalloc<int>(c, 1);
        g_spenc = dalloc<float>(c, size_t(Dp));
        g_sbc = dalloc<double>(c, 6);
        g_it = dalloc<int64_t>(c, 1);
        const char *env = std::getenv("SWR_TRAIN_GRAPHS");
        use_graphs = !(env && env[0] == '0');
        check_cuda(cudaEventCreate(&ev0), "event");
        check_cuda(cudaEventCreate(&ev1), "event");
    }

    void upload_gauss(const HostScene &hs)
    {
        check_cuda(cudaMemcpy(gp.center, hs.center_raw.data(), sizeof(float) * 2 * n, cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(gp.chol, hs.cholesky.data(), sizeof(float) * 3 * n, cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(gp.atten, hs.atten.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(gp.resp, hs.response.data(), sizeof(float) * 2 * n, cudaMemcpyHostToDevice), "H2D");
    }

    // the network's centre-encoding columns of x0 from the current centres, on the
    // host (glibc tanhf + sinf/cosf as in predict_residuals, deform.cpp:157-168);
    // also resets the device scene to host-derived inputs (refresh_scene_host)
    void host_center_inputs()
    {
        check_cuda(cudaStreamSynchronize(c.stream), "sync");
        std::vector<float> cr(size_t(2) * n), ch(size_t(3) * n), at(static_cast<size_t>(n)), rs(size_t(2) * n);
        check_cuda(cudaMemcpy(cr.data(), gp.center, 4 * cr.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(ch.data(), gp.chol, 4 * ch.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(at.data(), gp.atten, 4 * at.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(rs.data(), gp.resp, 4 * rs.size(), cudaMemcpyDeviceToHost), "D2H");
        refresh_scene_host(c, cr.data(), ch.data(), at.data(), rs.data());
        std::vector<float> enc(size_t(n) * Dc);
        for (int p = 0; p < n; p++)
        {
            const float v[2] = {float(kPi / 4) * (std::tanh(cr[2 * size_t(p)]) + 1.0f),
                                float(kPi) * (std::tanh(cr[2 * size_t(p) + 1]) + 1.0f)};
            encode_host(v, 2, cfg.bands_center, enc.data() + size_t(p) * Dc);
        }
        check_cuda(cudaMemcpy2D(x0, sizeof(float) * D, enc.data(), sizeof(float) * Dc, sizeof(float) * Dc, size_t(n),
                                cudaMemcpyHostToDevice),
                   "H2D centre encodings");
    }

    float floor_el() const { return float(kPi / 2.0 / H / 3.0); } // training.cpp:276-277
    float floor_az() const { return float(2.0 * kPi / W / 3.0); }

    // dataset normalization (dataset.cpp:35-44)
    void normalized_position(int idx, float out[3]) const
    {
        for (int a = 0; a < 3; a++)
        {
            const double range = ds_max[a] - ds_min[a];
            out[a] = range > 0.0 ? float((double(positions[3 * size_t(idx) + a]) - ds_min[a]) / range) : 0.5f;
        }
    }

    // ---------------------------------------------------------------- device step
    // Everything an iteration enqueues reads its per-iteration arguments through
    // a TrainSched (device tables + cursor), and every buffer is sized for the
    // worst case at creation (pairs <= n * tiles per position), so one iteration
    // is a fixed launch sequence: captured once per stage and replayed as a CUDA
    // graph, with no host round trip inside the loop.

    void render_and_backward(const TrainSched &sc, bool with_res)
    {
        cudaStream_t st = c.stream;
        launch_gather_target(c, d_spectra, sc, d_target, st);
        launch_setup(c, 1, with_res, st);
        launch_bin_count(c, 1, st);
        // the graph-captured step cannot know the pair count: the sort CTAs loop over
        // chunks, sized for ~4 pairs per primitive (measured ~3.3) instead of the cap
        launch_bin_sort(c, 1, -1, int(std::min<int64_t>(pair_cap, int64_t(4) * c.g.n + 1)), st);
        launch_raster(c, 1, d_pred, false, st);
        launch_hybrid_loss(c, d_pred, d_target, 1, cfg.lambda1, d_terms, d_lgrad, d_tmp, d_bad, st);
        launch_state_out(c, 1, with_res, d_state, st);
        launch_raster_backward(c, 1, d_state, d_lgrad, d_slots, st);
        launch_bwd_merge(c, 1, with_res, d_slots, grads, st);
    }

    void net_forward(const TrainSched &sc)
    {
        cudaStream_t st = c.stream;
        launch_position_encoding(c, x0, D, Dc, sc, Dp, st);
        const float *prev = x0;
        for (int i = 0; i < kTrunkLayers; i++)
        {
            const float *Wl = net_p + off_w[i], *bl = net_p + off_b[i];
            if (i == 0)
                launch_dense_fwd(c, x0, D, D, nullptr, 0, D, Wl, bl, width, h[0], st);
            else if (skip_layer(i))
                launch_dense_fwd(c, prev, width, width, x0, D, width + D, Wl, bl, width, h[i], st);
            else
                launch_dense_fwd(c, prev, width, width, nullptr, 0, width, Wl, bl, width, h[i], st);
            prev = h[i];
        }
        launch_heads_fwd(c, h[kTrunkLayers - 1], width, net_p + off_w[kTrunkLayers], net_p + off_b[kTrunkLayers],
                         c.w.res, int64_t(c.w.cap_b) * c.g.np, st);
    }

    void net_backward()
    {
        cudaStream_t st = c.stream;
        const float *Wh = net_p + off_w[kTrunkLayers];
        launch_heads_bwd(c, grads[4], grads[5], grads[6], Wh, Wh + 2 * width, Wh + 4 * width, h[kTrunkLayers - 1],
                         width, dz_a, dr5, st);
        launch_dense_bwd_weights(c, dr5, 5, h[kTrunkLayers - 1], width, width, nullptr, 0, width, part,
                                 net_g + off_w[kTrunkLayers], net_g + off_b[kTrunkLayers], st);
        float *dz = dz_a, *dz_next = dz_b;
        for (int i = kTrunkLayers - 1; i >= 0; i--)
        {
            float *gW = net_g + off_w[i], *gb = net_g + off_b[i];
            if (i == 0)
                launch_dense_bwd_weights(c, dz, width, x0, D, D, nullptr, 0, D, part, gW, gb, st);
            else if (skip_layer(i))
                launch_dense_bwd_weights(c, dz, width, h[i - 1], width, width, x0, D, width + D, part, gW, gb, st);
            else
                launch_dense_bwd_weights(c, dz, width, h[i - 1], width, width, nullptr, 0, width, part, gW, gb, st);
            if (i > 0)
            {
                launch_dense_bwd_input(c, dz, width, net_p + off_w[i], cols[i], h[i - 1], dz_next, st);
                std::swap(dz, dz_next);
            }
        }
    }

    // one full training iteration (training.cpp:312-376) on the stream
    void enqueue_step(bool coarse)
    {
        cudaStream_t st = c.stream;
        const AdamHp hp_g{cfg.lr_gaussian, 0.9, 0.999, 1e-8}, hp_n{cfg.lr_mlp, 0.9, 0.999, 1e-8};
        if (coarse)
        {
            render_and_backward(sched, false);
            launch_gauss_adam(c, gp, hp_g, sched, true, true, floor_el(), floor_az(), st);
        }
        else
        {
            net_forward(sched);
            render_and_backward(sched, true);
            net_backward();
            launch_adam_flat(c, net_p, net_g, net_m, net_v, P, hp_n, sched, st);
            launch_gauss_adam(c, gp, hp_g, sched, false, true, floor_el(), floor_az(), st);
        }
        launch_log_advance(c, d_terms, d_log, sched, st);
    }

    // replay `count` iterations of one stage: the first eagerly (lazy kernel
    // attributes, and a check), the rest through the stage's captured graph
    void enqueue_iterations(bool coarse, int64_t count)
    {
        cudaStream_t st = c.stream;
        if (count <= 0)
            return;
        const int gi = coarse ? 0 : 1;
        enqueue_step(coarse);
        check_cuda(cudaGetLastError(), "training launch");
        if (count == 1)
            return;
        if (!use_graphs)
        {
            for (int64_t k = 1; k < count; k++)
                enqueue_step(coarse);
            return;
        }
        if (!graph[gi])
        {
            const int64_t l0 = c.launches;
            cudaGraph_t g = nullptr;
            check_cuda(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
            enqueue_step(coarse);
            check_cuda(cudaStreamEndCapture(st, &g), "end capture");
            check_cuda(cudaGraphInstantiate(&graph[gi], g, 0), "graph instantiate");
            cudaGraphDestroy(g);
            graph_launches[gi] = c.launches - l0;
            c.launches = l0;
        }
        for (int64_t k = 1; k < count; k++)
            check_cuda(cudaGraphLaunch(graph[gi], st), "graph launch");
        c.launches += graph_launches[gi] * (count - 1);
    }

    // one forward/backward at the current parameters without an optimizer step:
    // pos01 != null = fine-stage pass (residuals from the network at that
    // normalized position), else coarse (no residuals); target = dataset sample
    void gradients(const float *pos01, int idx, double *terms)
    {
        cudaStream_t st = c.stream;
        check_cuda(cudaMemsetAsync(d_bad, 0, sizeof(int), st), "memset");
        host_center_inputs(); // the reference's exact render / encoding inputs
        std::vector<float> penc(static_cast<size_t>(Dp), 0.f);
        if (pos01)
            encode_host(pos01, 3, cfg.bands_position, penc.data());
        const int64_t zero = 0;
        check_cuda(cudaMemcpy(g_sidx, &idx, sizeof(int), cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(g_spenc, penc.data(), sizeof(float) * Dp, cudaMemcpyHostToDevice), "H2D");
        check_cuda(cudaMemcpy(g_it, &zero, sizeof(int64_t), cudaMemcpyHostToDevice), "H2D");
        const TrainSched gs{g_sidx, g_spenc, g_sbc, g_it};
        if (pos01)
        {
            net_forward(gs);
            render_and_backward(gs, true);
            net_backward();
        }
        else
            render_and_backward(gs, false);
        check_cuda(cudaGetLastError(), "gradient launch");
        check_cuda(cudaMemcpyAsync(terms, d_terms, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "gradients");
    }

    int64_t run(int64_t max_iters, double *log, double *ms)
    {
        cudaStream_t st = c.stream;
        const int64_t todo = std::max<int64_t>(0, std::min(max_iters, total - iteration));
        if (todo == 0)
        {
            if (ms)
                *ms = 0.0;
            return 0;
        }
        // host plan: the reference's Rng stream, stage switches and Adam step
        // counters (training.cpp:298-376) -> device tables
        const int64_t slot0 = iteration - it_base;
        std::vector<int> sidx(static_cast<size_t>(todo));
        std::vector<float> spenc(size_t(todo) * Dp, 0.f);
        std::vector<double> sbc(size_t(todo) * 6, 1.0);
        const double count = double(std::max<size_t>(train_idx.size(), 1));
        bool fine_seen = in_fine;
        int64_t first_fine = todo; // index of the first fine iteration of this run
        for (int64_t k = 0; k < todo; k++)
        {
            const int64_t it = iteration + k;
            const bool coarse = it < cfg.coarse_iters;
            if (!coarse && !fine_seen)
            {
                fine_seen = true; // moments and step counters restart (training.cpp:305-310)
                t_center = t_rest = t_net = 0;
            }
            if (!coarse && first_fine == todo)
                first_fine = k;
            const int idx = train_idx[size_t(rng.index(train_idx.size()))];
            sidx[size_t(k)] = idx;
            double *bc = &sbc[size_t(k) * 6];
            if (coarse)
            {
                t_center++;
                t_rest++;
                bc[0] = 1.0 - std::pow(0.9, double(t_center));
                bc[1] = 1.0 - std::pow(0.999, double(t_center));
            }
            else
            {
                float pos[3];
                normalized_position(idx, pos);
                const int64_t fine_it = it - cfg.coarse_iters;
                if (!(cfg.anneal_scale == 0.0 || fine_it >= cfg.anneal_threshold)) // training.cpp:116-128
                {
                    const double amp = cfg.anneal_scale * (2.0 / std::cbrt(count)) *
                                       (1.0 - double(fine_it) / double(cfg.anneal_threshold));
                    for (int a = 0; a < 3; a++)
                        pos[a] = pos[a] + float(rng.normal() * amp);
                }
                encode_host(pos, 3, cfg.bands_position, &spenc[size_t(k) * Dp]);
                t_net++;
                t_rest++;
                bc[4] = 1.0 - std::pow(0.9, double(t_net));
                bc[5] = 1.0 - std::pow(0.999, double(t_net));
            }
            bc[2] = 1.0 - std::pow(0.9, double(t_rest));
            bc[3] = 1.0 - std::pow(0.999, double(t_rest));
        }
        check_cuda(cudaMemcpy(d_sidx + slot0, sidx.data(), sizeof(int) * todo, cudaMemcpyHostToDevice), "H2D plan");
        check_cuda(cudaMemcpy(d_spenc + slot0 * Dp, spenc.data(), sizeof(float) * spenc.size(), cudaMemcpyHostToDevice),
                   "H2D plan");
        check_cuda(cudaMemcpy(d_sbc + slot0 * 6, sbc.data(), sizeof(double) * sbc.size(), cudaMemcpyHostToDevice),
                   "H2D plan");
        check_cuda(cudaMemcpy(sched.it, &slot0, sizeof(int64_t), cudaMemcpyHostToDevice), "H2D cursor");
        check_cuda(cudaMemsetAsync(d_bad, 0, sizeof(int), st), "memset");

        float f_total = 0.f;
        auto timed = [&](bool coarse, int64_t cnt) {
            check_cuda(cudaEventRecord(ev0, st), "event");
            enqueue_iterations(coarse, cnt);
            check_cuda(cudaEventRecord(ev1, st), "event");
            check_cuda(cudaStreamSynchronize(st), "training");
            float f = 0.f;
            check_cuda(cudaEventElapsedTime(&f, ev0, ev1), "event time");
            f_total += f;
        };
        if (first_fine > 0)
            timed(true, first_fine);
        if (first_fine < todo)
        {
            if (!in_fine)
            {
                reset_opt();
                in_fine = true;
            }
            if (!cenc_ready)
            {
                // centres are frozen in the fine stage: their encodings (and the
                // scene's centre-derived inputs) are computed once, on the host
                host_center_inputs();
                cenc_ready = true;
            }
            timed(false, todo - first_fine);
        }
        if (ms)
            *ms = f_total;
        std::vector<double> host(size_t(3) * todo);
        check_cuda(cudaMemcpy(host.data(), d_log + 3 * slot0, sizeof(double) * host.size(), cudaMemcpyDeviceToHost),
                   "D2H log");
        if (log)
            std::memcpy(log, host.data(), sizeof(double) * host.size());
        iteration += todo;
        int bad = 0;
        check_cuda(cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost), "D2H flag");
        for (int64_t k = 0; k < todo; k++)
            if (!std::isfinite(host[3 * k]))
                bad = 1;
        if (bad)
            throw std::runtime_error("hybrid loss is not finite"); // training.cpp:89-90
        return todo;
    }

    void save(const std::string &path)
    {
        std::vector<float> cr(size_t(2) * n), ch(size_t(3) * n), at(static_cast<size_t>(n)), rs(size_t(2) * n);
        check_cuda(cudaMemcpy(cr.data(), gp.center, sizeof(float) * cr.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(ch.data(), gp.chol, sizeof(float) * ch.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(at.data(), gp.atten, sizeof(float) * at.size(), cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemcpy(rs.data(), gp.resp, sizeof(float) * rs.size(), cudaMemcpyDeviceToHost), "D2H");
        std::vector<std::vector<float>> lw, lb;
        download_net(lw, lb);
        std::string out;
        auto put = [&](const void *p, size_t k) { out.append(static_cast<const char *>(p), k); };
        auto u32 = [&](uint32_t v) { put(&v, 4); };
        auto u64 = [&](uint64_t v) { put(&v, 8); };
        // checkpoint.cpp:50-93: header, section table, WRF2, WRFD, JSON trailer
        put("WRFC", 4);
        u32(1);
        u32(3);
        u32(0);
        const size_t table = out.size();
        for (int i = 0; i < 6; i++)
            u64(0);
        uint64_t off[3], size[3];
        off[0] = out.size();
        put("WRF2", 4); // splat.cpp:711-721
        u32(1);
        u32(uint32_t(n));
        u32(0);
        put(cr.data(), 4 * cr.size());
        put(ch.data(), 4 * ch.size());
        put(at.data(), 4 * at.size());
        put(rs.data(), 4 * rs.size());
        size[0] = out.size() - off[0];
        off[1] = out.size();
        put("WRFD", 4); // deform.cpp:328-352
        u32(1);
        u32(11);
        u32(uint32_t(width));
        u32(uint32_t(cfg.bands_center));
        u32(uint32_t(cfg.bands_position));
        for (int i = 0; i < 11; i++)
        {
            const uint32_t rows = uint32_t(lb[i].size());
            u32(rows);
            u32(uint32_t(lw[i].size() / std::max<size_t>(rows, 1)));
        }
        for (int i = 0; i < 11; i++)
        {
            put(lw[i].data(), 4 * lw[i].size());
            put(lb[i].data(), 4 * lb[i].size());
        }
        size[1] = out.size() - off[1];
        off[2] = out.size();
        nlohmann::json j;
        j["config"] = config_json(cfg);
        j["iteration"] = iteration;
        char hex[17];
        std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(manifest_hash));
        j["manifest_hash"] = std::string(hex);
        j["grid"] = {{"n_elevation", H}, {"n_azimuth", W}};
        j["bbox_min"] = std::vector<double>(bbox_min, bbox_min + 3);
        j["bbox_max"] = std::vector<double>(bbox_max, bbox_max + 3);
        const std::string trailer = j.dump();
        put(trailer.data(), trailer.size());
        size[2] = out.size() - off[2];
        for (int i = 0; i < 3; i++)
        {
            std::memcpy(&out[table + 16 * i], &off[i], 8);
            std::memcpy(&out[table + 16 * i + 8], &size[i], 8);
        }
        std::ofstream os(path, std::ios::binary);
        if (!os)
            throw std::runtime_error("cannot open " + path + " for writing");
        os.write(out.data(), std::streamsize(out.size()));
        if (!os)
            throw std::runtime_error("write failed: " + path);
    }
};

} // namespace swr

using namespace swr;

struct swr_trainer
{
    Trainer t;
};

extern "C" {

void swr_train_config_default(swr_train_config *c)
{
    c->primitives = 10000;
    c->bands_center = 10;
    c->bands_position = 6;
    c->width = 156;
    c->cutoff_radius = 3.0f;
    c->tile = 16;
    c->lr_gaussian = 1e-2;
    c->lr_mlp = 8e-3;
    c->lambda1 = 0.7;
    c->coarse_iters = 10000;
    c->fine_iters = 100000;
    c->anneal_scale = 1.0;
    c->anneal_threshold = 10000;
    c->seed = 1234;
}

int swr_trainer_create(const swr_train_config *cfg, swr_dataset *ds, const char *resume_wrfc, int device,
                       swr_trainer **out)
{
    return swr_guarded([&] {
        if (!cfg || !ds || !out)
            throw std::invalid_argument("null argument");
        const DatasetFile &d = ds->d;
        // training.cpp:201-208
        if (d.count < 1)
            throw std::invalid_argument("dataset has no samples");
        if (d.train.empty())
            throw std::invalid_argument("dataset has no training split");
        if (cfg->coarse_iters < 0 || cfg->fine_iters < 0)
            throw std::invalid_argument("iteration counts must be >= 0");
        if (!(cfg->lambda1 >= 0.0 && cfg->lambda1 <= 1.0))
            throw std::invalid_argument("lambda1 must lie in [0, 1]");
        auto holder = std::make_unique<swr_trainer>();
        Trainer &t = holder->t;
        t.cfg = *cfg;
        t.rng = RefRng(cfg->seed);
        t.H = d.H;
        t.W = d.W;
        t.samples = d.count;
        t.train_idx = d.train;
        std::memcpy(t.bbox_min, d.bbox_min, sizeof(t.bbox_min));
        std::memcpy(t.bbox_max, d.bbox_max, sizeof(t.bbox_max));
        std::memcpy(t.ds_min, d.bbox_min, sizeof(t.ds_min));
        std::memcpy(t.ds_max, d.bbox_max, sizeof(t.ds_max));
        t.manifest_hash = d.hash;

        HostScene hs;
        hs.H = d.H;
        hs.W = d.W;
        std::vector<std::vector<float>> lw, lb;
        if (resume_wrfc)
        {
            HostScene ck = parse_wrfc(resume_wrfc);
            if (!same_config(config_from_json(ck.config_json), *cfg))
                throw std::invalid_argument("resume checkpoint was trained with a different config");
            if (ck.manifest_hash != d.hash)
                throw std::runtime_error("resume checkpoint was trained on a different dataset");
            if (ck.H != d.H || ck.W != d.W)
                throw std::invalid_argument("resume checkpoint grid differs from the dataset");
            hs.n = ck.n;
            hs.center_raw = ck.center_raw;
            hs.cholesky = ck.cholesky;
            hs.atten = ck.atten;
            hs.response = ck.response;
            lw = ck.lw;
            lb = ck.lb;
            t.iteration = ck.iteration;
            std::memcpy(t.bbox_min, ck.bmin, sizeof(t.bbox_min)); // ck = *resume keeps its bbox
            std::memcpy(t.bbox_max, ck.bmax, sizeof(t.bbox_max));
        }
        else
        {
            // splat::init_random (splat.cpp:681-709) then DeformNet::init (deform.cpp:73-102)
            const int n = cfg->primitives;
            if (n < 1)
                throw std::invalid_argument("primitive count must be >= 1");
            hs.n = n;
            hs.center_raw.resize(size_t(2) * n);
            hs.response.resize(size_t(2) * n);
            hs.cholesky.resize(size_t(3) * n);
            hs.atten.assign(size_t(n), 0.f);
            for (int p = 0; p < n; p++)
            {
                hs.center_raw[2 * size_t(p)] = float(t.rng.uniform(-2.0, 2.0));
                hs.center_raw[2 * size_t(p) + 1] = float(t.rng.uniform(-2.0, 2.0));
            }
            for (int p = 0; p < n; p++)
            {
                hs.response[2 * size_t(p)] = float(0.0 + 0.01 * t.rng.normal());
                hs.response[2 * size_t(p) + 1] = float(0.0 + 0.01 * t.rng.normal());
            }
            const float sd_el = float(2.0 * ((kPi / 2.0) / d.H)), sd_az = float(2.0 * ((2.0 * kPi) / d.W));
            for (int p = 0; p < n; p++)
            {
                hs.cholesky[3 * size_t(p)] = sd_el;
                hs.cholesky[3 * size_t(p) + 1] = 0.0f;
                hs.cholesky[3 * size_t(p) + 2] = sd_az;
            }
            if (cfg->width < 1)
                throw std::invalid_argument("deform-net width must be >= 1");
            const int D = 2 * (2 * cfg->bands_center + 1) + 3 * (2 * cfg->bands_position + 1);
            lw.assign(11, {});
            lb.assign(11, {});
            for (int i = 0; i < kTrunkLayers; i++)
            {
                const int cols = i == 0 ? D : (skip_layer(i) ? cfg->width + D : cfg->width);
                lw[i].resize(size_t(cfg->width) * cols);
                lb[i].assign(size_t(cfg->width), 0.f);
                const double bound = 1.0 / std::sqrt(double(cols));
                for (auto &v : lw[i])
                    v = float(t.rng.uniform(-bound, bound));
            }
            const int hr[3] = {2, 2, 1};
            for (int k = 0; k < 3; k++)
            {
                lw[8 + k].assign(size_t(hr[k]) * cfg->width, 0.f);
                lb[8 + k].assign(size_t(hr[k]), 0.f);
            }
        }
        if (cfg->width > 160)
            throw std::invalid_argument("training supports deform-net widths up to 160");
        hs.cutoff = cfg->cutoff_radius;
        hs.tile = cfg->tile;
        std::memcpy(hs.bmin, t.bbox_min, sizeof(hs.bmin));
        std::memcpy(hs.bmax, t.bbox_max, sizeof(hs.bmax));
        hs.manifest_hash = t.manifest_hash;
        build_scene(t.c, hs, device); // render scene without the inference network
        t.n = hs.n;
        t.total = cfg->coarse_iters + cfg->fine_iters;
        t.in_fine = t.iteration >= cfg->coarse_iters;
        t.setup_net_layout();
        ensure_work(t.c, 1);
        t.c.w.want_perm = true; // the backward walks the CSR permutation of the bin sort
        t.alloc_buffers();
        t.upload_gauss(hs);
        t.upload_net(lw, lb);
        // every sample's spectrum on the device, sample order (dataset.cpp:205-258)
        const size_t per = size_t(2) * d.H * d.W;
        t.positions.resize(size_t(3) * d.count);
        t.d_spectra = dalloc<float>(t.c, per * size_t(d.count));
        const int64_t blk = 256;
        std::vector<float> buf(per * blk);
        std::vector<int32_t> ids(blk);
        for (int64_t b0 = 0; b0 < d.count; b0 += blk)
        {
            const int64_t m = std::min(blk, d.count - b0);
            for (int64_t k = 0; k < m; k++)
                ids[size_t(k)] = int32_t(b0 + k);
            d.read(ids.data(), m, t.positions.data() + 3 * b0, buf.data());
            check_cuda(cudaMemcpy(t.d_spectra + per * b0, buf.data(), sizeof(float) * per * m, cudaMemcpyHostToDevice),
                       "H2D spectra");
        }
        t.reset_opt();
        check_cuda(cudaStreamSynchronize(t.c.stream), "trainer init");
        *out = holder.release();
    });
}

void swr_trainer_destroy(swr_trainer *tr) { delete tr; }

int swr_trainer_run(swr_trainer *tr, int64_t max_iters, double *log, int64_t *done, double *device_ms)
{
    return swr_guarded([&] {
        if (max_iters < 0)
            throw std::invalid_argument("negative iteration count");
        check_cuda(cudaSetDevice(tr->t.c.device), "cudaSetDevice");
        const int64_t k = tr->t.run(max_iters, log, device_ms);
        if (done)
            *done = k;
    });
}

int64_t swr_trainer_iteration(swr_trainer *tr) { return tr->t.iteration; }

int swr_trainer_params(swr_trainer *tr, float *center_raw, float *cholesky, float *atten_logit, float *response,
                       float *const layer_w[11], float *const layer_b[11])
{
    return swr_guarded([&] {
        Trainer &t = tr->t;
        check_cuda(cudaSetDevice(t.c.device), "cudaSetDevice");
        const size_t n = size_t(t.n);
        if (center_raw)
            check_cuda(cudaMemcpy(center_raw, t.gp.center, sizeof(float) * 2 * n, cudaMemcpyDeviceToHost), "D2H");
        if (cholesky)
            check_cuda(cudaMemcpy(cholesky, t.gp.chol, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost), "D2H");
        if (atten_logit)
            check_cuda(cudaMemcpy(atten_logit, t.gp.atten, sizeof(float) * n, cudaMemcpyDeviceToHost), "D2H");
        if (response)
            check_cuda(cudaMemcpy(response, t.gp.resp, sizeof(float) * 2 * n, cudaMemcpyDeviceToHost), "D2H");
        if (layer_w || layer_b)
        {
            std::vector<std::vector<float>> lw, lb;
            t.download_net(lw, lb);
            for (int i = 0; i < 11; i++)
            {
                if (layer_w && layer_w[i])
                    std::memcpy(layer_w[i], lw[i].data(), sizeof(float) * lw[i].size());
                if (layer_b && layer_b[i])
                    std::memcpy(layer_b[i], lb[i].data(), sizeof(float) * lb[i].size());
            }
        }
    });
}

int swr_trainer_gradients(swr_trainer *tr, const float *pos01, int32_t sample, double *terms,
                          float *const render_grads[7], float *const layer_gw[11], float *const layer_gb[11])
{
    return swr_guarded([&] {
        Trainer &t = tr->t;
        if (sample < 0 || sample >= t.samples)
            throw std::invalid_argument("sample index out of range");
        check_cuda(cudaSetDevice(t.c.device), "cudaSetDevice");
        double tm[3];
        t.gradients(pos01, sample, tm);
        if (terms)
            std::memcpy(terms, tm, sizeof(tm));
        const int widths[7] = {2, 3, 1, 2, 2, 2, 1};
        if (render_grads)
            for (int k = 0; k < 7; k++)
                if (render_grads[k])
                    check_cuda(cudaMemcpy(render_grads[k], t.grads[k], sizeof(float) * size_t(t.n) * widths[k],
                                          cudaMemcpyDeviceToHost),
                               "D2H grads");
        if (pos01 && (layer_gw || layer_gb))
        {
            std::vector<float> flat(static_cast<size_t>(t.P));
            check_cuda(cudaMemcpy(flat.data(), t.net_g, sizeof(float) * t.P, cudaMemcpyDeviceToHost), "D2H");
            const int hr[3] = {2, 2, 1};
            for (int i = 0; i < 11; i++)
            {
                int64_t w0, b0, wn, bn;
                if (i < kTrunkLayers)
                {
                    w0 = t.off_w[i];
                    b0 = t.off_b[i];
                    wn = int64_t(t.width) * t.cols[i];
                    bn = t.width;
                }
                else
                {
                    const int row = i == 8 ? 0 : (i == 9 ? 2 : 4);
                    w0 = t.off_w[kTrunkLayers] + int64_t(row) * t.width;
                    b0 = t.off_b[kTrunkLayers] + row;
                    wn = int64_t(hr[i - 8]) * t.width;
                    bn = hr[i - 8];
                }
                if (layer_gw && layer_gw[i])
                    std::memcpy(layer_gw[i], flat.data() + w0, sizeof(float) * wn);
                if (layer_gb && layer_gb[i])
                    std::memcpy(layer_gb[i], flat.data() + b0, sizeof(float) * bn);
            }
        }
    });
}

int swr_trainer_save(swr_trainer *tr, const char *path)
{
    return swr_guarded([&] {
        if (!path)
            throw std::invalid_argument("null path");
        check_cuda(cudaSetDevice(tr->t.c.device), "cudaSetDevice");
        tr->t.save(path);
    });
}

} // extern "C"
