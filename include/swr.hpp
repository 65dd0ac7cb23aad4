// swr.hpp — C++ host API over the C ABI (swr.h), mirroring the reference's
// render-path API so that callers switch by namespace (wrfsplat:: ->
// wrfsplat::b200::). Two layers:
//
// (1) The reference's own signatures and value types:
//   splat::GaussianSetT / ResidualsT / RasterParamsT / RasterWorkspaceT   splat.hpp:43-141
//   splat::rasterize(set, res, params, out, ws), rasterize(set, res, params)  splat.hpp:152-155
//   deform::EncodingSpec / DeformNetT / DeformWorkspaceT                  deform.hpp:34-105
//   deform::predict_residuals(net, set, pos01, ws, out)                   deform.hpp:106-109
//   tasks::pooled_magnitude(spectrum), tasks::aoa_extract(spectrum)       tasks.hpp:41, 79
//   train::Checkpoint {set, net, config, iteration, manifest_hash, bbox}  training.hpp:114-124
//   train::load_checkpoint / normalize_position / render_at              training.hpp:133-154
// Reference-typed calls run on a device context cached per thread and keyed by
// the content of the set (and net / raster params); a Checkpoint registers its
// own context, so rasterize(ck.set, ...) and predict_residuals(ck.net, ck.set,
// ...) reuse the device-resident scene. The workspaces are filled like the
// reference's (state, ranges, tile bins) or, for the deform net, left to the
// device.
//
// (2) Batched and context-explicit calls: render_batch, rasterize(ck, ...),
// predict_residuals(ck, ...), aoa_extract(ck, ...), metrics, evaluate, the
// trainer and the beam scanner.
//
// Error behaviour follows the reference: size / grid problems throw
// std::invalid_argument, I/O / format / device problems std::runtime_error.
// Header-only; link with libswr.so.
#pragma once

#include "swr.h"

#include <complex>
#include <cstdint>
#include <cstddef>
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace wrfsplat::b200
{

namespace detail
{
inline void check(int rc)
{
    if (rc == SWR_OK)
        return;
    const std::string msg = swr_last_error();
    if (rc == SWR_EINVAL)
        throw std::invalid_argument(msg);
    if (rc == SWR_EDOMAIN)
        throw std::domain_error(msg);
    throw std::runtime_error(msg);
}
inline std::shared_ptr<swr_ctx> own(swr_ctx *c) { return std::shared_ptr<swr_ctx>(c, &swr_scene_destroy); }
} // namespace detail

// spectrum.hpp:30-60: grid + interleaved [re, im] cells, elevation the slow axis
struct AngularGrid
{
    int n_elevation = 0, n_azimuth = 0;
    int cells() const { return n_elevation * n_azimuth; }
    double elevation_cell() const { return (3.141592653589793238462643383279502884 / 2.0) / n_elevation; }
    double azimuth_cell() const { return (2.0 * 3.141592653589793238462643383279502884) / n_azimuth; }
    double elevation_center(int i) const { return (i + 0.5) * elevation_cell(); }
    double azimuth_center(int j) const { return (j + 0.5) * azimuth_cell(); }
    bool operator==(const AngularGrid &o) const { return n_elevation == o.n_elevation && n_azimuth == o.n_azimuth; }
};

template <class T>
struct SpectrumT
{
    AngularGrid grid;
    std::vector<T> data; // 2 * cells, [re, im] per cell

    SpectrumT() = default;
    explicit SpectrumT(AngularGrid g) : grid(g), data(std::size_t(2) * g.cells(), T(0)) {}
    T &re(int i, int j) { return data[2 * (std::size_t(i) * grid.n_azimuth + j)]; }
    T &im(int i, int j) { return data[2 * (std::size_t(i) * grid.n_azimuth + j) + 1]; }
    const T &re(int i, int j) const { return data[2 * (std::size_t(i) * grid.n_azimuth + j)]; }
    const T &im(int i, int j) const { return data[2 * (std::size_t(i) * grid.n_azimuth + j) + 1]; }
};
using Spectrum = SpectrumT<float>;

namespace splat
{
// splat.hpp:43-56 (float only: the device path computes in FP32)
template <class T>
struct GaussianSetT
{
    static_assert(std::is_same_v<T, float>, "the B200 renderer takes float sets");
    AngularGrid grid;
    int n = 0;
    std::vector<T> center_raw; // n x 2, pre-tanh (elevation, azimuth)
    std::vector<T> cholesky;   // n x 3, (l1, l2, l3)
    std::vector<T> atten_logit;
    std::vector<T> response;   // n x 2
    void resize(int count)
    {
        n = count;
        center_raw.assign(std::size_t(2) * count, T(0));
        cholesky.assign(std::size_t(3) * count, T(0));
        atten_logit.assign(std::size_t(count), T(0));
        response.assign(std::size_t(2) * count, T(0));
    }
};
using GaussianSet = GaussianSetT<float>;

// splat.hpp:61-72
template <class T>
struct ResidualsT
{
    int n = 0;
    std::vector<T> d_center, d_response, d_atten; // n x 2, n x 2, n
    void resize(int count)
    {
        n = count;
        d_center.assign(std::size_t(2) * count, T(0));
        d_response.assign(std::size_t(2) * count, T(0));
        d_atten.assign(std::size_t(count), T(0));
    }
};
using Residuals = ResidualsT<float>;

// splat.hpp:107-116
template <class T>
struct RasterParamsT
{
    T cutoff_radius = T(3);
    int tile = 16;
    bool operator==(const RasterParamsT &o) const { return cutoff_radius == o.cutoff_radius && tile == o.tile; }
};
using RasterParams = RasterParamsT<float>;

// splat.hpp:129-141 (filled like the reference's: state, ranges, tile bins, centres)
template <class T>
struct RasterWorkspaceT
{
    std::vector<T> state;
    std::vector<int> row_range, col_range, tile_count, tile_offset, tile_prims;
    std::vector<T> grad_slots, el_center, az_center, plane;
};
using RasterWorkspace = RasterWorkspaceT<float>;
} // namespace splat

namespace deform
{
// deform.hpp:34-44
struct EncodingSpec
{
    int bands_center = 10, bands_position = 6;
    int center_dim() const { return 2 * (2 * bands_center + 1); }
    int position_dim() const { return 3 * (2 * bands_position + 1); }
    int input_dim() const { return center_dim() + position_dim(); }
    bool operator==(const EncodingSpec &o) const
    {
        return bands_center == o.bands_center && bands_position == o.bands_position;
    }
};

// deform.hpp:57-83: 8 trunk layers + heads, row-major [rows x cols]
template <class T>
struct DeformNetT
{
    struct Layer
    {
        int rows = 0, cols = 0;
        std::vector<T> w, b;
        void resize(int r, int c)
        {
            rows = r;
            cols = c;
            w.assign(std::size_t(r) * c, T(0));
            b.assign(std::size_t(r), T(0));
        }
    };
    EncodingSpec enc;
    int width = 156;
    std::vector<Layer> trunk; // 8
    Layer head_center, head_response, head_atten;
    std::size_t parameter_count() const
    {
        std::size_t k = 0;
        for (const auto &l : trunk)
            k += l.w.size() + l.b.size();
        for (const Layer *l : {&head_center, &head_response, &head_atten})
            k += l->w.size() + l->b.size();
        return k;
    }
};
using DeformNet = DeformNetT<float>;

// deform.hpp:94-103 (the forward state lives on the device; kept for signature parity)
template <class T>
struct DeformWorkspaceT
{
    int n = 0;
    std::vector<T> input;
    std::vector<std::vector<T>> h, zcat;
    std::vector<T> dh, dcat;
};
using DeformWorkspace = DeformWorkspaceT<float>;
} // namespace deform

namespace train
{
// training.hpp:96-112
struct TrainConfig
{
    int primitives = 10000;
    deform::EncodingSpec enc;
    int width = 156;
    splat::RasterParams raster;
    double lr_gaussian = 1e-2, lr_mlp = 8e-3, lambda1 = 0.7;
    std::int64_t coarse_iters = 10000, fine_iters = 100000;
    double anneal_scale = 1.0;
    std::int64_t anneal_threshold = 10000;
    std::uint64_t seed = 1234;
};
} // namespace train

namespace detail
{
inline std::uint64_t fnv(std::uint64_t h, const void *p, std::size_t n)
{
    const auto *b = static_cast<const unsigned char *>(p);
    for (std::size_t i = 0; i < n; i++)
        h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
template <class V>
std::uint64_t fnv_vec(std::uint64_t h, const V &v)
{
    const std::uint64_t sz = v.size();
    h = fnv(h, &sz, sizeof(sz));
    return v.empty() ? h : fnv(h, v.data(), v.size() * sizeof(v[0]));
}
inline std::uint64_t set_key(const splat::GaussianSet &s)
{
    std::uint64_t h = 1469598103934665603ull;
    h = fnv(h, &s.grid, sizeof(s.grid));
    h = fnv(h, &s.n, sizeof(s.n));
    for (const auto *v : {&s.center_raw, &s.cholesky, &s.atten_logit, &s.response})
        h = fnv_vec(h, *v);
    return h;
}
inline std::uint64_t raster_key(std::uint64_t set, const splat::RasterParams &p)
{
    std::uint64_t h = fnv(set ^ 0x52u, &p.cutoff_radius, sizeof(p.cutoff_radius));
    return fnv(h, &p.tile, sizeof(p.tile));
}
inline std::uint64_t net_key(std::uint64_t set, const deform::DeformNet &n)
{
    std::uint64_t h = fnv(set ^ 0x4eu, &n.enc, sizeof(n.enc));
    h = fnv(h, &n.width, sizeof(n.width));
    for (const auto &l : n.trunk)
        h = fnv_vec(fnv_vec(h, l.w), l.b);
    for (const auto *l : {&n.head_center, &n.head_response, &n.head_atten})
        h = fnv_vec(fnv_vec(h, l->w), l->b);
    return h;
}
// A few device contexts per thread, most recently used first
class ContextCache
{
  public:
    std::shared_ptr<swr_ctx> find(std::uint64_t key)
    {
        for (std::size_t i = 0; i < items_.size(); i++)
            if (items_[i].first == key)
            {
                auto it = items_[i];
                items_.erase(items_.begin() + std::ptrdiff_t(i));
                items_.insert(items_.begin(), it);
                return it.second;
            }
        return nullptr;
    }
    void put(std::uint64_t key, std::shared_ptr<swr_ctx> c)
    {
        for (std::size_t i = 0; i < items_.size(); i++)
            if (items_[i].first == key)
            {
                items_.erase(items_.begin() + std::ptrdiff_t(i));
                break;
            }
        items_.insert(items_.begin(), {key, std::move(c)});
        if (items_.size() > 6)
            items_.pop_back();
    }

  private:
    std::vector<std::pair<std::uint64_t, std::shared_ptr<swr_ctx>>> items_;
};
inline ContextCache &cache()
{
    thread_local ContextCache c;
    return c;
}
inline void check_set(const splat::GaussianSet &s)
{
    if (s.n < 0 || s.center_raw.size() != std::size_t(2) * s.n || s.cholesky.size() != std::size_t(3) * s.n ||
        s.atten_logit.size() != std::size_t(s.n) || s.response.size() != std::size_t(2) * s.n)
        throw std::invalid_argument("gaussian set arrays do not match n");
}
inline void check_res(const splat::GaussianSet &s, const splat::Residuals *r)
{
    if (r && (r->n != s.n || r->d_center.size() != std::size_t(2) * s.n ||
              r->d_response.size() != std::size_t(2) * s.n || r->d_atten.size() != std::size_t(s.n)))
        throw std::invalid_argument("residual count does not match the primitive count");
}
inline std::shared_ptr<swr_ctx> make_ctx(const splat::GaussianSet &s, const deform::DeformNet *net,
                                         const splat::RasterParams &p)
{
    const float *lw[11] = {}, *lb[11] = {};
    int width = 0, bc = 10, bp = 6;
    if (net)
    {
        if (net->trunk.size() != 8)
            throw std::invalid_argument("deform net must have 8 trunk layers");
        for (int i = 0; i < 8; i++)
        {
            lw[i] = net->trunk[std::size_t(i)].w.data();
            lb[i] = net->trunk[std::size_t(i)].b.data();
        }
        lw[8] = net->head_center.w.data();
        lb[8] = net->head_center.b.data();
        lw[9] = net->head_response.w.data();
        lb[9] = net->head_response.b.data();
        lw[10] = net->head_atten.w.data();
        lb[10] = net->head_atten.b.data();
        width = net->width;
        bc = net->enc.bands_center;
        bp = net->enc.bands_position;
    }
    swr_ctx *c = nullptr;
    check(swr_scene_create(s.grid.n_elevation, s.grid.n_azimuth, s.n, s.center_raw.data(), s.cholesky.data(),
                           s.atten_logit.data(), s.response.data(), width, bc, bp, net ? lw : nullptr,
                           net ? lb : nullptr, p.cutoff_radius, p.tile, nullptr, nullptr, -1, &c));
    return own(c);
}
inline std::shared_ptr<swr_ctx> grid_ctx(const AngularGrid &g)
{
    std::uint64_t h = fnv(0x47u, &g, sizeof(g));
    if (auto c = cache().find(h))
        return c;
    swr_ctx *c = nullptr;
    const float none = 0.0f;
    check(swr_scene_create(g.n_elevation, g.n_azimuth, 0, &none, &none, &none, &none, 0, 10, 6, nullptr, nullptr,
                           3.0f, 16, nullptr, nullptr, -1, &c));
    auto p = own(c);
    cache().put(h, p);
    return p;
}
} // namespace detail

namespace train
{
// training.hpp:114-124: the reference's value members (host copies of the scene
// as loaded) plus the device context that renders it
struct Checkpoint
{
    splat::GaussianSet set;
    deform::DeformNet net;
    TrainConfig config;
    std::int64_t iteration = 0;
    std::uint64_t manifest_hash = 0;
    std::array<double, 3> bbox_min{}, bbox_max{};

    Checkpoint() = default;
    explicit Checkpoint(swr_ctx *ctx) : ctx_(detail::own(ctx))
    {
        detail::check(swr_scene_get_info(ctx, &info_));
        set.grid = {info_.n_elevation, info_.n_azimuth};
        set.resize(info_.n);
        detail::check(swr_scene_get_arrays(ctx, set.center_raw.data(), set.cholesky.data(), set.atten_logit.data(),
                                           set.response.data()));
        config.primitives = info_.n;
        config.raster = {info_.cutoff_radius, info_.tile};
        config.enc = {info_.bands_center, info_.bands_position};
        config.width = info_.width;
        std::uint64_t mh = 0;
        detail::check(swr_scene_get_meta(ctx, &iteration, &mh));
        manifest_hash = mh;
        for (int a = 0; a < 3; a++)
        {
            bbox_min[std::size_t(a)] = info_.bbox_min[a];
            bbox_max[std::size_t(a)] = info_.bbox_max[a];
        }
        const std::uint64_t sk = detail::set_key(set);
        detail::cache().put(detail::raster_key(sk, config.raster), ctx_);
        if (info_.width > 0)
        {
            net.enc = config.enc;
            net.width = info_.width;
            net.trunk.resize(8);
            auto fill = [&](int i, deform::DeformNet::Layer &l) {
                int r = 0, c = 0;
                detail::check(swr_scene_get_layer(ctx, i, &r, &c, nullptr, nullptr));
                l.resize(r, c);
                detail::check(swr_scene_get_layer(ctx, i, &r, &c, l.w.data(), l.b.data()));
            };
            for (int i = 0; i < 8; i++)
                fill(i, net.trunk[std::size_t(i)]);
            fill(8, net.head_center);
            fill(9, net.head_response);
            fill(10, net.head_atten);
            detail::cache().put(detail::net_key(sk, net), ctx_);
        }
    }
    swr_ctx *handle() const { return ctx_.get(); }
    const swr_scene_info &info() const { return info_; }
    AngularGrid grid() const { return {info_.n_elevation, info_.n_azimuth}; }
    void set_option(const char *key, double value) { detail::check(swr_set_option(ctx_.get(), key, value)); }

  private:
    std::shared_ptr<swr_ctx> ctx_;
    swr_scene_info info_{};
};

inline Checkpoint load_checkpoint(const std::string &path, int device = 0)
{
    swr_ctx *ctx = nullptr;
    detail::check(swr_scene_create_wrfc(path.c_str(), device, &ctx));
    return Checkpoint(ctx);
}

inline std::array<float, 3> normalize_position(const Checkpoint &ck, const std::array<float, 3> &pos)
{
    std::array<float, 3> out{};
    detail::check(swr_normalize_positions(ck.handle(), pos.data(), 1, out.data()));
    return out;
}

// Batched render_at: positions in metres -> spectra (one per position)
inline std::vector<Spectrum> render_batch(const Checkpoint &ck, const std::vector<std::array<float, 3>> &positions)
{
    const auto g = ck.grid();
    const size_t per = size_t(2) * g.cells();
    std::vector<float> flat(per * positions.size());
    if (!positions.empty())
        detail::check(swr_render(ck.handle(), positions.front().data(), int64_t(positions.size()), SWR_OUT_SPECTRA,
                                 flat.data(), nullptr, nullptr, nullptr, nullptr));
    std::vector<Spectrum> out(positions.size());
    for (size_t b = 0; b < positions.size(); b++)
    {
        out[b].grid = g;
        out[b].data.assign(flat.begin() + per * b, flat.begin() + per * (b + 1));
    }
    return out;
}

// training.hpp:154
inline Spectrum render_at(const Checkpoint &ck, const std::array<float, 3> &position)
{
    return render_batch(ck, {position}).front();
}

// Multi-GPU: the same checkpoint on several devices (devices[0] is the root); a batch
// of positions is split contiguously over them and every spectrum comes back in
// order (csrc/group.cpp; no reference counterpart: the reference renders on one CPU)
class DeviceGroup
{
  public:
    DeviceGroup(const std::string &path, const std::vector<int> &devices)
    {
        swr_group *g = nullptr;
        detail::check(swr_group_create_wrfc(path.c_str(), devices.data(), int(devices.size()), &g));
        g_.reset(g);
        swr_ctx *c = nullptr;
        detail::check(swr_group_context(g, 0, &c));
        swr_scene_info info{};
        detail::check(swr_scene_get_info(c, &info));
        grid_ = AngularGrid{info.n_elevation, info.n_azimuth};
    }
    std::vector<Spectrum> render_batch(const std::vector<std::array<float, 3>> &positions) const
    {
        const size_t per = size_t(2) * grid_.cells();
        std::vector<float> flat(per * positions.size());
        if (!positions.empty())
            detail::check(swr_group_render(g_.get(), positions.front().data(), int64_t(positions.size()),
                                           SWR_OUT_SPECTRA, flat.data(), nullptr, nullptr, nullptr, nullptr));
        std::vector<Spectrum> out(positions.size());
        for (size_t b = 0; b < positions.size(); b++)
        {
            out[b].grid = grid_;
            out[b].data.assign(flat.begin() + per * b, flat.begin() + per * (b + 1));
        }
        return out;
    }
    swr_group *handle() const { return g_.get(); }

  private:
    std::unique_ptr<swr_group, void (*)(swr_group *)> g_{nullptr, &swr_group_destroy};
    AngularGrid grid_;
};
} // namespace train

namespace splat
{
// splat.hpp:152-155: rasterize(set, residuals-or-null, params, out, ws) (T = float;
// callers write rasterize<float>(...) as the reference's do)
template <class T>
void rasterize(const GaussianSetT<T> &set, const ResidualsT<T> *residuals, const RasterParamsT<T> &params,
               SpectrumT<T> &out, RasterWorkspaceT<T> &ws)
{
    detail::check_set(set);
    detail::check_res(set, residuals);
    const std::uint64_t key = detail::raster_key(detail::set_key(set), params);
    auto ctx = detail::cache().find(key);
    if (!ctx)
    {
        ctx = detail::make_ctx(set, nullptr, params);
        detail::cache().put(key, ctx);
    }
    const float *dc = residuals ? residuals->d_center.data() : nullptr;
    const float *dr = residuals ? residuals->d_response.data() : nullptr;
    const float *da = residuals ? residuals->d_atten.data() : nullptr;
    out = Spectrum(set.grid);
    detail::check(swr_rasterize(ctx.get(), dc, dr, da, 1, out.data.data()));
    // the workspace contents the reference leaves behind (splat.cpp:159-294)
    const int n = set.n;
    ws.state.assign(std::size_t(11) * n, 0.0f);
    ws.row_range.assign(std::size_t(2) * n, 0);
    ws.col_range.assign(std::size_t(2) * n, 0);
    std::vector<int32_t> per_prim(std::size_t(std::max(n, 1)));
    detail::check(swr_setup(ctx.get(), dc, dr, da, 1, ws.state.data(), ws.row_range.data(), ws.col_range.data(),
                            per_prim.data()));
    swr_scene_info info{};
    detail::check(swr_scene_get_info(ctx.get(), &info));
    const int t = params.tile < 1 ? 16 : params.tile;
    const int tiles = ((set.grid.n_elevation + t - 1) / t) * ((set.grid.n_azimuth + t - 1) / t);
    ws.tile_offset.assign(std::size_t(tiles) + 1, 0);
    int64_t pairs = 0;
    detail::check(swr_bin(ctx.get(), dc, dr, da, 1, ws.tile_offset.data(), nullptr, 0, &pairs));
    ws.tile_prims.assign(std::size_t(pairs), 0);
    detail::check(swr_bin(ctx.get(), dc, dr, da, 1, ws.tile_offset.data(), ws.tile_prims.data(), pairs, &pairs));
    ws.tile_count.resize(std::size_t(tiles));
    for (int k = 0; k < tiles; k++)
        ws.tile_count[std::size_t(k)] = ws.tile_offset[std::size_t(k) + 1] - ws.tile_offset[std::size_t(k)];
    ws.el_center.resize(std::size_t(set.grid.n_elevation));
    ws.az_center.resize(std::size_t(set.grid.n_azimuth));
    for (int i = 0; i < set.grid.n_elevation; i++)
        ws.el_center[std::size_t(i)] = float(set.grid.elevation_center(i));
    for (int j = 0; j < set.grid.n_azimuth; j++)
        ws.az_center[std::size_t(j)] = float(set.grid.azimuth_center(j));
}

template <class T>
SpectrumT<T> rasterize(const GaussianSetT<T> &set, const ResidualsT<T> *residuals, const RasterParamsT<T> &params)
{
    SpectrumT<T> out;
    RasterWorkspaceT<T> ws;
    rasterize(set, residuals, params, out, ws);
    return out;
}

// context-explicit form (the scene of a loaded checkpoint, no workspace)
inline void rasterize(const train::Checkpoint &ck, const Residuals *res, Spectrum &out)
{
    const auto g = ck.grid();
    out.grid = g;
    out.data.assign(size_t(2) * g.cells(), 0.0f);
    if (res && res->n != ck.info().n)
        throw std::invalid_argument("residual count does not match the primitive count");
    detail::check(swr_rasterize(ck.handle(), res ? res->d_center.data() : nullptr,
                                res ? res->d_response.data() : nullptr, res ? res->d_atten.data() : nullptr, 1,
                                out.data.data()));
}
} // namespace splat

namespace deform
{
// deform.hpp:106-109: residuals of every primitive at one normalized position
template <class T>
void predict_residuals(const DeformNetT<T> &net, const splat::GaussianSetT<T> &set, const std::array<T, 3> &position,
                       DeformWorkspaceT<T> &ws, splat::ResidualsT<T> &out)
{
    detail::check_set(set);
    if (net.trunk.size() != 8)
        throw std::invalid_argument("deform net must have 8 trunk layers");
    const std::uint64_t key = detail::net_key(detail::set_key(set), net);
    auto ctx = detail::cache().find(key);
    if (!ctx)
    {
        ctx = detail::make_ctx(set, &net, splat::RasterParams{});
        detail::cache().put(key, ctx);
    }
    out.resize(set.n);
    ws.n = set.n;
    detail::check(swr_predict_residuals(ctx.get(), position.data(), 1, out.d_center.data(), out.d_response.data(),
                                        out.d_atten.data()));
}

// context-explicit form
inline void predict_residuals(const train::Checkpoint &ck, const std::array<float, 3> &pos01, splat::Residuals &out)
{
    const int n = ck.info().n;
    out.resize(n);
    detail::check(swr_predict_residuals(ck.handle(), pos01.data(), 1, out.d_center.data(), out.d_response.data(),
                                        out.d_atten.data()));
}
} // namespace deform

namespace tasks
{
// tasks.hpp:71-77
struct AoAEstimate
{
    int row = 0, col = 0;
    double azimuth = 0.0, elevation = 0.0;
};

namespace detail_heads
{
inline void heads(swr_ctx *ctx, const Spectrum &s, double &pooled, int32_t rc[2], double ang[2])
{
    if (s.grid.cells() < 1)
        throw std::invalid_argument("empty spectrum");
    if (s.data.size() != std::size_t(2) * s.grid.cells())
        throw std::invalid_argument("spectrum data does not match its grid");
    detail::check(swr_heads(ctx, s.data.data(), 1, &pooled, rc, ang));
}
} // namespace detail_heads

// tasks.hpp:79 / tasks.cpp:154-169: argmax |A| (first maximum in row-major order)
inline AoAEstimate aoa_extract(const Spectrum &s)
{
    if (s.grid.cells() < 1)
        throw std::invalid_argument("empty spectrum");
    int32_t rc[2];
    double ang[2], pooled;
    detail_heads::heads(detail::grid_ctx(s.grid).get(), s, pooled, rc, ang);
    return {rc[0], rc[1], ang[1], ang[0]};
}

// tasks.hpp:41 / tasks.cpp:32-39: mean |A| over the spectrum
inline double pooled_magnitude(const Spectrum &s)
{
    int32_t rc[2];
    double ang[2], pooled;
    detail_heads::heads(detail::grid_ctx(s.grid).get(), s, pooled, rc, ang);
    return pooled;
}

// context-explicit forms
inline AoAEstimate aoa_extract(const train::Checkpoint &ck, const Spectrum &s)
{
    int32_t rc[2];
    double ang[2], pooled;
    detail_heads::heads(ck.handle(), s, pooled, rc, ang);
    return {rc[0], rc[1], ang[1], ang[0]};
}

inline double pooled_magnitude(const train::Checkpoint &ck, const Spectrum &s)
{
    int32_t rc[2];
    double ang[2], pooled;
    detail_heads::heads(ck.handle(), s, pooled, rc, ang);
    return pooled;
}
} // namespace tasks

// spectrum.hpp:73-84: evaluation metrics (the context supplies the grid)
inline double psnr(const train::Checkpoint &ck, const Spectrum &a, const Spectrum &b, double peak = 1.0)
{
    if (a.data.size() != b.data.size())
        throw std::invalid_argument("spectrum shape mismatch");
    double v = 0.0;
    detail::check(swr_metrics(ck.handle(), a.data.data(), b.data.data(), 1, peak, &v, nullptr, nullptr));
    return v;
}
inline double ssim(const train::Checkpoint &ck, const Spectrum &a, const Spectrum &b, double peak = 1.0)
{
    if (a.data.size() != b.data.size())
        throw std::invalid_argument("spectrum shape mismatch");
    double v = 0.0;
    detail::check(swr_metrics(ck.handle(), a.data.data(), b.data.data(), 1, peak, nullptr, &v, nullptr));
    return v;
}
inline double l1(const train::Checkpoint &ck, const Spectrum &a, const Spectrum &b)
{
    if (a.data.size() != b.data.size())
        throw std::invalid_argument("spectrum shape mismatch");
    double v = 0.0;
    detail::check(swr_metrics(ck.handle(), a.data.data(), b.data.data(), 1, 1.0, nullptr, nullptr, &v));
    return v;
}

// spectrum.hpp:73-84 with the reference's signatures (the grid comes from the spectra)
namespace detail
{
inline double metric(const Spectrum &a, const Spectrum &b, double peak, int which)
{
    if (!(a.grid == b.grid) || a.data.size() != b.data.size() || a.data.size() != std::size_t(2) * a.grid.cells())
        throw std::invalid_argument("spectrum shape mismatch");
    double v[3] = {0.0, 0.0, 0.0};
    check(swr_metrics(grid_ctx(a.grid).get(), a.data.data(), b.data.data(), 1, peak, which == 0 ? &v[0] : nullptr,
                      which == 1 ? &v[1] : nullptr, which == 2 ? &v[2] : nullptr));
    return v[which];
}
} // namespace detail
inline double psnr(const Spectrum &a, const Spectrum &b, double peak = 1.0) { return detail::metric(a, b, peak, 0); }
inline double ssim(const Spectrum &a, const Spectrum &b, double peak = 1.0) { return detail::metric(a, b, peak, 1); }
inline double l1(const Spectrum &a, const Spectrum &b) { return detail::metric(a, b, 1.0, 2); }

namespace train
{
// spectrum.hpp:99-104
struct MetricRow
{
    int sample_id = 0;
    double psnr_db = 0.0, ssim = 0.0, l1 = 0.0;
};

// train::evaluate (training.cpp:380-406) over (position, target spectrum) samples
inline std::vector<MetricRow> evaluate(const Checkpoint &ck, const std::vector<std::array<float, 3>> &positions,
                                       const std::vector<Spectrum> &targets)
{
    if (positions.size() != targets.size())
        throw std::invalid_argument("one target spectrum per position");
    const size_t B = positions.size();
    std::vector<float> pos(3 * B), tgt;
    for (size_t b = 0; b < B; b++)
    {
        for (int a = 0; a < 3; a++)
            pos[3 * b + a] = positions[b][a];
        tgt.insert(tgt.end(), targets[b].data.begin(), targets[b].data.end());
    }
    std::vector<double> p(B), s(B), l(B);
    detail::check(swr_evaluate(ck.handle(), pos.data(), tgt.data(), (int64_t)B, 1.0, p.data(), s.data(), l.data()));
    std::vector<MetricRow> rows(B);
    for (size_t b = 0; b < B; b++)
        rows[b] = {int(b), p[b], s[b], l[b]};
    return rows;
}
} // namespace train

namespace splat
{
// splat.hpp:77-89
struct RenderGrads
{
    int n = 0;
    std::vector<float> center_raw, cholesky, atten_logit, response, d_center, d_response, d_atten;
};

// splat::rasterize_backward (splat.cpp:494-669) for one position
inline RenderGrads rasterize_backward(const train::Checkpoint &ck, const Residuals *res, const Spectrum &upstream)
{
    const int n = ck.info().n;
    if (res && res->n != n)
        throw std::invalid_argument("residual count does not match the primitive count");
    if (upstream.data.size() != size_t(2) * ck.grid().cells())
        throw std::invalid_argument("upstream spectrum does not match the grid");
    RenderGrads g;
    g.n = n;
    g.center_raw.assign(size_t(2) * n, 0.f);
    g.cholesky.assign(size_t(3) * n, 0.f);
    g.atten_logit.assign(size_t(n), 0.f);
    g.response.assign(size_t(2) * n, 0.f);
    g.d_center.assign(size_t(2) * n, 0.f);
    g.d_response.assign(size_t(2) * n, 0.f);
    g.d_atten.assign(size_t(n), 0.f);
    detail::check(swr_rasterize_backward(ck.handle(), res ? res->d_center.data() : nullptr,
                                         res ? res->d_response.data() : nullptr, res ? res->d_atten.data() : nullptr,
                                         1, upstream.data.data(), g.center_raw.data(), g.cholesky.data(),
                                         g.atten_logit.data(), g.response.data(), g.d_center.data(),
                                         g.d_response.data(), g.d_atten.data()));
    return g;
}
} // namespace splat

namespace train
{
// training.hpp:63-68
struct LossTerms
{
    double loss = 0.0, l1_term = 0.0, ssim_term = 0.0;
};

// train::hybrid_loss (training.cpp:62-106); grad may be null
inline LossTerms hybrid_loss(const Checkpoint &ck, const Spectrum &prediction, const Spectrum &target, double lambda1,
                             Spectrum *grad)
{
    if (prediction.data.size() != target.data.size() || prediction.data.size() != size_t(2) * ck.grid().cells())
        throw std::invalid_argument("spectrum shape mismatch");
    double t[3];
    if (grad)
    {
        grad->grid = prediction.grid;
        grad->data.assign(prediction.data.size(), 0.f);
    }
    detail::check(swr_hybrid_loss(ck.handle(), prediction.data.data(), target.data.data(), 1, lambda1, t,
                                  grad ? grad->data.data() : nullptr));
    return {t[0], t[1], t[2]};
}

// TrainConfig (training.hpp:96-112), the reference defaults
inline swr_train_config default_config()
{
    swr_train_config c;
    swr_train_config_default(&c);
    return c;
}

// train::train (training.cpp:198-376) on one B200: returns the trained model
// saved to `out_path` (a WRFC the reference loads) and the per-iteration
// (loss, l1_term, ssim_term) rows of its log
inline std::vector<std::array<double, 3>> train(const std::string &dataset_dir, const swr_train_config &cfg,
                                                const std::string &out_path, const char *resume_path = nullptr,
                                                int device = 0)
{
    swr_dataset *ds = nullptr;
    detail::check(swr_dataset_open(dataset_dir.c_str(), &ds));
    std::unique_ptr<swr_dataset, void (*)(swr_dataset *)> dsg(ds, &swr_dataset_close);
    swr_trainer *tr = nullptr;
    detail::check(swr_trainer_create(&cfg, ds, resume_path, device, &tr));
    std::unique_ptr<swr_trainer, void (*)(swr_trainer *)> trg(tr, &swr_trainer_destroy);
    const int64_t todo = std::max<int64_t>(0, cfg.coarse_iters + cfg.fine_iters - swr_trainer_iteration(tr));
    std::vector<std::array<double, 3>> log(static_cast<size_t>(todo));
    int64_t done = 0;
    double ms = 0.0;
    detail::check(swr_trainer_run(tr, todo, todo ? log[0].data() : nullptr, &done, &ms));
    log.resize(size_t(done));
    detail::check(swr_trainer_save(tr, out_path.c_str()));
    return log;
}
} // namespace train

namespace sim
{
// wavesim.hpp:32-39
struct ArrayConfig
{
    int k_elements = 16;
    double spacing = 0.0625;
    double wavelength = 0.125;
};

// SteeringTable + beam_scan (wavesim.cpp:183-252) on the device
class BeamScanner
{
  public:
    BeamScanner(const ArrayConfig &a, const AngularGrid &g, int device = 0) : grid_(g), k_(a.k_elements)
    {
        swr_steering *st = nullptr;
        detail::check(swr_steering_create(a.k_elements, a.spacing, a.wavelength, g.n_elevation, g.n_azimuth, device,
                                          &st));
        st_.reset(st);
    }
    // channels [B][K] complex -> spectra [B][cells][2] (double)
    std::vector<double> scan(const std::vector<std::complex<double>> &channels) const
    {
        const int64_t B = int64_t(channels.size()) / k_;
        std::vector<double> out(size_t(B) * 2 * grid_.cells());
        detail::check(swr_beam_scan(st_.get(), reinterpret_cast<const double *>(channels.data()), B, out.data()));
        return out;
    }

  private:
    AngularGrid grid_;
    int k_;
    std::unique_ptr<swr_steering, void (*)(swr_steering *)> st_{nullptr, &swr_steering_destroy};
};
} // namespace sim

} // namespace wrfsplat::b200
