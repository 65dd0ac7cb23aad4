// swr.hpp — C++ host API over the C ABI (swr.h), mirroring the reference's
// render-path API so that callers switch by namespace:
//
//   reference (/root/reference/proj/include/wrfsplat)        this header
//   -----------------------------------------------------    -------------------------------------------
//   train::load_checkpoint(path)          training.hpp:133    wrfsplat::b200::train::load_checkpoint
//   train::normalize_position(ck, pos)    training.hpp:149    wrfsplat::b200::train::normalize_position
//   train::render_at(ck, pos)             training.hpp:154    wrfsplat::b200::train::render_at
//   (loop over render_at)                                     wrfsplat::b200::train::render_batch
//   deform::predict_residuals(...)        deform.hpp:106      wrfsplat::b200::deform::predict_residuals
//   splat::rasterize(set, res, params)    splat.hpp:152       wrfsplat::b200::splat::rasterize
//   tasks::pooled_magnitude(spectrum)     tasks.hpp:41        wrfsplat::b200::tasks::pooled_magnitude
//   tasks::aoa_extract(spectrum)          tasks.hpp:79        wrfsplat::b200::tasks::aoa_extract
//
// Error behaviour follows the reference: size / grid problems throw
// std::invalid_argument, I/O / format / device problems std::runtime_error.
// Header-only; link with libswr.so.
#pragma once

#include "swr.h"

#include <array>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
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
};

struct Spectrum
{
    AngularGrid grid;
    std::vector<float> data; // 2 * cells
};

namespace train
{
// A scene resident on one B200 (Gaussian set + deform net + raster params + bbox)
class Checkpoint
{
  public:
    Checkpoint() = default;
    explicit Checkpoint(swr_ctx *ctx) : ctx_(ctx, &swr_scene_destroy)
    {
        detail::check(swr_scene_get_info(ctx, &info_));
    }
    swr_ctx *handle() const { return ctx_.get(); }
    const swr_scene_info &info() const { return info_; }
    AngularGrid grid() const { return {info_.n_elevation, info_.n_azimuth}; }
    void set_option(const char *key, double value) { detail::check(swr_set_option(ctx_.get(), key, value)); }

  private:
    std::shared_ptr<swr_ctx> ctx_{nullptr, &swr_scene_destroy};
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

inline Spectrum render_at(const Checkpoint &ck, const std::array<float, 3> &position)
{
    return render_batch(ck, {position}).front();
}
} // namespace train

namespace splat
{
// splat.hpp:61-72, one position
struct Residuals
{
    int n = 0;
    std::vector<float> d_center, d_response, d_atten; // n x 2, n x 2, n
};

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
inline void predict_residuals(const train::Checkpoint &ck, const std::array<float, 3> &pos01, splat::Residuals &out)
{
    const int n = ck.info().n;
    out.n = n;
    out.d_center.assign(size_t(2) * n, 0.0f);
    out.d_response.assign(size_t(2) * n, 0.0f);
    out.d_atten.assign(size_t(n), 0.0f);
    detail::check(swr_predict_residuals(ck.handle(), pos01.data(), 1, out.d_center.data(), out.d_response.data(),
                                        out.d_atten.data()));
}
} // namespace deform

namespace tasks
{
struct AoAEstimate
{
    int row = 0, col = 0;
    double azimuth = 0.0, elevation = 0.0;
};

inline AoAEstimate aoa_extract(const train::Checkpoint &ck, const Spectrum &s)
{
    if (s.grid.cells() < 1)
        throw std::invalid_argument("empty spectrum");
    int32_t rc[2];
    double ang[2];
    double pooled;
    detail::check(swr_heads(ck.handle(), s.data.data(), 1, &pooled, rc, ang));
    return {rc[0], rc[1], ang[1], ang[0]};
}

inline double pooled_magnitude(const train::Checkpoint &ck, const Spectrum &s)
{
    int32_t rc[2];
    double ang[2];
    double pooled;
    detail::check(swr_heads(ck.handle(), s.data.data(), 1, &pooled, rc, ang));
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

} // namespace wrfsplat::b200
