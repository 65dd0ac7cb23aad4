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

#include <complex>
#include <algorithm>
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
