// C entry points into the reference library built from /root/reference sources.
// TEST INFRASTRUCTURE ONLY (the CPU checker and the `--impl reference` bench arm):
// nothing in the product links or loads this. Every function forwards to the
// reference's own public API:
//   train::load_checkpoint / save_checkpoint   checkpoint.cpp:100-146 / :51-98
//   train::normalize_position / render_at      training.cpp:178-195
//   deform::predict_residuals                  deform.hpp:106-109 (restated GEMM, see deform_restated.cpp)
//   splat::rasterize (workspace exposed)        splat.cpp:312-482, prepare() :159-294
//   tasks::aoa_extract / pooled_magnitude       tasks.cpp:154-169 / :32-39
// Exceptions are caught and mapped to status codes (0 ok, 1 invalid_argument,
// 2 runtime_error, 3 other) with the message kept for wref_last_error().

#include <omp.h>

#include <complex>
#include <cstring>
#include <stdexcept>
#include <string>

#include "wrfsplat/deform.hpp"
#include "wrfsplat/splat.hpp"
#include "wrfsplat/tasks.hpp"
#include "wrfsplat/training.hpp"
#include "wrfsplat/wavesim.hpp"

using namespace wrfsplat;

namespace
{
thread_local std::string g_err;

template <class F>
int guarded(F &&f)
{
    try
    {
        f();
        return 0;
    }
    catch (const std::invalid_argument &e)
    {
        g_err = e.what();
        return 1;
    }
    catch (const std::runtime_error &e)
    {
        g_err = e.what();
        return 2;
    }
    catch (const std::exception &e)
    {
        g_err = e.what();
        return 3;
    }
}

train::Checkpoint *ck_of(void *h) { return static_cast<train::Checkpoint *>(h); }

void fill_spectrum(const Spectrum &s, float *dst)
{
    std::memcpy(dst, s.data.data(), s.data.size() * sizeof(float));
}

Spectrum wrap_spectrum(const float *src, int H, int W)
{
    Spectrum s(AngularGrid{H, W});
    std::memcpy(s.data.data(), src, s.data.size() * sizeof(float));
    return s;
}
} // namespace

extern "C" {

const char *wref_last_error() { return g_err.c_str(); }

void wref_set_threads(int n) { omp_set_num_threads(n); }
int wref_max_threads() { return omp_get_max_threads(); }

void *wref_ck_load(const char *path)
{
    train::Checkpoint *out = nullptr;
    const int rc = guarded([&] { out = new train::Checkpoint(train::load_checkpoint(path)); });
    return rc == 0 ? out : nullptr;
}

// Build a checkpoint from raw arrays. lw/lb hold the 11 layers in WRFD order
// (8 trunk, center, response, atten head); lw == nullptr leaves the net empty
// (rasterize-only scenes).
void *wref_ck_create(int H, int W, int n, const float *center_raw, const float *cholesky,
                     const float *atten_logit, const float *response, int width, int bands_c,
                     int bands_p, const float *const *lw, const float *const *lb, float cutoff,
                     int tile, const double *bbox_min, const double *bbox_max)
{
    auto *ck = new train::Checkpoint();
    const int rc = guarded([&] {
        ck->set.grid = AngularGrid{H, W};
        ck->set.resize(n);
        std::memcpy(ck->set.center_raw.data(), center_raw, sizeof(float) * 2 * std::size_t(n));
        std::memcpy(ck->set.cholesky.data(), cholesky, sizeof(float) * 3 * std::size_t(n));
        std::memcpy(ck->set.atten_logit.data(), atten_logit, sizeof(float) * std::size_t(n));
        std::memcpy(ck->set.response.data(), response, sizeof(float) * 2 * std::size_t(n));
        ck->config.raster.cutoff_radius = cutoff;
        ck->config.raster.tile = tile;
        ck->config.primitives = n;
        if (lw)
        {
            ck->net.width = width;
            ck->net.enc.bands_center = bands_c;
            ck->net.enc.bands_position = bands_p;
            ck->config.width = width;
            ck->config.enc = ck->net.enc;
            Rng dummy(0);
            ck->net.init(dummy); // allocates shapes; every value is overwritten below
            deform::DeformNet::Layer *ls[11];
            for (int i = 0; i < 8; i++)
                ls[i] = &ck->net.trunk[std::size_t(i)];
            ls[8] = &ck->net.head_center;
            ls[9] = &ck->net.head_response;
            ls[10] = &ck->net.head_atten;
            for (int i = 0; i < 11; i++)
            {
                std::memcpy(ls[i]->w.data(), lw[i], sizeof(float) * ls[i]->w.size());
                std::memcpy(ls[i]->b.data(), lb[i], sizeof(float) * ls[i]->b.size());
            }
        }
        for (int a = 0; a < 3; a++)
        {
            ck->bbox_min[std::size_t(a)] = bbox_min ? bbox_min[a] : 0.0;
            ck->bbox_max[std::size_t(a)] = bbox_max ? bbox_max[a] : 1.0;
        }
    });
    if (rc != 0)
    {
        delete ck;
        return nullptr;
    }
    return ck;
}

// tasks::save_rssi_model (tasks.cpp:131-137): the checkpoint + calibration keys
int wref_save_rssi_model(void *h, const char *path, double slope, double intercept)
{
    return guarded([&] {
        tasks::RssiModel m;
        m.ck = *ck_of(h);
        m.slope = slope;
        m.intercept = intercept;
        tasks::save_rssi_model(path, m);
    });
}

// tasks::load_rssi_model (tasks.cpp:139-150): calibration of an RSSI model file
int wref_load_rssi_model(const char *path, double *slope_intercept)
{
    return guarded([&] {
        const auto m = tasks::load_rssi_model(path);
        slope_intercept[0] = m.slope;
        slope_intercept[1] = m.intercept;
    });
}

int wref_ck_save(void *h, const char *path)
{
    return guarded([&] { train::save_checkpoint(path, *ck_of(h)); });
}

void wref_ck_free(void *h) { delete ck_of(h); }

// grid (H, W), n, net width and bands, raster params, bbox (6 doubles)
int wref_ck_info(void *h, int *ints6, float *cutoff, double *bbox6)
{
    const auto &ck = *ck_of(h);
    ints6[0] = ck.set.grid.n_elevation;
    ints6[1] = ck.set.grid.n_azimuth;
    ints6[2] = ck.set.n;
    ints6[3] = ck.net.width;
    ints6[4] = ck.net.enc.bands_center;
    ints6[5] = ck.config.raster.tile;
    *cutoff = ck.config.raster.cutoff_radius;
    for (int a = 0; a < 3; a++)
    {
        bbox6[a] = ck.bbox_min[std::size_t(a)];
        bbox6[3 + a] = ck.bbox_max[std::size_t(a)];
    }
    return ck.net.enc.bands_position;
}

// Copy out the Gaussian set and the 11 layers (caller sizes the buffers)
int wref_ck_arrays(void *h, float *center_raw, float *cholesky, float *atten, float *response,
                   float *const *lw, float *const *lb)
{
    const auto &ck = *ck_of(h);
    const auto &s = ck.set;
    std::memcpy(center_raw, s.center_raw.data(), sizeof(float) * s.center_raw.size());
    std::memcpy(cholesky, s.cholesky.data(), sizeof(float) * s.cholesky.size());
    std::memcpy(atten, s.atten_logit.data(), sizeof(float) * s.atten_logit.size());
    std::memcpy(response, s.response.data(), sizeof(float) * s.response.size());
    if (lw && ck.net.trunk.size() == 8)
    {
        const deform::DeformNet::Layer *ls[11];
        for (int i = 0; i < 8; i++)
            ls[i] = &ck.net.trunk[std::size_t(i)];
        ls[8] = &ck.net.head_center;
        ls[9] = &ck.net.head_response;
        ls[10] = &ck.net.head_atten;
        for (int i = 0; i < 11; i++)
        {
            std::memcpy(lw[i], ls[i]->w.data(), sizeof(float) * ls[i]->w.size());
            std::memcpy(lb[i], ls[i]->b.data(), sizeof(float) * ls[i]->b.size());
        }
    }
    return 0;
}

int wref_normalize(void *h, const float *pos_m, float *out01)
{
    return guarded([&] {
        const auto p = train::normalize_position(*ck_of(h), {pos_m[0], pos_m[1], pos_m[2]});
        out01[0] = p[0];
        out01[1] = p[1];
        out01[2] = p[2];
    });
}

int wref_predict(void *h, const float *pos01, float *d_center, float *d_response, float *d_atten)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        deform::DeformWorkspace ws;
        splat::Residuals res;
        deform::predict_residuals(ck.net, ck.set, {pos01[0], pos01[1], pos01[2]}, ws, res);
        std::memcpy(d_center, res.d_center.data(), sizeof(float) * res.d_center.size());
        std::memcpy(d_response, res.d_response.data(), sizeof(float) * res.d_response.size());
        std::memcpy(d_atten, res.d_atten.data(), sizeof(float) * res.d_atten.size());
    });
}

// rasterize(set, residuals-or-null, params) and expose the workspace.
// state: n*11 floats, rows/cols: n*2 ints, tile_offset: tiles+1 ints,
// tile_prims: up to prims_cap ints (the true pair count lands in *n_pairs).
int wref_rasterize(void *h, const float *d_center, const float *d_response, const float *d_atten,
                   float *spectrum, float *state, int *rows, int *cols, int *tile_offset,
                   int *tile_prims, long long prims_cap, long long *n_pairs)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        splat::Residuals res;
        const splat::Residuals *rp = nullptr;
        if (d_center)
        {
            res.resize(ck.set.n);
            std::memcpy(res.d_center.data(), d_center, sizeof(float) * res.d_center.size());
            std::memcpy(res.d_response.data(), d_response, sizeof(float) * res.d_response.size());
            std::memcpy(res.d_atten.data(), d_atten, sizeof(float) * res.d_atten.size());
            rp = &res;
        }
        splat::RasterWorkspace ws;
        Spectrum out;
        splat::rasterize<float>(ck.set, rp, ck.config.raster, out, ws);
        if (spectrum)
            fill_spectrum(out, spectrum);
        if (state)
            std::memcpy(state, ws.state.data(), sizeof(float) * ws.state.size());
        if (rows)
            std::memcpy(rows, ws.row_range.data(), sizeof(int) * ws.row_range.size());
        if (cols)
            std::memcpy(cols, ws.col_range.data(), sizeof(int) * ws.col_range.size());
        if (tile_offset)
            std::memcpy(tile_offset, ws.tile_offset.data(), sizeof(int) * ws.tile_offset.size());
        if (n_pairs)
            *n_pairs = (long long)ws.tile_prims.size();
        if (tile_prims)
        {
            const std::size_t m = std::min<std::size_t>(ws.tile_prims.size(), std::size_t(prims_cap));
            std::memcpy(tile_prims, ws.tile_prims.data(), sizeof(int) * m);
        }
    });
}

// rasterize_backward(set, residuals-or-null, params, upstream): the seven
// RenderGrads fields, concatenated in declaration order into `grads`
// (n * (2+3+1+2+2+2+1) floats).
int wref_rasterize_backward(void *h, const float *d_center, const float *d_response, const float *d_atten,
                            const float *upstream, float *grads)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        splat::Residuals res;
        const splat::Residuals *rp = nullptr;
        if (d_center)
        {
            res.resize(ck.set.n);
            std::memcpy(res.d_center.data(), d_center, sizeof(float) * res.d_center.size());
            std::memcpy(res.d_response.data(), d_response, sizeof(float) * res.d_response.size());
            std::memcpy(res.d_atten.data(), d_atten, sizeof(float) * res.d_atten.size());
            rp = &res;
        }
        const Spectrum up = wrap_spectrum(upstream, ck.set.grid.n_elevation, ck.set.grid.n_azimuth);
        const auto g = splat::rasterize_backward<float>(ck.set, rp, ck.config.raster, up);
        float *dst = grads;
        for (const auto *v : {&g.center_raw, &g.cholesky, &g.atten_logit, &g.response, &g.d_center, &g.d_response,
                              &g.d_atten})
        {
            std::memcpy(dst, v->data(), sizeof(float) * v->size());
            dst += v->size();
        }
    });
}

// hybrid_loss(prediction, target, lambda1, grad-or-null): terms = (loss,
// l1_term, ssim_term); returns 1 on the reference's non-finite error.
int wref_hybrid_loss(const float *pred, const float *target, int H, int W, double lambda1, double *terms, float *grad)
{
    try
    {
        const auto p = wrap_spectrum(pred, H, W), t = wrap_spectrum(target, H, W);
        Spectrum g;
        const auto lt = train::hybrid_loss<float>(p, t, lambda1, grad ? &g : nullptr);
        terms[0] = lt.loss;
        terms[1] = lt.l1_term;
        terms[2] = lt.ssim_term;
        if (grad)
            fill_spectrum(g, grad);
        return 0;
    }
    catch (const std::runtime_error &)
    {
        return 1;
    }
    catch (const std::exception &)
    {
        return 2;
    }
}

int wref_render_at(void *h, const float *pos_m, float *spectrum)
{
    return guarded([&] {
        const auto s = train::render_at(*ck_of(h), {pos_m[0], pos_m[1], pos_m[2]});
        fill_spectrum(s, spectrum);
    });
}

// Batched consumer loop over render_at (the CPU baseline).
// mode 0: reference as shipped — positions in sequence, OpenMP inside each render.
// mode 1: position-parallel — one position per thread, nested regions serial.
// Any output pointer may be null. aoa_rc = [B][2] ints, aoa_ang = [B][2] (el, az).
int wref_render_batch(void *h, int B, const float *pos_m, float *spectra, double *pooled,
                      int *aoa_rc, double *aoa_ang, int mode)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        const std::size_t per = std::size_t(2) * ck.set.grid.cells();
        auto one = [&](int b) {
            const Spectrum s = train::render_at(ck, {pos_m[3 * b], pos_m[3 * b + 1], pos_m[3 * b + 2]});
            if (spectra)
                std::memcpy(spectra + per * std::size_t(b), s.data.data(), per * sizeof(float));
            if (pooled)
                pooled[b] = tasks::pooled_magnitude(s);
            if (aoa_rc || aoa_ang)
            {
                const auto e = tasks::aoa_extract(s);
                if (aoa_rc)
                {
                    aoa_rc[2 * b] = e.row;
                    aoa_rc[2 * b + 1] = e.col;
                }
                if (aoa_ang)
                {
                    aoa_ang[2 * b] = e.elevation;
                    aoa_ang[2 * b + 1] = e.azimuth;
                }
            }
        };
        if (mode == 0)
        {
            for (int b = 0; b < B; b++)
                one(b);
        }
        else
        {
            const int keep = omp_get_max_active_levels();
            omp_set_max_active_levels(1);
            std::string first_err;
#pragma omp parallel for schedule(dynamic, 1)
            for (int b = 0; b < B; b++)
            {
                try
                {
                    one(b);
                }
                catch (const std::exception &e)
                {
#pragma omp critical
                    first_err = e.what();
                }
            }
            omp_set_max_active_levels(keep);
            if (!first_err.empty())
                throw std::runtime_error(first_err);
        }
    });
}

int wref_aoa(const float *spectrum, int H, int W, int *row, int *col, double *el, double *az)
{
    return guarded([&] {
        const auto e = tasks::aoa_extract(wrap_spectrum(spectrum, H, W));
        *row = e.row;
        *col = e.col;
        *el = e.elevation;
        *az = e.azimuth;
    });
}

double wref_pooled(const float *spectrum, int H, int W)
{
    return tasks::pooled_magnitude(wrap_spectrum(spectrum, H, W));
}

// spectrum.cpp:145-250 on the reference's own functions: out = (psnr, ssim, l1).
// Returns 0, 1 for std::domain_error (non-finite), 2 for std::invalid_argument.
int wref_metrics(const float *a, const float *b, int H, int W, double peak, double *out)
{
    try
    {
        const auto sa = wrap_spectrum(a, H, W), sb = wrap_spectrum(b, H, W);
        out[0] = psnr(sa, sb, peak);
        out[2] = l1(sa, sb);
        out[1] = ssim(sa, sb, peak);
        return 0;
    }
    catch (const std::domain_error &)
    {
        return 1;
    }
    catch (const std::invalid_argument &)
    {
        return 2;
    }
}

int wref_magnitude(const float *spectrum, int H, int W, float *out)
{
    const auto m = magnitude(wrap_spectrum(spectrum, H, W));
    std::memcpy(out, m.data(), sizeof(float) * m.size());
    return 0;
}

void wref_materialize_center_f(float rel, float raz, float *el, float *az)
{
    const auto c = splat::materialize_center<float>(rel, raz);
    *el = c.elevation;
    *az = c.azimuth;
}

void wref_materialize_center_d(double rel, double raz, double *el, double *az)
{
    const auto c = splat::materialize_center<double>(rel, raz);
    *el = c.elevation;
    *az = c.azimuth;
}

int wref_encode_f(const float *values, int count, int bands, float *out)
{
    deform::encode<float>(values, count, bands, out);
    return 0;
}

float wref_kernel_weight(void *h, int idx, float az, float el, const float *d_center,
                         const float *d_response, const float *d_atten)
{
    float out = -1.0f;
    guarded([&] {
        const auto &ck = *ck_of(h);
        splat::Residuals res;
        const splat::Residuals *rp = nullptr;
        if (d_center)
        {
            res.resize(ck.set.n);
            std::memcpy(res.d_center.data(), d_center, sizeof(float) * res.d_center.size());
            std::memcpy(res.d_response.data(), d_response, sizeof(float) * res.d_response.size());
            std::memcpy(res.d_atten.data(), d_atten, sizeof(float) * res.d_atten.size());
            rp = &res;
        }
        out = splat::kernel_weight<float>(ck.set, idx, az, el, rp);
    });
    return out;
}

// The reference's init_random + DeformNet::init for seeded parity scenes
// (splat.cpp:681-709, deform.cpp:72-102; draw order: set, then net).
void *wref_ck_init_random(int H, int W, int n, unsigned long long seed)
{
    auto *ck = new train::Checkpoint();
    const int rc = guarded([&] {
        Rng rng(seed);
        ck->set = splat::init_random(AngularGrid{H, W}, n, rng);
        ck->net.init(rng);
        ck->config.primitives = n;
        ck->bbox_min = {0, 0, 0};
        ck->bbox_max = {1, 1, 1};
    });
    if (rc != 0)
    {
        delete ck;
        return nullptr;
    }
    return ck;
}

// ----------------------------------------------------------- datasets
// Simulate a dataset with the reference's own physics (default shoebox scene,
// positions sampled 0.3 m from the walls) and save it (dataset.cpp:61-157, 184-203).
int wref_make_dataset(const char *dir, int H, int W, int count, unsigned long long seed,
                      unsigned long long *hash, double *bbox6)
{
    return guarded([&] {
        sim::Scene scene;
        Rng rng(seed);
        const auto positions = sim::sample_positions(scene, count, 0.3, rng);
        const auto ds = sim::generate_dataset(scene, AngularGrid{H, W}, positions, seed);
        sim::save_dataset(ds, dir);
        *hash = ds.manifest_hash;
        for (int a = 0; a < 3; a++)
        {
            bbox6[a] = ds.bbox_min[std::size_t(a)];
            bbox6[3 + a] = ds.bbox_max[std::size_t(a)];
        }
    });
}

// load_dataset (dataset.cpp:205-258): sample count, hash, and the records in file order
long long wref_dataset_load(const char *dir, unsigned long long *hash, float *pos, float *spectra, long long cap)
{
    long long n = -1;
    guarded([&] {
        const auto ds = sim::load_dataset(dir);
        *hash = ds.manifest_hash;
        n = (long long)ds.samples.size();
        if (pos && spectra)
            for (long long i = 0; i < n && i < cap; i++)
            {
                const auto &smp = ds.samples[std::size_t(i)];
                std::memcpy(pos + 3 * i, smp.position.data(), 12);
                std::memcpy(spectra + i * smp.spectrum.data.size(), smp.spectrum.data.data(),
                            4 * smp.spectrum.data.size());
            }
    });
    return n;
}

void wref_ck_set_dataset(void *h, unsigned long long hash, const double *bbox6)
{
    auto &ck = *ck_of(h);
    ck.manifest_hash = hash;
    for (int a = 0; a < 3; a++)
    {
        ck.bbox_min[std::size_t(a)] = bbox6[a];
        ck.bbox_max[std::size_t(a)] = bbox6[3 + a];
    }
}

// train::train(load_dataset(dir), cfg, log_path, resume) -> a new checkpoint
// handle (nullptr on error; *kind = 1 invalid_argument, 2 hash_mismatch, 3 other).
// ints5 = primitives, bands_center, bands_position, width, tile;
// dbl5 = cutoff_radius, lr_gaussian, lr_mlp, lambda1, anneal_scale;
// ll3 = coarse_iters, fine_iters, anneal_threshold.
void *wref_train(const char *dir, const int *ints5, const double *dbl5, const long long *ll3,
                 unsigned long long seed, const char *log_path, void *resume, int *kind)
{
    *kind = 0;
    try
    {
        const auto ds = sim::load_dataset(dir);
        train::TrainConfig cfg;
        cfg.primitives = ints5[0];
        cfg.enc.bands_center = ints5[1];
        cfg.enc.bands_position = ints5[2];
        cfg.width = ints5[3];
        cfg.raster.tile = ints5[4];
        cfg.raster.cutoff_radius = float(dbl5[0]);
        cfg.lr_gaussian = dbl5[1];
        cfg.lr_mlp = dbl5[2];
        cfg.lambda1 = dbl5[3];
        cfg.anneal_scale = dbl5[4];
        cfg.coarse_iters = ll3[0];
        cfg.fine_iters = ll3[1];
        cfg.anneal_threshold = ll3[2];
        cfg.seed = seed;
        return new train::Checkpoint(
            train::train(ds, cfg, log_path ? std::string(log_path) : std::string(), resume ? ck_of(resume) : nullptr));
    }
    catch (const train::hash_mismatch &e)
    {
        g_err = e.what();
        *kind = 2;
    }
    catch (const std::invalid_argument &e)
    {
        g_err = e.what();
        *kind = 1;
    }
    catch (const std::exception &e)
    {
        g_err = e.what();
        *kind = 3;
    }
    return nullptr;
}

// The training iteration's gradient chain at the checkpoint's parameters
// (training.cpp:320-345): pos01 != nullptr = fine (predict_residuals ->
// rasterize -> hybrid_loss -> rasterize_backward -> deform_backward), else
// coarse. grads7 = RenderGrads fields concatenated; gw/gb = DeformGrads.
int wref_gradients(void *h, const float *pos01, const float *target, double lambda1, double *terms, float *grads7,
                   float *const *gw, float *const *gb)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        const Spectrum tgt = wrap_spectrum(target, ck.set.grid.n_elevation, ck.set.grid.n_azimuth);
        splat::RasterWorkspace rws;
        Spectrum pred, lgrad;
        splat::RenderGrads g;
        deform::DeformWorkspace dws;
        splat::Residuals res;
        const splat::Residuals *rp = nullptr;
        if (pos01)
        {
            deform::predict_residuals(ck.net, ck.set, {pos01[0], pos01[1], pos01[2]}, dws, res);
            rp = &res;
        }
        splat::rasterize<float>(ck.set, rp, ck.config.raster, pred, rws);
        const auto lt = train::hybrid_loss(pred, tgt, lambda1, &lgrad);
        terms[0] = lt.loss;
        terms[1] = lt.l1_term;
        terms[2] = lt.ssim_term;
        splat::rasterize_backward<float>(ck.set, rp, ck.config.raster, lgrad, g, rws);
        float *dst = grads7;
        for (const auto *v : {&g.center_raw, &g.cholesky, &g.atten_logit, &g.response, &g.d_center, &g.d_response,
                              &g.d_atten})
        {
            std::memcpy(dst, v->data(), sizeof(float) * v->size());
            dst += v->size();
        }
        if (pos01)
        {
            splat::Residuals rg;
            rg.resize(ck.set.n);
            rg.d_center = g.d_center;
            rg.d_response = g.d_response;
            rg.d_atten = g.d_atten;
            deform::DeformGrads dg;
            dg.resize_like(ck.net);
            deform::deform_backward(ck.net, dws, rg, dg);
            const deform::DeformNet::Layer *L[11];
            for (int i = 0; i < 8; i++)
                L[i] = &dg.trunk[std::size_t(i)];
            L[8] = &dg.head_center;
            L[9] = &dg.head_response;
            L[10] = &dg.head_atten;
            for (int i = 0; i < 11; i++)
            {
                std::memcpy(gw[i], L[i]->w.data(), sizeof(float) * L[i]->w.size());
                std::memcpy(gb[i], L[i]->b.data(), sizeof(float) * L[i]->b.size());
            }
        }
    });
}

// deform_backward (deform.cpp:264-326) after predict_residuals at pos01 for a
// given upstream dL/dresiduals; gw/gb = DeformGrads in layer_list order
int wref_deform_backward(void *h, const float *pos01, const float *up_c, const float *up_r, const float *up_a,
                         float *const *gw, float *const *gb)
{
    return guarded([&] {
        const auto &ck = *ck_of(h);
        deform::DeformWorkspace dws;
        splat::Residuals res, up;
        deform::predict_residuals(ck.net, ck.set, {pos01[0], pos01[1], pos01[2]}, dws, res);
        up.resize(ck.set.n);
        std::memcpy(up.d_center.data(), up_c, sizeof(float) * up.d_center.size());
        std::memcpy(up.d_response.data(), up_r, sizeof(float) * up.d_response.size());
        std::memcpy(up.d_atten.data(), up_a, sizeof(float) * up.d_atten.size());
        deform::DeformGrads dg;
        dg.resize_like(ck.net);
        deform::deform_backward(ck.net, dws, up, dg);
        const deform::DeformNet::Layer *L[11];
        for (int i = 0; i < 8; i++)
            L[i] = &dg.trunk[std::size_t(i)];
        L[8] = &dg.head_center;
        L[9] = &dg.head_response;
        L[10] = &dg.head_atten;
        for (int i = 0; i < 11; i++)
        {
            std::memcpy(gw[i], L[i]->w.data(), sizeof(float) * L[i]->w.size());
            std::memcpy(gb[i], L[i]->b.data(), sizeof(float) * L[i]->b.size());
        }
    });
}

// build_steering_table (wavesim.cpp:183-211) for the default array geometry
// overrides; wr/wi [cells][k]
int wref_steering_table(int k, double spacing, double wavelength, int H, int W, double *wr, double *wi)
{
    return guarded([&] {
        sim::ArrayConfig a;
        a.k_elements = k;
        a.spacing = spacing;
        a.wavelength = wavelength;
        const auto t = sim::build_steering_table(a, AngularGrid{H, W});
        std::memcpy(wr, t.wr.data(), sizeof(double) * t.wr.size());
        std::memcpy(wi, t.wi.data(), sizeof(double) * t.wi.size());
    });
}

// beam_scan(channel, array, grid) (wavesim.cpp:213-259); channel [k][2], out [cells][2]
int wref_beam_scan(int k, double spacing, double wavelength, int H, int W, const double *channel, double *out)
{
    return guarded([&] {
        sim::ArrayConfig a;
        a.k_elements = k;
        a.spacing = spacing;
        a.wavelength = wavelength;
        std::vector<std::complex<double>> h(static_cast<std::size_t>(k));
        for (int e = 0; e < k; e++)
            h[std::size_t(e)] = {channel[2 * e], channel[2 * e + 1]};
        const auto s = sim::beam_scan(h, a, AngularGrid{H, W});
        std::memcpy(out, s.data.data(), sizeof(double) * s.data.size());
    });
}

// the channels generate_dataset scans for wref_make_dataset's positions
// (dataset.cpp:61-84: default Scene, sample_positions(scene, count, 0.3,
// Rng(seed)), trace_paths, channel_response): channels [count][K][2], valid [count]
int wref_sample_channels(int count, unsigned long long seed, double *channels, int *valid)
{
    return guarded([&] {
        sim::Scene scene;
        Rng rng(seed);
        const auto positions = sim::sample_positions(scene, count, 0.3, rng);
        const int k = scene.array.k_elements;
        for (int i = 0; i < count; i++)
        {
            const auto paths = sim::trace_paths(scene, positions[std::size_t(i)]);
            valid[i] = paths.empty() ? 0 : 1;
            const auto h = sim::channel_response(paths, scene.array);
            for (int e = 0; e < k; e++)
            {
                channels[(std::size_t(i) * k + e) * 2] = h[std::size_t(e)].real();
                channels[(std::size_t(i) * k + e) * 2 + 1] = h[std::size_t(e)].imag();
            }
        }
    });
}

void wref_ck_set_iteration(void *h, long long it) { ck_of(h)->iteration = it; }
long long wref_ck_iteration(void *h) { return ck_of(h)->iteration; }

// train::evaluate (training.cpp:380-406) on a saved dataset: rows [n][4] =
// (sample id, psnr, ssim, l1); returns the row count (-1 on error, -2 on hash mismatch)
long long wref_evaluate(void *h, const char *dir, int split, double *rows, long long cap)
{
    long long n = -1;
    try
    {
        const auto ds = sim::load_dataset(dir);
        const auto r = train::evaluate(*ck_of(h), ds, split == 0 ? train::Split::train
                                                                 : split == 1 ? train::Split::test : train::Split::all);
        n = (long long)r.size();
        for (long long i = 0; i < n && i < cap; i++)
        {
            rows[4 * i] = r[std::size_t(i)].sample_id;
            rows[4 * i + 1] = r[std::size_t(i)].psnr_db;
            rows[4 * i + 2] = r[std::size_t(i)].ssim;
            rows[4 * i + 3] = r[std::size_t(i)].l1;
        }
    }
    catch (const train::hash_mismatch &e)
    {
        g_err = e.what();
        n = -2;
    }
    catch (const std::exception &e)
    {
        g_err = e.what();
        n = -1;
    }
    return n;
}

// The acceptance gate's criterion-1 instances, replayed exactly
// (acceptance.cpp:130-147 random_float_set, :159-199 criterion_1): one
// wrfsplat::Rng(20250814) stream, 50 instances, grid <= 16 x 32, n <= 64,
// odd instances with residuals U[-0.05, 0.05], cutoff off. Per instance i
// (arrays padded to 64 primitives / 16 x 32 cells):
//   hwn[3i..]            H, W, n
//   cr[i][64][2], ch[i][64][3], at[i][64], rs[i][64][2], dc/dr[i][64][2], da[i][64]
//   out[i][16*32*2]      splat::rasterize<float> (the reference's tiled forward)
//   dense[i][16*32*2]    the criterion's FP64 dense oracle, restated from
//                        acceptance.cpp:53-109 (kernel_oracle + dense_oracle)
int wref_criterion1(int *hwn, float *cr, float *ch, float *at, float *rs, float *dc, float *dr, float *da,
                    float *out, double *dense)
{
    return guarded([&] {
        Rng rng(20250814);
        for (int inst = 0; inst < 50; inst++)
        {
            const AngularGrid g{4 + int(rng.index(13)), 8 + int(rng.index(25))};
            const int n = 1 + int(rng.index(64));
            splat::GaussianSetT<float> set;
            set.grid = g;
            set.resize(n);
            for (int p = 0; p < n; p++)
            {
                set.center_raw[2 * std::size_t(p)] = float(rng.uniform(-1.5, 1.5));
                set.center_raw[2 * std::size_t(p) + 1] = float(rng.uniform(-1.5, 1.5));
                set.cholesky[3 * std::size_t(p)] = float(rng.uniform(0.05, 0.4));
                set.cholesky[3 * std::size_t(p) + 1] = float(rng.uniform(-0.2, 0.2));
                set.cholesky[3 * std::size_t(p) + 2] = float(rng.uniform(0.05, 0.4));
                set.atten_logit[std::size_t(p)] = float(rng.uniform(-1.0, 1.0));
                set.response[2 * std::size_t(p)] = float(rng.uniform(-0.5, 0.5));
                set.response[2 * std::size_t(p) + 1] = float(rng.uniform(-0.5, 0.5));
            }
            splat::ResidualsT<float> res;
            const bool with_res = (inst % 2) == 1;
            if (with_res)
            {
                res.resize(n);
                for (auto *vec : {&res.d_center, &res.d_response})
                    for (auto &v : *vec)
                        v = float(rng.uniform(-0.05, 0.05));
                for (auto &v : res.d_atten)
                    v = float(rng.uniform(-0.05, 0.05));
            }
            splat::RasterParams pr;
            pr.cutoff_radius = 0.0f;
            const auto o = splat::rasterize<float>(set, with_res ? &res : nullptr, pr);
            hwn[3 * inst] = g.n_elevation;
            hwn[3 * inst + 1] = g.n_azimuth;
            hwn[3 * inst + 2] = n;
            const std::size_t P = std::size_t(inst) * 64;
            std::memcpy(cr + 2 * P, set.center_raw.data(), sizeof(float) * 2 * n);
            std::memcpy(ch + 3 * P, set.cholesky.data(), sizeof(float) * 3 * n);
            std::memcpy(at + P, set.atten_logit.data(), sizeof(float) * n);
            std::memcpy(rs + 2 * P, set.response.data(), sizeof(float) * 2 * n);
            if (with_res)
            {
                std::memcpy(dc + 2 * P, res.d_center.data(), sizeof(float) * 2 * n);
                std::memcpy(dr + 2 * P, res.d_response.data(), sizeof(float) * 2 * n);
                std::memcpy(da + P, res.d_atten.data(), sizeof(float) * n);
            }
            std::memcpy(out + std::size_t(inst) * 1024, o.data.data(), sizeof(float) * o.data.size());
            // dense FP64 oracle (acceptance.cpp:53-109)
            const double pi = 3.141592653589793238462643383279502884;
            double *dd = dense + std::size_t(inst) * 1024;
            for (int i = 0; i < g.n_elevation; i++)
                for (int j = 0; j < g.n_azimuth; j++)
                {
                    const std::size_t c = std::size_t(i) * g.n_azimuth + j;
                    double sre = 0.0, sim = 0.0;
                    for (int p = 0; p < n; p++)
                    {
                        double c_el = pi / 4 * (std::tanh(double(set.center_raw[2 * std::size_t(p)])) + 1.0);
                        double c_az = pi * (std::tanh(double(set.center_raw[2 * std::size_t(p) + 1])) + 1.0);
                        const double l1 = std::max(double(set.cholesky[3 * std::size_t(p)]), double(splat::chol_floor));
                        const double l2 = set.cholesky[3 * std::size_t(p) + 1];
                        const double l3 = std::max(double(set.cholesky[3 * std::size_t(p) + 2]), double(splat::chol_floor));
                        double delta = 1.0 / (1.0 + std::exp(-double(set.atten_logit[std::size_t(p)])));
                        double re = set.response[2 * std::size_t(p)], im = set.response[2 * std::size_t(p) + 1];
                        if (with_res)
                        {
                            c_el += res.d_center[2 * std::size_t(p)];
                            c_az += res.d_center[2 * std::size_t(p) + 1];
                            delta = std::min(std::max(delta + double(res.d_atten[std::size_t(p)]), 0.0), 1.0);
                            re += res.d_response[2 * std::size_t(p)];
                            im += res.d_response[2 * std::size_t(p) + 1];
                        }
                        const double d0 = g.elevation_center(i) - c_el;
                        double d1 = g.azimuth_center(j) - c_az;
                        while (d1 >= pi)
                            d1 -= 2.0 * pi;
                        while (d1 < -pi)
                            d1 += 2.0 * pi;
                        const double s00 = l1 * l1, s01 = l1 * l2, s11 = l2 * l2 + l3 * l3;
                        const double det = s00 * s11 - s01 * s01;
                        const double q = (s11 * d0 * d0 - 2.0 * s01 * d0 * d1 + s00 * d1 * d1) / det;
                        const double k = delta * std::exp(-0.5 * q);
                        sre += re * k;
                        sim += im * k;
                    }
                    dd[2 * c] = sre;
                    dd[2 * c + 1] = sim;
                }
        }
    });
}

} // extern "C"
