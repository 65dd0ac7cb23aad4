// The reference's own callers of the render path, written the way the reference
// writes them (same calls, same argument shapes, same value types) but against
// wrfsplat::b200 -- the drop-in claim of include/swr.hpp:
//
//   evaluate   per-sample body of train::evaluate       training.cpp:387-399
//   aoa        per-sample body of tasks::eval_aoa       tasks.cpp:176-181
//   pooled     tasks::predict_pooled                    tasks.cpp:54-57
//   bench      canonical loop of wrfsplat_cli cmd_bench wrfsplat_cli.cpp:225-237
//
// Usage: ref_callers checkpoint.wrfc x y z [x y z ...]. One line per position:
//   <i> <sum pred> <psnr(pred, render_at)> <aoa row> <aoa col> <aoa az> <aoa el> <pooled>
// then "bench <pairs> <sum canonical> <tile_count total>".
#include "swr.hpp"

#include <cstdio>
#include <cstdlib>

namespace wrfsplat_b200_callers
{
using namespace wrfsplat::b200;

struct Sample
{
    std::array<float, 3> position;
};

int run(const char *path, const std::vector<Sample> &samples)
{
    const train::Checkpoint ck = train::load_checkpoint(path);

    // train::evaluate (training.cpp:387-399): workspaces reused across samples
    deform::DeformWorkspace dws;
    splat::Residuals res;
    splat::RasterWorkspace rws;
    Spectrum pred;
    for (std::size_t idx = 0; idx < samples.size(); idx++)
    {
        const auto &sample = samples[idx];
        deform::predict_residuals(ck.net, ck.set, train::normalize_position(ck, sample.position), dws, res);
        splat::rasterize<float>(ck.set, &res, ck.config.raster, pred, rws);
        // tasks::eval_aoa (tasks.cpp:180) and tasks::predict_pooled (tasks.cpp:56)
        const auto est = tasks::aoa_extract(train::render_at(ck, sample.position));
        const double pooled = tasks::pooled_magnitude(train::render_at(ck, sample.position));
        double sum = 0.0;
        for (float v : pred.data)
            sum += v;
        std::printf("%zu %.9g %.9g %d %d %.17g %.17g %.17g\n", idx, sum, psnr(pred, train::render_at(ck, sample.position)),
                    est.row, est.col, est.azimuth, est.elevation, pooled);
    }

    // wrfsplat_cli cmd_bench (wrfsplat_cli.cpp:225-237): canonical renders, one workspace
    Spectrum out;
    splat::RasterWorkspace ws;
    splat::rasterize<float>(ck.set, nullptr, ck.config.raster, out, ws);
    for (int i = 0; i < 3; i++)
        splat::rasterize<float>(ck.set, nullptr, ck.config.raster, out, ws);
    double sum = 0.0;
    for (float v : out.data)
        sum += v;
    long long counted = 0;
    for (int c : ws.tile_count)
        counted += c;
    std::printf("bench %zu %.9g %lld\n", ws.tile_prims.size(), sum, counted);
    return 0;
}
} // namespace wrfsplat_b200_callers

int main(int argc, char **argv)
{
    if (argc < 5 || (argc - 2) % 3 != 0)
    {
        std::fprintf(stderr, "usage: %s checkpoint.wrfc x y z [x y z ...]\n", argv[0]);
        return 2;
    }
    std::vector<wrfsplat_b200_callers::Sample> samples;
    for (int a = 2; a + 2 < argc; a += 3)
        samples.push_back({{float(std::atof(argv[a])), float(std::atof(argv[a + 1])), float(std::atof(argv[a + 2]))}});
    try
    {
        return wrfsplat_b200_callers::run(argv[1], samples);
    }
    catch (const std::invalid_argument &e)
    {
        std::fprintf(stderr, "invalid argument: %s\n", e.what());
        return 3;
    }
    catch (const std::exception &e)
    {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
}
