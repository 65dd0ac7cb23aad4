// Drop-in demo of the C++ host API (include/swr.hpp): the reference's
// eval_aoa / predict_pooled loop shape (tasks.cpp:54-57, 171-206) written
// against wrfsplat::b200 instead of wrfsplat. Prints one line per position:
//   <index> <sum of spectrum values> <pooled magnitude> <aoa row> <aoa col>
#include "swr.hpp"

#include <cstdio>
#include <cstdlib>

namespace w = wrfsplat::b200;

int main(int argc, char **argv)
{
    if (argc < 5 || (argc - 2) % 3 != 0)
    {
        std::fprintf(stderr, "usage: %s checkpoint.wrfc x y z [x y z ...]\n", argv[0]);
        return 2;
    }
    try
    {
        const auto ck = w::train::load_checkpoint(argv[1]);
        std::vector<std::array<float, 3>> pos;
        for (int a = 2; a + 2 < argc; a += 3)
            pos.push_back({float(std::atof(argv[a])), float(std::atof(argv[a + 1])), float(std::atof(argv[a + 2]))});
        const auto spectra = w::train::render_batch(ck, pos);
        for (size_t b = 0; b < spectra.size(); b++)
        {
            double sum = 0.0;
            for (float v : spectra[b].data)
                sum += v;
            const auto aoa = w::tasks::aoa_extract(ck, spectra[b]);
            std::printf("%zu %.9g %.17g %d %d\n", b, sum, w::tasks::pooled_magnitude(ck, spectra[b]), aoa.row, aoa.col);
        }
        // single-position path, residuals and rasterize parity with render_at
        const auto p01 = w::train::normalize_position(ck, pos[0]);
        w::splat::Residuals res;
        w::deform::predict_residuals(ck, p01, res);
        w::Spectrum s;
        w::splat::rasterize(ck, &res, s);
        const auto one = w::train::render_at(ck, pos[0]);
        double diff = 0.0;
        for (size_t k = 0; k < s.data.size(); k++)
            diff = std::max(diff, double(std::abs(s.data[k] - one.data[k])));
        std::printf("rasterize-vs-render_at %.3g\n", diff);
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
    return 0;
}
