// A C++ caller sharding a batch over several GPUs through the library
// (train::DeviceGroup over swr_group_*): prints, per position,
//   <index> <sum of spectrum values>
// and then "max-diff-vs-render_batch <x>" against one context's render_batch.
// usage: group_demo checkpoint.wrfc n_members x y z [x y z ...]
// (members are all device 0 on a one-GPU machine: the sharding and the gather
// to the root are exercised; NCCL needs distinct devices).
#include "swr.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace w = wrfsplat::b200;

int main(int argc, char **argv)
{
    if (argc < 6 || (argc - 3) % 3)
    {
        std::fprintf(stderr, "usage: %s checkpoint.wrfc n_members x y z [x y z ...]\n", argv[0]);
        return 2;
    }
    try
    {
        const int members = std::atoi(argv[2]);
        std::vector<std::array<float, 3>> pos;
        for (int i = 3; i + 2 < argc; i += 3)
            pos.push_back({std::strtof(argv[i], nullptr), std::strtof(argv[i + 1], nullptr),
                           std::strtof(argv[i + 2], nullptr)});
        const w::train::DeviceGroup group(argv[1], std::vector<int>(size_t(members), 0));
        const auto got = group.render_batch(pos);
        const auto ck = w::train::load_checkpoint(argv[1]);
        const auto want = w::train::render_batch(ck, pos);
        double diff = 0.0;
        for (size_t b = 0; b < pos.size(); b++)
        {
            double sum = 0.0;
            for (size_t i = 0; i < got[b].data.size(); i++)
            {
                sum += got[b].data[i];
                diff = std::fmax(diff, std::fabs(double(got[b].data[i]) - double(want[b].data[i])));
            }
            std::printf("%zu %.9g\n", b, sum);
        }
        std::printf("max-diff-vs-render_batch %.3g\n", diff);
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
