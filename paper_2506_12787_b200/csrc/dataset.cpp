// Dataset I/O: the on-disk format on either
// side of render / evaluate. A dataset directory holds manifest.json and
// spectra.bin (wavesim.hpp:159-163, dataset.cpp:159-258): one record per sample
// in manifest order, position as 3 float32 then [H][W][2] float32, little
// endian, nothing after the last record. This reader validates the manifest
// like load_dataset (format / version, sizes), hashes the manifest bytes with
// FNV-1a 64 (common.cpp:40-48, the fingerprint checkpoints carry) and serves
// records by index with positioned reads, so evaluation streams chunks instead
// of loading every spectrum.
#include "swr.h"
#include "swr_internal.h"

#include <json.hpp>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace swr
{

uint64_t fnv1a64(const void *data, size_t size)
{
    const auto *p = static_cast<const unsigned char *>(data);
    uint64_t h = 0xcbf29ce484222325ull; // FNV-1a 64 offset basis
    for (size_t i = 0; i < size; i++)
    {
        h ^= p[i];
        h *= 0x100000001b3ull; // FNV prime
    }
    return h;
}

DatasetFile::~DatasetFile()
{
    if (fp)
        std::fclose(static_cast<FILE *>(fp));
}

void DatasetFile::open(const std::string &dir)
{
    std::ifstream mf(dir + "/manifest.json", std::ios::binary);
    if (!mf)
        throw std::runtime_error("cannot open " + dir + "/manifest.json");
    std::stringstream buf;
    buf << mf.rdbuf();
    const std::string manifest = buf.str();
    const auto j = nlohmann::json::parse(manifest);
    if (j.value("format", "") != "wrfsplat-dataset" || j.value("version", 0) != 1)
        throw std::runtime_error(dir + "/manifest.json is not a version-1 dataset manifest");
    H = j.at("grid").at("n_elevation").get<int>();
    W = j.at("grid").at("n_azimuth").get<int>();
    count = j.at("sample_count").get<int64_t>();
    train = j.at("train_indices").get<std::vector<int>>();
    test = j.at("test_indices").get<std::vector<int>>();
    excluded = j.at("excluded_indices").get<std::vector<int>>();
    const auto bmin = j.at("bbox_min").get<std::vector<double>>(), bmax = j.at("bbox_max").get<std::vector<double>>();
    for (int a = 0; a < 3; a++)
    {
        bbox_min[a] = bmin.at(a);
        bbox_max[a] = bmax.at(a);
    }
    normalization = j.at("normalization").get<double>();
    hash = fnv1a64(manifest.data(), manifest.size());
    if (H < 1 || W < 1 || count < 0)
        throw std::runtime_error(dir + "/manifest.json has an invalid grid or sample count");
    for (const auto *v : {&train, &test})
        for (int i : *v)
            if (i < 0 || i >= count)
                throw std::runtime_error(dir + "/manifest.json has a split index out of range");

    FILE *f = std::fopen((dir + "/spectra.bin").c_str(), "rb");
    if (!f)
        throw std::runtime_error("cannot open " + dir + "/spectra.bin");
    fp = f;
    record_floats = 3 + int64_t(2) * H * W;
    std::fseek(f, 0, SEEK_END);
    const int64_t bytes = (int64_t)std::ftell(f);
    const int64_t want = count * record_floats * 4;
    // load_dataset reads count records sequentially and then requires EOF
    if (bytes < want)
        throw std::runtime_error("unexpected end of file");
    if (bytes > want)
        throw std::runtime_error(dir + "/spectra.bin has trailing bytes");
}

void DatasetFile::read(const int32_t *idx, int64_t n, float *pos, float *spectra) const
{
    FILE *f = static_cast<FILE *>(fp);
    const int64_t cells2 = record_floats - 3;
    std::vector<float> rec(static_cast<size_t>(record_floats));
    for (int64_t k = 0; k < n; k++)
    {
        const int64_t i = idx ? idx[k] : k;
        if (i < 0 || i >= count)
            throw std::invalid_argument("sample index out of range");
        if (std::fseek(f, long(i * record_floats * 4), SEEK_SET) != 0 ||
            std::fread(rec.data(), 4, size_t(record_floats), f) != size_t(record_floats))
            throw std::runtime_error("unexpected end of file");
        if (pos)
            std::memcpy(pos + 3 * k, rec.data(), 12);
        if (spectra)
            std::memcpy(spectra + cells2 * k, rec.data() + 3, 4 * size_t(cells2));
    }
}

std::vector<int> DatasetFile::split(int which) const
{
    if (which == 0)
        return train;
    if (which == 1)
        return test;
    std::vector<int> all(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; i++)
        all[size_t(i)] = int(i);
    return all;
}

} // namespace swr

using namespace swr;

extern "C" {

int swr_dataset_open(const char *dir, swr_dataset **out)
{
    return swr_guarded([&] {
        if (!dir || !out)
            throw std::invalid_argument("null argument");
        auto *h = new swr_dataset();
        try
        {
            h->d.open(dir);
        }
        catch (...)
        {
            delete h;
            throw;
        }
        *out = h;
    });
}

void swr_dataset_close(swr_dataset *ds) { delete ds; }

int swr_dataset_get_info(swr_dataset *ds, swr_dataset_info *info)
{
    return swr_guarded([&] {
        const DatasetFile &d = ds->d;
        info->n_elevation = d.H;
        info->n_azimuth = d.W;
        info->samples = d.count;
        info->n_train = int64_t(d.train.size());
        info->n_test = int64_t(d.test.size());
        info->n_excluded = int64_t(d.excluded.size());
        info->manifest_hash = d.hash;
        info->normalization = d.normalization;
        for (int a = 0; a < 3; a++)
        {
            info->bbox_min[a] = d.bbox_min[a];
            info->bbox_max[a] = d.bbox_max[a];
        }
    });
}

int swr_dataset_split(swr_dataset *ds, int split, int32_t *indices, int64_t *count)
{
    return swr_guarded([&] {
        if (split < 0 || split > 2)
            throw std::invalid_argument("split must be 0 (train), 1 (test) or 2 (all)");
        const auto v = ds->d.split(split);
        *count = int64_t(v.size());
        if (indices)
            std::memcpy(indices, v.data(), sizeof(int32_t) * v.size());
    });
}

int swr_dataset_read(swr_dataset *ds, const int32_t *indices, int64_t count, float *pos, float *spectra)
{
    return swr_guarded([&] {
        if (count < 0)
            throw std::invalid_argument("negative count");
        ds->d.read(indices, count, pos, spectra);
    });
}

} // extern "C"
