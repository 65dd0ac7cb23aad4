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

#include <array>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <future>
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
    mode = j.at("mode").get<std::string>();
    if (mode != "tx_moving" && mode != "rx_moving") // mobility_from_string, wavesim.cpp:67-74
        throw std::invalid_argument("unknown mobility mode: " + mode);
    k_elements = j.at("array").at("k_elements").get<int>();
    spacing = j.at("array").at("spacing").get<double>();
    wavelength = j.at("array").at("wavelength").get<double>();
    const auto rm = j.at("scene").at("room").get<std::array<double, 3>>();
    const auto fx = j.at("scene").at("fixed_node").get<std::array<double, 3>>();
    for (int a = 0; a < 3; a++)
    {
        room[a] = rm[a];
        fixed_node[a] = fx[a];
    }
    reflectivity = j.at("scene").at("reflectivity").get<double>();
    max_bounces = j.at("scene").at("max_bounces").get<int>();
    seed = j.at("seed").get<uint64_t>();
    rssi_dbm = j.at("rssi_dbm").get<std::vector<double>>();
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

// manifest_json (dataset.cpp:159-181): same keys, same value types, nlohmann's
// dump(2) (std::map order, its shortest round-trip doubles) + newline, so the
// bytes -- and the FNV-1a fingerprint checkpoints carry -- match the reference's.
static std::string manifest_of(const swr_dataset_meta &m, int64_t sample_count)
{
    if (!m.mode)
        throw std::invalid_argument("null mode");
    const std::string mode(m.mode);
    if (mode != "tx_moving" && mode != "rx_moving")
        throw std::invalid_argument("unknown mobility mode: " + mode);
    auto ints = [](const int32_t *p, int64_t n) {
        if (n < 0 || (n > 0 && !p))
            throw std::invalid_argument("bad index array");
        return std::vector<int>(p, p + n);
    };
    auto arr3 = [](const double *v) { return std::array<double, 3>{v[0], v[1], v[2]}; };
    nlohmann::json j;
    j["format"] = "wrfsplat-dataset";
    j["version"] = 1;
    j["mode"] = mode;
    j["grid"] = {{"n_elevation", m.n_elevation}, {"n_azimuth", m.n_azimuth}};
    j["array"] = {{"k_elements", m.k_elements}, {"spacing", m.spacing}, {"wavelength", m.wavelength}};
    j["scene"] = {{"room", arr3(m.room)},
                  {"reflectivity", m.reflectivity},
                  {"max_bounces", m.max_bounces},
                  {"fixed_node", arr3(m.fixed_node)}};
    j["normalization"] = m.normalization;
    j["seed"] = m.seed;
    j["sample_count"] = int(sample_count);
    j["train_indices"] = ints(m.train_indices, m.n_train);
    j["test_indices"] = ints(m.test_indices, m.n_test);
    j["excluded_indices"] = ints(m.excluded_indices, m.n_excluded);
    j["bbox_min"] = arr3(m.bbox_min);
    j["bbox_max"] = arr3(m.bbox_max);
    if (m.n_rssi < 0 || (m.n_rssi > 0 && !m.rssi_dbm))
        throw std::invalid_argument("bad rssi array");
    j["rssi_dbm"] = std::vector<double>(m.rssi_dbm, m.rssi_dbm + m.n_rssi);
    return j.dump(2) + "\n";
}

} // namespace swr

using namespace swr;

// save_dataset (dataset.cpp:183-203) as a stream: spectra.bin is written record by
// record (position as 3 float32, then [H][W][2] float32), manifest.json at close
struct swr_dataset_writer
{
    std::string dir;
    int H = 0, W = 0;
    FILE *f = nullptr;
    int64_t written = 0;
    std::vector<float> rec;
    ~swr_dataset_writer()
    {
        if (f)
            std::fclose(f);
    }
    void put(const float *pos, const float *spec, int64_t count)
    {
        const size_t cells2 = size_t(2) * H * W;
        rec.resize(3 + cells2);
        for (int64_t k = 0; k < count; k++)
        {
            std::memcpy(rec.data(), pos + 3 * k, 12);
            std::memcpy(rec.data() + 3, spec + cells2 * k, 4 * cells2);
            if (std::fwrite(rec.data(), 4, rec.size(), f) != rec.size())
                throw std::runtime_error("cannot write " + dir + "/spectra.bin");
        }
        written += count;
    }
};

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

int swr_dataset_get_meta(swr_dataset *ds, swr_dataset_meta *m)
{
    return swr_guarded([&] {
        if (!ds || !m)
            throw std::invalid_argument("null argument");
        const DatasetFile &d = ds->d;
        m->n_elevation = d.H;
        m->n_azimuth = d.W;
        m->mode = d.mode.c_str();
        m->k_elements = d.k_elements;
        m->spacing = d.spacing;
        m->wavelength = d.wavelength;
        m->reflectivity = d.reflectivity;
        m->max_bounces = d.max_bounces;
        m->normalization = d.normalization;
        m->seed = d.seed;
        for (int a = 0; a < 3; a++)
        {
            m->room[a] = d.room[a];
            m->fixed_node[a] = d.fixed_node[a];
            m->bbox_min[a] = d.bbox_min[a];
            m->bbox_max[a] = d.bbox_max[a];
        }
        static_assert(sizeof(int) == sizeof(int32_t), "int32 indices");
        m->train_indices = reinterpret_cast<const int32_t *>(d.train.data());
        m->test_indices = reinterpret_cast<const int32_t *>(d.test.data());
        m->excluded_indices = reinterpret_cast<const int32_t *>(d.excluded.data());
        m->n_train = int64_t(d.train.size());
        m->n_test = int64_t(d.test.size());
        m->n_excluded = int64_t(d.excluded.size());
        m->rssi_dbm = d.rssi_dbm.data();
        m->n_rssi = int64_t(d.rssi_dbm.size());
    });
}

int swr_dataset_manifest_json(const swr_dataset_meta *meta, int64_t sample_count, char *buf, size_t cap,
                              size_t *len, uint64_t *hash)
{
    return swr_guarded([&] {
        if (!meta)
            throw std::invalid_argument("null meta");
        const std::string m = manifest_of(*meta, sample_count);
        if (len)
            *len = m.size();
        if (hash)
            *hash = fnv1a64(m.data(), m.size());
        if (buf)
        {
            if (cap < m.size())
                throw std::invalid_argument("manifest buffer too small");
            std::memcpy(buf, m.data(), m.size());
        }
    });
}

int swr_dataset_writer_open(const char *dir, int32_t n_elevation, int32_t n_azimuth, swr_dataset_writer **out)
{
    return swr_guarded([&] {
        if (!dir || !out)
            throw std::invalid_argument("null argument");
        if (n_elevation < 1 || n_azimuth < 1)
            throw std::invalid_argument("grid dimensions must be positive");
        std::filesystem::create_directories(dir);
        auto w = std::make_unique<swr_dataset_writer>();
        w->dir = dir;
        w->H = n_elevation;
        w->W = n_azimuth;
        w->f = std::fopen((w->dir + "/spectra.bin").c_str(), "wb");
        if (!w->f)
            throw std::runtime_error("cannot write " + w->dir + "/spectra.bin");
        *out = w.release();
    });
}

int swr_dataset_writer_append(swr_dataset_writer *w, const float *pos, const float *spectra, int64_t count)
{
    return swr_guarded([&] {
        if (!w || (count > 0 && (!pos || !spectra)))
            throw std::invalid_argument("null argument");
        if (count < 0)
            throw std::invalid_argument("negative count");
        w->put(pos, spectra, count);
    });
}

int swr_dataset_writer_render(swr_dataset_writer *w, swr_ctx *ctx, const float *pos_m, int64_t count)
{
    return swr_guarded([&] {
        if (!w || !ctx || (count > 0 && !pos_m))
            throw std::invalid_argument("null argument");
        if (count < 0)
            throw std::invalid_argument("negative count");
        swr_scene_info info{};
        if (swr_scene_get_info(ctx, &info) != SWR_OK)
            throw std::runtime_error(swr_last_error());
        if (info.n_elevation != w->H || info.n_azimuth != w->W)
            throw std::invalid_argument("scene grid differs from the dataset writer's");
        const int64_t chunk = 256;
        const size_t cells2 = size_t(2) * w->H * w->W;
        // two pinned staging buffers: chunk k's records go to the file on a worker
        // thread while chunk k+1 renders
        float *stage[2] = {nullptr, nullptr};
        for (auto &p : stage)
            check_cuda(cudaMallocHost((void **)&p, sizeof(float) * cells2 * chunk), "pinned staging");
        std::future<void> pending;
        try
        {
            for (int64_t b0 = 0, k = 0; b0 < count; b0 += chunk, k++)
            {
                const int64_t n = std::min(chunk, count - b0);
                float *buf = stage[k & 1];
                if (pending.valid() && k >= 2)
                    pending.get(); // the write that used this buffer (k - 2) is done
                const int rc = swr_render(ctx, pos_m + 3 * b0, n, SWR_OUT_SPECTRA, buf, nullptr, nullptr, nullptr,
                                          nullptr);
                if (rc != SWR_OK)
                    throw std::runtime_error(swr_last_error());
                if (pending.valid())
                    pending.get();
                pending = std::async(std::launch::async, [w, pos_m, b0, n, buf] { w->put(pos_m + 3 * b0, buf, n); });
            }
            if (pending.valid())
                pending.get();
        }
        catch (...)
        {
            if (pending.valid())
                pending.wait();
            for (auto p : stage)
                cudaFreeHost(p);
            throw;
        }
        for (auto p : stage)
            cudaFreeHost(p);
    });
}

int swr_dataset_writer_close(swr_dataset_writer *w, const swr_dataset_meta *meta, uint64_t *manifest_hash)
{
    std::unique_ptr<swr_dataset_writer> own(w);
    return swr_guarded([&] {
        if (!w || !meta)
            throw std::invalid_argument("null argument");
        if (meta->n_elevation != w->H || meta->n_azimuth != w->W)
            throw std::invalid_argument("manifest grid differs from the records'");
        const std::string m = manifest_of(*meta, w->written);
        if (std::fclose(w->f) != 0)
        {
            w->f = nullptr;
            throw std::runtime_error("cannot write " + w->dir + "/spectra.bin");
        }
        w->f = nullptr;
        std::ofstream os(w->dir + "/manifest.json", std::ios::binary);
        if (!os)
            throw std::runtime_error("cannot write " + w->dir + "/manifest.json");
        os << m;
        os.close();
        if (!os)
            throw std::runtime_error("cannot write " + w->dir + "/manifest.json");
        if (manifest_hash)
            *manifest_hash = fnv1a64(m.data(), m.size());
    });
}

int swr_dataset_save(const char *dir, const swr_dataset_meta *meta, const float *pos, const float *spectra,
                     int64_t count, uint64_t *manifest_hash)
{
    if (!meta)
        return swr_guarded([] { throw std::invalid_argument("null meta"); });
    swr_dataset_writer *w = nullptr;
    int rc = swr_dataset_writer_open(dir, meta->n_elevation, meta->n_azimuth, &w);
    if (rc != SWR_OK)
        return rc;
    rc = swr_dataset_writer_append(w, pos, spectra, count);
    if (rc != SWR_OK)
    {
        delete w;
        return rc;
    }
    return swr_dataset_writer_close(w, meta, manifest_hash);
}

} // extern "C"
