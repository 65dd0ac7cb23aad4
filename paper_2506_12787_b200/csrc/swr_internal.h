// Internal types shared by the CUDA translation units of libswr.so.
#pragma once

#include <cuda_runtime.h>

// Device-side checks of the checked build (libswr_checked.so, linked by build.py next to libswr.so):
// an index or invariant that fails prints where and traps the kernel. compute-sanitizer
// is unavailable on the GPU pool, so these stand in for memcheck / racecheck on the
// render path (tests/test_checked.py). Compiled out of the product library.
#if defined(SWR_CHECKED) && defined(__CUDACC__)
#include <cstdio>
#define SWR_DCHECK(cond, what)                                                                                    \
    do                                                                                                             \
    {                                                                                                              \
        if (!(cond))                                                                                               \
        {                                                                                                          \
            printf("swr check failed: %s (%s:%d) block (%d,%d) thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
                   blockIdx.y, threadIdx.x);                                                                        \
            __trap();                                                                                              \
        }                                                                                                          \
    } while (0)
#else
#define SWR_DCHECK(cond, what)                                                                                    \
    do                                                                                                             \
    {                                                                                                              \
    } while (0)
#endif

#include <cstdint>
#include <string>
#include <algorithm>
#include <array>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace swr
{

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr int kTrunk = 8;
#ifndef SWR_KSORT
#define SWR_KSORT 2048 // measured: 2048 beats 1024, 4096, 8192 (bin 3.26 -> 2.77 ms per 1024 spectra at 50k)
#endif
constexpr int kSort = SWR_KSORT;    // pairs per sort chunk (one CTA)
constexpr int kStateStride = 11; // splat.cpp:133-147

// Per-scene constants the kernels read (passed by value).
struct Grid
{
    int H, W, n, np;      // np: n padded to a multiple of 16
    int tile, th, tw, tiles;
    int cut;              // cutoff_radius > 0
    float cut2;           // cutoff^2 or +inf
    float radius;
    double cell_el, cell_az;
};

// Device-resident static scene (per Gaussian, planar SoA, length np).
struct SceneDev
{
    float *el0, *az0;      // materialized centres (host glibc tanhf, splat.cpp:60-65)
    float *delta0;         // sigmoid(logit) (host glibc expf, splat.cpp:105-106)
    float *re0, *im0;      // response
    float4 *shape;         // (i00, i01, i11, inv_l1) — static: residuals never touch the covariance
    float *inv_l3, *l2;    // remaining state fields (parity output only)
    double2 *half;         // FP64 bbox half widths (radius*l1, radius*sqrt(l2^2+l3^2)), splat.cpp:223-225
    float *el_c, *az_c;    // float(cell centres) (splat.cpp:180-185)
    float4 *bwd;           // backward chain-rule constants (splat.cpp:633-664): (1 - tanh^2 el, az raw),
                           // l1 >= floor, l3 >= floor (1 / 0)
};

// Deformation MLP on the device.
struct NetDev
{
    int width, wp;         // width, padded width (multiple of 32)
    int bands_c, bands_p, dc, dp, d;
    float *whT;            // [7][wp][wp] hidden->hidden weights, k-major (layers 1..7), zero padded
    float *bias;           // [8][wp]
    float *cg;             // [np][4][wp] centre-encoding contribution of layers 0,2,4,6 (no bias)
    float *wpos;           // [4][wp][dp] position-encoding columns of layers 0,2,4,6
    float *wcen;           // [4][wp][dc] centre-encoding columns of layers 0,2,4,6
    float *heads;          // [5][wp] head weights (centre 2, response 2, atten 1)
    float *hbias;          // [5]
    // tcgen05 path (k_mlp_tc2.cu): fp16 hi/lo of w * 2^tc_exp[l], UMMA canonical K-major layout
    float *c_tc = nullptr;      // cg repacked per 32-Gaussian block as tcgen05.cp sources (layers 2/4/6 scaled)
    uint16_t *w_tc2 = nullptr;  // packed weights, layers 1..7, in the kernel's consumption order
    uint16_t *wh_tc2 = nullptr; // heads B operand (2 ranks x 16 columns)
    int tc_exp[9] = {};         // per-layer weight scale exponents (index l = 1..7), [8] heads
    int tc_ascale[8] = {};      // activation scale exponent k_l of each trunk layer's output (scene-load probe)
    float tc_amax[8] = {};      // the probe's largest ReLU output per trunk layer
    float *bias_tc = nullptr;   // [8][wp] bias_l x 2^k_l (read by the tensor-core epilogues)
    uint16_t *w_wide = nullptr; // width-512 tensor-core MLP (k_mlp_wide.cu): packed fp16 hi/lo weights, layers 1..7
};

// Per-chunk scratch (positions per chunk = cap_b).
struct Work
{
    int64_t cap_b = 0, cap_pairs = 0;
    float *pos01 = nullptr;     // [cap_b][4]
    float *pterm = nullptr;     // [cap_b][4][wp] position contribution (+bias) of layers 0,2,4,6
    float *res = nullptr;       // [5][cap_b][np] residual planes (dEl, dAz, dRe, dIm, dDelta)
    float4 *dyn = nullptr;      // [cap_b][np] (el, az, k_re, k_im)
    int4 *rng = nullptr;        // [cap_b][np] (r0, r1, j0, len)
    int *cnt = nullptr;         // [cap_b][np] tiles per primitive
    int64_t *seg = nullptr;     // [cap_b + 1] segment (position) base offsets into the pair array
    int *poff = nullptr;        // [cap_b][np] exclusive pair offset of each primitive within its segment
    int *tile_off = nullptr;    // [cap_b][tiles + 1] CSR offsets within the segment
    int *chunk_hist = nullptr;  // [cap_b][max_chunks][tiles]
    int max_chunks = 0;
    uint16_t *keys = nullptr;   // [cap_pairs] tile of each pair (primitive order)
    int *vals = nullptr;        // [cap_pairs] primitive of each pair (primitive order)
    int *sorted = nullptr;      // [cap_pairs] tile_prims (tile-major, primitive order inside)
    int *perm = nullptr;        // [cap_pairs] CSR slot of each emitted pair (backward only)
    bool want_perm = false;
    float4 *tile_part = nullptr; // [cap_b][tiles] (max |A|, argmax cell as float bits, sum |A| hi, lo)
    double *tile_sum = nullptr; // [cap_b][tiles]
    int64_t *stats = nullptr;      // device: (total pairs, longest segment, non-finite residual flag) of the current chunk
    unsigned long long *reruns = nullptr; // device: chunks whose fp16 MLP overflowed and re-ran in FP32 (gated path)
    // evaluation metrics (k_metrics.cu): SSIM scratch, non-finite flag, outputs, staging
    int met_cap = 0;
    double *met_tmp = nullptr, *met_out = nullptr;
    int *met_bad = nullptr;
    float *met_pred = nullptr, *met_target = nullptr;
    int64_t *host_pairs = nullptr; // pinned mirror of stats
    uint16_t *wide_act[2] = {nullptr, nullptr}; // width-512 MLP activations (fp16 hi/lo, UMMA layout)
    int64_t wide_rows = 0;
};

struct HostScene;

struct Ctx
{
    int device = 0;
    Grid g{};
    SceneDev s{};
    NetDev net{};
    bool has_net = false;
    double bbox_min[3]{}, bbox_max[3]{};
    uint64_t manifest_hash = 0; // FNV-1a of the training dataset manifest (training.hpp:124)
    float cutoff = 3.0f;
    int tile = 16;
    int mlp_precision = 0;
    int chunk = 256;
    int copy_chunk = 256; // swr_render with host spectra: positions per chunk and per raster / D2H slice
    int chunk_cap = 1 << 30;            // largest chunk whose pair list fits 32-bit offsets (pair_bound)
    int64_t pairs_per_pos_max = 1;      // pair_bound: (tile, primitive) pairs of one position, any residuals
    bool stage_timing = false;
    double rssi_slope = 1.0, rssi_intercept = 0.0;
    bool rssi_calibrated = false; // from the WRFC trailer or set through the options
    cudaStream_t stream = nullptr;
    Work w;
    int64_t launches = 0;
    int64_t pairs_last = 0;
    int64_t mlp_reruns = 0;             // chunks whose fp16 tensor-core MLP overflowed and re-ran in FP32 (sync path)
    bool pairs_on_host = true;          // pairs_last is host-known (sync path) or still in w.stats (async path)
    const int64_t *gate = nullptr;      // set while launching the FP32 re-run chain: kernels run only if *gate != 0
    size_t mem_total = 0;               // device memory, bytes (async pair-buffer budget)
    int64_t wide_block_rows = int64_t(1) << 21; // width-512 MLP: rows per layer-GEMM block (option "wide_block_rows")
    // experiment knobs (tools/experiments/round2/partition_exp.py): cap on the tcgen05 MLP's CTA pairs
    // (0 = as many as fit) and extra dynamic shared memory per MLP CTA (keeps raster CTAs off its SMs)
    int mlp_max_clusters = 0, mlp_smem_pad = 0;
    int64_t async_pair_budget = -1;     // pair-buffer bytes per chunk for the host-sync-free path (-1: default)
    double stage_ms[6]{};               // accumulated while stage_timing is on (swr_stage_times resolves)
    std::vector<std::array<cudaEvent_t, 7>> stage_pending; // recorded per chunk, read lazily
    std::vector<void *> allocs;
    void *host_stage = nullptr; // persistent staging of the host-buffer API (capi.cpp)
    std::shared_ptr<const HostScene> host; // the scene as loaded (reference layouts), for swr_scene_get_*
    cudaEvent_t order_ev = nullptr; // last work of the previous C-ABI call (StreamOrder, capi.cpp)
    bool order_pending = false;
    // a swr_render_device call is being captured into a CUDA graph (StreamOrder): no
    // allocation, host synchronisation or cross-call event may happen inside it
    bool capturing = false;
};

void check_cuda(cudaError_t e, const char *what);

// One-time setup per device (kernel attributes and occupancy queries are per
// device; thread-safe, retried if the initialiser throws).
struct DeviceOnce
{
    static constexpr int kMax = 64;
    std::once_flag flag[kMax];
    int value[kMax] = {};
    template <class F>
    int get(int dev, F &&init)
    {
        if (dev < 0 || dev >= kMax)
            throw std::invalid_argument("CUDA device ordinal out of range");
        std::call_once(flag[dev], [&] { value[dev] = init(); });
        return value[dev];
    }
};

template <class T>
inline T *dalloc(Ctx &c, size_t count)
{
    void *p = nullptr;
    if (c.capturing)
        throw std::invalid_argument("swr_render_device under CUDA-graph capture needs its work buffers sized "
                                    "first: make one uncaptured call with the same (or a larger) batch");
    check_cuda(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    c.allocs.push_back(p);
    return static_cast<T *>(p);
}

inline void dfree(Ctx &c, void *p)
{
    if (!p)
        return;
    if (c.capturing)
        throw std::invalid_argument("swr_render_device under CUDA-graph capture cannot re-size work buffers");
    cudaFree(p);
    c.allocs.erase(std::remove(c.allocs.begin(), c.allocs.end(), p), c.allocs.end());
}

template <class T>
inline T *upload(Ctx &c, const std::vector<T> &v)
{
    T *d = dalloc<T>(c, v.size());
    check_cuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return d;
}

struct HostScene
{
    int H, W, n;
    std::vector<float> center_raw, cholesky, atten, response;
    int width = 0, bands_c = 10, bands_p = 6;
    std::vector<std::vector<float>> lw, lb; // 11 layers or empty
    float cutoff = 3.0f;
    int tile = 16;
    double bmin[3] = {0, 0, 0}, bmax[3] = {1, 1, 1};
    uint64_t manifest_hash = 0; // checkpoint.cpp:40,133 (hex string in the trailer)
    std::string config_json;    // trailer "config" object (checkpoint.cpp:36), WRFC files only
    int64_t iteration = 0;      // trailer "iteration"
    bool has_rssi = false;      // trailer rssi_slope / rssi_intercept (save_rssi_model, tasks.cpp:131-150)
    double rssi_slope = 1.0, rssi_intercept = 0.0;
};

// ------------------------------------------------------------ training (k_train.cu, train.cpp)
struct AdamHp
{
    double lr, beta1, beta2, eps; // AdamParams (training.hpp:44-50)
};

// Gaussian parameters, Adam moments and gradients on the device (reference layouts)
struct GaussDev
{
    float *center, *chol, *atten, *resp;                   // [n][2], [n][3], [n], [n][2]
    float *m_center, *v_center, *m_chol, *v_chol, *m_atten, *v_atten, *m_resp, *v_resp;
    const float *g_center, *g_chol, *g_atten, *g_resp;     // rasterize_backward outputs
};

// Per-iteration arguments read on the device (so one captured iteration replays
// as a CUDA graph): entry *it of each table; log_advance bumps *it.
struct TrainSched
{
    const int *idx;     // [iters] training sample
    const float *penc;  // [iters][dp] position encoding (fine stage)
    const double *bc;   // [iters][6] Adam bias corrections (centre, rest, network)
    int64_t *it;        // device cursor
};

void launch_gauss_adam(Ctx &c, const GaussDev &gp, const AdamHp &hp, const TrainSched &sc, bool step_center,
                       bool step_rest, float floor_el, float floor_az, cudaStream_t st);
void launch_adam_flat(Ctx &c, float *p, const float *g, float *m, float *v, int64_t count, const AdamHp &hp,
                      const TrainSched &sc, cudaStream_t st);
void launch_position_encoding(Ctx &c, float *x, int d, int dc, const TrainSched &sc, int dp, cudaStream_t st);
void launch_gather_target(Ctx &c, const float *spectra, const TrainSched &sc, float *out, cudaStream_t st);
void launch_log_advance(Ctx &c, const double *terms, double *log, const TrainSched &sc, cudaStream_t st);
void launch_dense_fwd(Ctx &c, const float *a1, int ld1, int ka, const float *a2, int ld2, int K, const float *W,
                      const float *b, int width, float *h, cudaStream_t st);
void launch_heads_fwd(Ctx &c, const float *h7, int width, const float *Wh, const float *bh, float *planes,
                      int64_t plane, cudaStream_t st);
void launch_dense_bwd_input(Ctx &c, const float *dz, int width, const float *W, int cols, const float *h_prev,
                            float *dz_prev, cudaStream_t st);
size_t dw_partial_floats(int n, int R, int C);
void launch_dense_bwd_weights(Ctx &c, const float *dz, int R, const float *a1, int ld1, int ka, const float *a2,
                              int ld2, int K, float *part, float *dW, float *db, cudaStream_t st);
void launch_heads_bwd(Ctx &c, const float *d_center, const float *d_response, const float *d_atten,
                      const float *Wc, const float *Wr, const float *Wa, const float *h7, int width, float *dz7,
                      float *dr5, cudaStream_t st);

// scene / work-buffer management shared by the C ABI and the trainer (capi.cpp)
void build_scene(Ctx &c, const HostScene &hs, int device);
struct SceneFields
{
    std::vector<float> el0, az0, d0, re0, im0, il3, l2v;
    std::vector<float4> shape, bwd;
    std::vector<double2> half;
};
SceneFields scene_fields(const Grid &g, int n, const float *center_raw, const float *cholesky, const float *atten,
                         const float *response);
void refresh_scene_host(Ctx &c, const float *center_raw, const float *cholesky, const float *atten,
                        const float *response);
void ensure_work(Ctx &c, int64_t nb);
void ensure_pairs(Ctx &c, int64_t pairs, int nb, int64_t max_seg);
HostScene parse_wrfc(const char *path);

// kernels (k_mlp.cu, k_render.cu). All launch on `st` and bump ctx.launches.
void launch_pos_prep(Ctx &c, const float *d_pos_m, int nb, bool normalized, cudaStream_t st);
void launch_mlp(Ctx &c, int nb, cudaStream_t st);
void launch_center_terms(Ctx &c, const float *d_cenc, cudaStream_t st);
void launch_setup(Ctx &c, int nb, bool with_res, cudaStream_t st);
void launch_state_out(Ctx &c, int nb, bool with_res, float *d_state, cudaStream_t st);
void launch_bin_count(Ctx &c, int nb, cudaStream_t st);   // per-segment scan + segment bases
void launch_bin_sort(Ctx &c, int nb, int64_t pairs, int max_seg, cudaStream_t st);
// positions [s_base, s_base + nb) of the current chunk (the spectra pointer is the chunk's)
void launch_raster(Ctx &c, int nb, float *d_spec, bool want_heads, cudaStream_t st, int warps = 0, int s_base = 0);
void launch_heads(Ctx &c, int nb, uint32_t flags, double *d_pooled, double *d_rssi,
                  int32_t *d_aoa_rc, double *d_aoa_ang, cudaStream_t st);
void launch_heads_from_spectra(Ctx &c, int nb, const float *d_spec, cudaStream_t st);

bool mlp_tc_available();
bool mlp_uses_tc(const Ctx &c);
void probe_activations(Ctx &c, int nb, float out[8], cudaStream_t st);
void launch_mlp_tc2(Ctx &c, int nb, cudaStream_t st);
void launch_mlp_wide(Ctx &c, int nb, cudaStream_t st);
void prepare_wide_weights(Ctx &c, const std::vector<float> &whT, const std::vector<float> &heads,
                          const std::vector<float> &bias);
int mlp_tc2_trace(long long *out);
void prepare_tc2_weights(Ctx &c, const std::vector<float> &whT, const std::vector<float> &heads,
                         const std::vector<float> &bias);
size_t metrics_tmp_doubles(const Ctx &c, int nb);
void launch_metrics(Ctx &c, const float *d_pred, const float *d_target, int nb, double peak, double *d_psnr,
                    double *d_ssim, double *d_l1, double *d_tmp, int *d_bad, cudaStream_t st);
size_t loss_tmp_doubles(const Ctx &c, int nb);
void launch_raster_backward(Ctx &c, int nb, const float *d_state, const float *d_upstream, float *d_slots,
                            cudaStream_t st);
void launch_bwd_merge(Ctx &c, int nb, bool with_res, const float *d_slots, float *const out[7], cudaStream_t st);
void launch_hybrid_loss(Ctx &c, const float *d_pred, const float *d_target, int nb, double lambda1, double *d_terms,
                        float *d_grad, double *d_tmp, int *d_bad, cudaStream_t st);

void check_cuda(cudaError_t e, const char *what);
// run f, mapping the reference's exception types to swr_status (capi.cpp)
int swr_guarded(const std::function<void()> &f);

// spectra.bin + manifest.json reader (dataset.cpp, dataset.cpp:159-258 of the reference)
uint64_t fnv1a64(const void *data, size_t size);
struct DatasetFile
{
    int H = 0, W = 0;
    int64_t count = 0, record_floats = 0;
    std::vector<int> train, test, excluded;
    double bbox_min[3]{}, bbox_max[3]{}, normalization = 1.0;
    uint64_t hash = 0;
    // the rest of the manifest (round trip through the writer)
    std::string mode;
    int k_elements = 0, max_bounces = 0;
    double spacing = 0, wavelength = 0, reflectivity = 0, room[3]{}, fixed_node[3]{};
    uint64_t seed = 0;
    std::vector<double> rssi_dbm;
    void *fp = nullptr;
    ~DatasetFile();
    void open(const std::string &dir);
    void read(const int32_t *idx, int64_t n, float *pos, float *spectra) const;
    std::vector<int> split(int which) const;
};

} // namespace swr

// opaque handle of the C ABI (swr.h)
struct swr_dataset
{
    swr::DatasetFile d;
};
