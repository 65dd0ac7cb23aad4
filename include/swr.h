/* swr.h — C ABI of the B200-native SwiftWRF spectrum renderer (libswr.so).
 *
 * This is the drop-in boundary for the reference's render path. The reference
 * (/root/reference/proj) is a statically linked C++ library with no FFI; each
 * entry point below replaces the C++ call named beside it, batched over TX
 * positions. Plain C types only (no torch, no C++); every call returns a
 * swr_status and keeps a per-thread message for swr_last_error(). The C++
 * wrapper include/swr.hpp rethrows them with the reference's exception types
 * (std::invalid_argument / std::runtime_error).
 *
 * Threading: one context per host thread, or external serialisation. A
 * context owns its device memory; host buffers are owned by the caller.
 * Layouts follow the reference: positions [B][3] metres (x, y, z); spectra
 * [B][H][W][2] interleaved (re, im), elevation the slow axis
 * (spectrum.hpp:47-60); residuals planar per field (see swr_predict_residuals).
 */
#ifndef SWR_H
#define SWR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct swr_ctx swr_ctx;

enum swr_status
{
    SWR_OK = 0,
    SWR_EINVAL = 1,   /* std::invalid_argument in the reference (size / grid mismatch) */
    SWR_ERUNTIME = 2, /* std::runtime_error (I/O, magic, version) */
    SWR_ECUDA = 3,    /* device error (no sm_100 device, launch failure, OOM) */
    SWR_EDOMAIN = 4,  /* std::domain_error (non-finite spectrum value in a metric, spectrum.cpp:44-49) */
};

/* render flags (swr_render / swr_render_device) */
#define SWR_OUT_SPECTRA 1u /* write spectra [B][H][W][2] */
#define SWR_OUT_POOLED 2u  /* pooled magnitude per position (tasks.cpp:32-39) */
#define SWR_OUT_RSSI 4u    /* slope * pooled + intercept (tasks.cpp:109) */
#define SWR_OUT_AOA 8u     /* argmax cell (row, col) + cell-centre angles (tasks.cpp:154-169) */
#define SWR_NO_RESIDUALS 16u /* canonical render: skip the deformation net (rasterize(set, nullptr)) */

/* MLP arithmetic (swr_set_option "mlp_precision") */
/* default: SWR_MLP_FP16X3 for widths <= 160, SWR_MLP_FP32 above */
#define SWR_MLP_FP32 0   /* FP32 FMA on the CUDA cores */
#define SWR_MLP_FP16X3 1 /* tcgen05, FP32-grade: fp16 hi/lo splits of scaled operands, 3 products, fp32 accumulate */
#define SWR_MLP_FP16 2   /* tcgen05 single fp16 product (fast tier, ~1e-3 relative residual error) */

typedef struct
{
    int n_elevation, n_azimuth; /* grid (spectrum.hpp:30-42) */
    int n;                      /* Gaussians */
    int width, bands_center, bands_position;
    float cutoff_radius;        /* RasterParams (splat.hpp:107-116) */
    int tile;
    double bbox_min[3], bbox_max[3];
    int64_t pairs_last;         /* tile/primitive pairs binned by the last render chunk */
} swr_scene_info;

/* Scene + weights load. Replaces train::load_checkpoint (training.hpp:133,
 * checkpoint.cpp:100-146). device < 0 selects the current CUDA device. */
int swr_scene_create_wrfc(const char *path, int device, swr_ctx **out);

/* Host-only read of a WRFC file's header and trailer (no device needed): grid,
 * primitive count, net dims, raster params, bbox and, for an RSSI model saved by
 * tasks::save_rssi_model (tasks.cpp:131-150), its calibration: rssi_cal[0] =
 * slope, rssi_cal[1] = intercept, *has_rssi = 1. Any output may be NULL. */
int swr_wrfc_peek(const char *path, swr_scene_info *info, double *rssi_cal, int *has_rssi);

/* Same from raw arrays in the reference layouts (GaussianSetT, splat.hpp:43-56;
 * DeformNetT layers in WRFD order: 8 trunk, head centre/response/atten,
 * row-major [rows x cols], deform.hpp:57-83). layer_w/layer_b may be NULL for
 * a rasterize-only scene. */
int swr_scene_create(int n_elevation, int n_azimuth, int n, const float *center_raw,
                     const float *cholesky, const float *atten_logit, const float *response,
                     int width, int bands_center, int bands_position, const float *const *layer_w,
                     const float *const *layer_b, float cutoff_radius, int tile,
                     const double *bbox_min, const double *bbox_max, int device, swr_ctx **out);

void swr_scene_destroy(swr_ctx *ctx);
int swr_scene_get_info(swr_ctx *ctx, swr_scene_info *info);

/* The scene as loaded, in the reference layouts (host copies kept by the
 * context): GaussianSetT arrays (splat.hpp:43-56; NULL skips a field), deform
 * layer `layer` in WRFD order 0..10 (deform.hpp:57-83; w [rows][cols] row-major,
 * b [rows]; NULL w/b queries the shape only), checkpoint iteration and
 * manifest hash (training.hpp:114-124). What the reference's train::Checkpoint
 * holds by value, so swr.hpp can offer the same members. */
int swr_scene_get_arrays(swr_ctx *ctx, float *center_raw, float *cholesky, float *atten_logit,
                         float *response);
int swr_scene_get_layer(swr_ctx *ctx, int layer, int *rows, int *cols, float *w, float *b);
int swr_scene_get_meta(swr_ctx *ctx, int64_t *iteration, uint64_t *manifest_hash);

/* Options: "mlp_precision" (SWR_MLP_*), "chunk" (positions per device chunk),
 * "copy_chunk" (swr_render with host spectra: positions per chunk and per raster /
 * D2H slice, default 256 -- each chunk's copy runs under the next chunk's MLP),
 * "async_pair_budget" (bytes of bin buffers a chunk may size to the scene's pair
 * bound without a host read of the pair count; -1 = min(24 GiB, memory / 4)),
 * "rssi_slope" / "rssi_intercept" (affine RSSI calibration, tasks.cpp:60-94; read
 * from the trailer of an RSSI model, load_rssi_model tasks.cpp:139-150; SWR_OUT_RSSI
 * fails with SWR_ERUNTIME while the scene has none, as load_rssi_model does),
 * "stage_timing" (1: record per-stage CUDA events), "stage_reset" (zero the
 * accumulated stage times). */
int swr_set_option(swr_ctx *ctx, const char *key, double value);
/* Current value of an option (the keys above except "stage_reset"). The default
 * "chunk" depends on the scene: ~12.8M (Gaussian, position) rows, 256..1024. */
int swr_get_option(swr_ctx *ctx, const char *key, double *value);

/* Batched render_at (training.cpp:189-195) + heads, host buffers, synchronous.
 * pos_m: [B][3] metres. Any output may be NULL when its flag is off.
 * aoa_rc: [B][2] (row, col); aoa_ang: [B][2] (elevation, azimuth) radians. */
int swr_render(swr_ctx *ctx, const float *pos_m, int64_t B, uint32_t flags, float *spectra,
               double *pooled, double *rssi_dbm, int32_t *aoa_rc, double *aoa_ang);

/* Same with device pointers, stream-ordered on `stream` (a cudaStream_t;
 * NULL = the context's stream). No host synchronisation: the bin buffers are
 * sized to the scene's pair bound (any residuals) and an fp16 overflow re-runs a
 * chunk's MLP in FP32 through device-gated kernels (scenes whose bound exceeds
 * min(24 GiB, memory / 4) per chunk read the pair count back instead).
 * Capturable into a CUDA graph (cudaStreamBeginCapture on `stream`) once an
 * uncaptured call with the same or a larger B has sized the work buffers; the
 * graph's replays then re-read d_pos_m and rewrite the outputs in place. Replays
 * share the context's work buffers, so the caller orders them against other calls
 * on the same context (same stream, or events). The other entry points that take
 * a stream synchronise with the host and refuse a capturing one (SWR_EINVAL). */
int swr_render_device(swr_ctx *ctx, const float *d_pos_m, int64_t B, uint32_t flags,
                      float *d_spectra, double *d_pooled, double *d_rssi, int32_t *d_aoa_rc,
                      double *d_aoa_ang, void *stream);

/* ---- multi-GPU (csrc/group.cpp) ------------------------------
 * Positions split contiguously (B / P per device, the first B % P one more: shard.py's
 * shard_range), the scene and weights
 * replicated on every device, no inter-device dependency while rendering, one
 * gather of the outputs. */
typedef struct swr_group swr_group;
/* one context per device from the same WRFC file (devices[0] is the root) */
int swr_group_create_wrfc(const char *path, const int *devices, int n_dev, swr_group **out);
/* over existing contexts (borrowed: they outlive the group; ctxs[0] is the root) */
int swr_group_create(swr_ctx *const *ctxs, int n, swr_group **out);
void swr_group_destroy(swr_group *g);
int swr_group_size(swr_group *g, int *n);
int swr_group_context(swr_group *g, int i, swr_ctx **out); /* options per member */
/* host buffers: every device renders its shard into its slice (one host thread each) */
int swr_group_render(swr_group *g, const float *pos_m, int64_t B, uint32_t flags, float *spectra,
                     double *pooled, double *rssi_dbm, int32_t *aoa_rc, double *aoa_ang);
/* device buffers on the root, stream-ordered on `stream` (root device): positions
 * scattered peer to peer, each shard rendered chunk by chunk, each chunk sent to the
 * root as it completes (NCCL ncclSend/ncclRecv, one communicator per device; peer
 * copies when a device is listed twice), overlapping the next chunk's rendering */
int swr_group_render_device(swr_group *g, const float *d_pos_m, int64_t B, uint32_t flags, float *d_spectra,
                            double *d_pooled, double *d_rssi, int32_t *d_aoa_rc, double *d_aoa_ang,
                            void *stream);
/* between processes (one process per GPU): rank 0 makes an ncclUniqueId (128 bytes)
 * and shares it; each rank builds a communicator over its context */
typedef struct swr_comm swr_comm;
int swr_nccl_unique_id(void *id128);
int swr_comm_create(swr_ctx *ctx, const void *id128, int nranks, int rank, swr_comm **out);
void swr_comm_destroy(swr_comm *comm);
/* every rank renders its counts[rank] positions (d_pos on its device, shards in rank
 * order); rank 0 receives all spectra into d_spec_root [sum counts][H][W][2] chunk by
 * chunk (its own shard rendered in place) and its own pooled magnitudes into
 * d_pooled_root (may be NULL). flags: SWR_OUT_SPECTRA and/or SWR_OUT_POOLED. */
int swr_render_gather(swr_comm *comm, const float *d_pos_m, const int64_t *counts, uint32_t flags,
                      float *d_spec_root, double *d_pooled_root, void *stream);

/* ---- per-stage parity hooks (host buffers, synchronous) ---------------- */

/* normalize_position (training.cpp:178-187): pos01 [B][3] */
int swr_normalize_positions(swr_ctx *ctx, const float *pos_m, int64_t B, float *pos01);

/* deform::predict_residuals (deform.cpp:140-207) for B normalized positions.
 * Outputs in the reference ResidualsT layouts, one block per position:
 * d_center [B][n][2], d_response [B][n][2], d_atten [B][n]. */
int swr_predict_residuals(swr_ctx *ctx, const float *pos01, int64_t B, float *d_center,
                          float *d_response, float *d_atten);

/* prepare() per-primitive setup (splat.cpp:159-249) with caller residuals
 * (NULL = zero residuals, i.e. rasterize(set, nullptr)). state [B][n][11] in
 * the order of splat.cpp:133-147; rows/cols [B][n][2]; tile_count [B][n]. */
int swr_setup(swr_ctx *ctx, const float *d_center, const float *d_response, const float *d_atten,
              int64_t B, float *state, int32_t *rows, int32_t *cols, int32_t *tile_count);

/* CSR tile bins (splat.cpp:251-292) per position: tile_offset [B][tiles+1]
 * (relative to the position's first pair), tile_prims concatenated over
 * positions (capacity cap entries), total in *n_pairs. */
int swr_bin(swr_ctx *ctx, const float *d_center, const float *d_response, const float *d_atten,
            int64_t B, int32_t *tile_offset, int32_t *tile_prims, int64_t cap, int64_t *n_pairs);

/* splat::rasterize (splat.cpp:312-482) with caller residuals (NULL = none):
 * spectra [B][H][W][2]. */
int swr_rasterize(swr_ctx *ctx, const float *d_center, const float *d_response,
                  const float *d_atten, int64_t B, float *spectra);

/* Heads on caller spectra [B][H][W][2] (tasks.cpp:32-39, 154-169). */
int swr_heads(swr_ctx *ctx, const float *spectra, int64_t B, double *pooled, int32_t *aoa_rc,
              double *aoa_ang);

/* Evaluation metrics of predicted against target spectra, both [B][H][W][2] on
 * the context's grid: PSNR in dB (clamped at 100, spectrum.cpp:145-161), SSIM
 * (11x11 Gaussian window, per channel, averaged, spectrum.cpp:177-250), L1 mean
 * absolute difference (spectrum.cpp:163-172); all statistics in double. Any
 * output may be NULL (skips that metric). peak = the reference's `peak`
 * argument (1.0 in train::evaluate). Replaces wrfsplat::psnr / ssim / l1.
 * SWR_EDOMAIN on a non-finite value, SWR_EINVAL when the grid is below 11x11
 * and SSIM is requested. Host buffers, synchronous: */
int swr_metrics(swr_ctx *ctx, const float *pred, const float *target, int64_t B, double peak,
                double *psnr, double *ssim, double *l1);
/* same on device pointers (outputs too), ordered on `stream` (a cudaStream_t,
 * NULL = the context's stream); returns after the work completes */
int swr_metrics_device(swr_ctx *ctx, const float *d_pred, const float *d_target, int64_t B,
                       double peak, double *d_psnr, double *d_ssim, double *d_l1, void *stream);
/* train::evaluate (training.cpp:380-406) batched: render each TX position
 * (metres, [B][3]) and score it against target[b] ([B][H][W][2], host); the
 * spectra stay on the device, only the metrics come back. */
int swr_evaluate(swr_ctx *ctx, const float *pos_m, const float *target, int64_t B, double peak,
                 double *psnr, double *ssim, double *l1);

/* ------------------------------------------------------------ datasets
 * Reader of the reference's dataset directory (manifest.json + spectra.bin,
 * wavesim.hpp:159-163; load_dataset, dataset.cpp:205-258): validates the
 * manifest and the file size like load_dataset (SWR_ERUNTIME otherwise) and
 * serves records by sample index without loading the whole file. Host only
 * (no device needed). */
typedef struct swr_dataset swr_dataset;
typedef struct
{
    int n_elevation, n_azimuth;
    int64_t samples, n_train, n_test, n_excluded;
    uint64_t manifest_hash; /* FNV-1a 64 of the manifest bytes (common.cpp:40-48) */
    double normalization;
    double bbox_min[3], bbox_max[3];
} swr_dataset_info;
int swr_dataset_open(const char *dir, swr_dataset **out);
void swr_dataset_close(swr_dataset *ds);
int swr_dataset_get_info(swr_dataset *ds, swr_dataset_info *info);
/* split: 0 train, 1 test, 2 all (training.cpp:145-160); indices may be NULL (count only) */
int swr_dataset_split(swr_dataset *ds, int split, int32_t *indices, int64_t *count);
/* records by index (NULL indices = the first `count`): pos [count][3], spectra [count][H][W][2] */
int swr_dataset_read(swr_dataset *ds, const int32_t *indices, int64_t count, float *pos, float *spectra);
/* The full manifest of a dataset (wavesim.hpp:125-139 Dataset minus the samples;
 * manifest_json, dataset.cpp:159-181). Arrays point into storage owned by the
 * swr_dataset they came from (valid while it is open) or by the caller. */
typedef struct
{
    int32_t n_elevation, n_azimuth;
    const char *mode; /* "tx_moving" | "rx_moving" (wavesim.cpp:62-74) */
    int32_t k_elements;
    double spacing, wavelength;
    double room[3];
    double reflectivity;
    int32_t max_bounces;
    double fixed_node[3];
    double normalization;
    uint64_t seed;
    const int32_t *train_indices, *test_indices, *excluded_indices;
    int64_t n_train, n_test, n_excluded;
    double bbox_min[3], bbox_max[3];
    const double *rssi_dbm;
    int64_t n_rssi;
} swr_dataset_meta;
int swr_dataset_get_meta(swr_dataset *ds, swr_dataset_meta *meta);
/* manifest_json (dataset.cpp:159-181) for `sample_count` records: the exact bytes the
 * reference writes (nlohmann::json dump(2) + newline). len receives the size (the
 * buffer may be NULL to query it); hash = FNV-1a 64 of those bytes. */
int swr_dataset_manifest_json(const swr_dataset_meta *meta, int64_t sample_count, char *buf, size_t cap,
                              size_t *len, uint64_t *hash);
/* Writer of the same directory layout (save_dataset, dataset.cpp:183-203): records are
 * streamed to spectra.bin as they come (host buffers or rendered on the GPU) and
 * manifest.json is written at close with sample_count = records written. */
typedef struct swr_dataset_writer swr_dataset_writer;
int swr_dataset_writer_open(const char *dir, int32_t n_elevation, int32_t n_azimuth, swr_dataset_writer **out);
/* pos [count][3] (metres), spectra [count][H][W][2], host memory */
int swr_dataset_writer_append(swr_dataset_writer *w, const float *pos, const float *spectra, int64_t count);
/* render the spectra of pos_m [count][3] on ctx's device (render_at, batched) and
 * append them; the file write of one chunk overlaps the rendering of the next */
int swr_dataset_writer_render(swr_dataset_writer *w, swr_ctx *ctx, const float *pos_m, int64_t count);
/* writes manifest.json (meta's grid must match the writer's) and closes; w is freed
 * even on error. manifest_hash may be NULL. */
int swr_dataset_writer_close(swr_dataset_writer *w, const swr_dataset_meta *meta, uint64_t *manifest_hash);
/* save_dataset in one call (host records) */
int swr_dataset_save(const char *dir, const swr_dataset_meta *meta, const float *pos, const float *spectra,
                     int64_t count, uint64_t *manifest_hash);
/* train::evaluate (training.cpp:380-406): render every sample of the split and
 * score it against its stored spectrum (peak 1). sample_ids / metrics are
 * [split size]. SWR_ERUNTIME if the checkpoint's manifest_hash differs from the
 * dataset's (train::hash_mismatch). */
int swr_evaluate_dataset(swr_ctx *ctx, swr_dataset *ds, int split, int32_t *sample_ids, double *psnr,
                         double *ssim, double *l1);
/* the dataset fingerprint of a scene built from arrays (swr_scene_create_wrfc reads it
 * from the checkpoint trailer, checkpoint.cpp:133) */
int swr_scene_set_manifest_hash(swr_ctx *ctx, uint64_t hash);

/* ------------------------------------------------------------ backward
 * splat::rasterize_backward (splat.cpp:494-669) per position: residuals as for
 * swr_rasterize (NULL = canonical render), upstream = dL/dA [B][H][W][2];
 * outputs in the reference's RenderGrads layout (splat.hpp:77-89), [B][n][2|3|1]:
 * center_raw, cholesky, atten_logit, response (raw fields, chain rule applied)
 * and d_center, d_response, d_atten (wrt the residuals). Any output may be NULL. */
int swr_rasterize_backward(swr_ctx *ctx, const float *d_center, const float *d_response,
                           const float *d_atten, int64_t B, const float *upstream, float *g_center_raw,
                           float *g_cholesky, float *g_atten_logit, float *g_response, float *g_d_center,
                           float *g_d_response, float *g_d_atten);
/* train::hybrid_loss (training.cpp:62-106): lambda1 * L1 + (1 - lambda1) * (1 - SSIM)
 * per (prediction, target) pair; terms [B][3] = (loss, l1_term, ssim_term),
 * grad [B][H][W][2] = dLoss/dprediction (NULL: value only). */
int swr_hybrid_loss(swr_ctx *ctx, const float *pred, const float *target, int64_t B, double lambda1,
                    double *terms, float *grad);

/* ------------------------------------------------------------ training
 * train::train (training.cpp:198-376) on the device: the coarse stage (Gaussians
 * only) then the fine stage (deform net + Gaussians, centres frozen), one
 * training sample per iteration drawn with the reference's Rng stream
 * (mt19937_64; init_random and DeformNet::init draw orders, splat.cpp:681-709,
 * deform.cpp:73-102), Adam per field group (training.cpp:39-57), hybrid loss
 * (training.cpp:62-106), rasterize_backward and deform_backward
 * (deform.cpp:264-326) as CUDA kernels. FP32 like the reference. */
typedef struct
{
    int32_t primitives;       /* Gaussian count (TrainConfig, training.hpp:96-112) */
    int32_t bands_center;     /* encoding bands (10) */
    int32_t bands_position;   /* (6) */
    int32_t width;            /* deform-net hidden width (156; <= 160 here) */
    float cutoff_radius;      /* raster cutoff (3) */
    int32_t tile;             /* raster tile edge (16) */
    double lr_gaussian;       /* 1e-2 */
    double lr_mlp;            /* 8e-3 */
    double lambda1;           /* L1 weight of the hybrid loss (0.7) */
    int64_t coarse_iters;     /* 10000 */
    int64_t fine_iters;       /* 100000 */
    double anneal_scale;      /* coordinate-noise gamma (1) */
    int64_t anneal_threshold; /* coordinate-noise tau (10000) */
    uint64_t seed;            /* 1234 */
} swr_train_config;

typedef struct swr_trainer swr_trainer;

/* The reference defaults (training.hpp:96-112). */
void swr_train_config_default(swr_train_config *cfg);
/* Fresh run (resume_wrfc NULL: init_random + net init from cfg.seed) or resume
 * from a checkpoint written with the same config on the same dataset
 * (SWR_EINVAL on a config mismatch, SWR_ERUNTIME on a manifest-hash mismatch,
 * training.cpp:212-219). The dataset's samples are copied to the device; ds may
 * be closed afterwards. */
int swr_trainer_create(const swr_train_config *cfg, swr_dataset *ds, const char *resume_wrfc, int device,
                       swr_trainer **out);
void swr_trainer_destroy(swr_trainer *tr);
/* Run up to max_iters further iterations of the schedule (stops at
 * coarse_iters + fine_iters). log [done][3] = (loss, l1_term, ssim_term) per
 * iteration (the reference's CSV columns), NULL to skip; *done = iterations run;
 * *device_ms = device time of the run. SWR_ERUNTIME on a non-finite loss. */
int swr_trainer_run(swr_trainer *tr, int64_t max_iters, double *log, int64_t *done, double *device_ms);
/* Completed iterations (Checkpoint::iteration). */
int64_t swr_trainer_iteration(swr_trainer *tr);
/* Current parameters in the reference layouts; layer_w/b in layer_list order
 * (8 trunk layers, head_center, head_response, head_atten); any NULL skipped. */
int swr_trainer_params(swr_trainer *tr, float *center_raw, float *cholesky, float *atten_logit, float *response,
                       float *const layer_w[11], float *const layer_b[11]);
/* One training forward/backward at the current parameters, no optimizer step:
 * pos01 (normalized, 3 floats) != NULL runs the fine-stage chain
 * (predict_residuals -> rasterize -> hybrid_loss -> rasterize_backward ->
 * deform_backward, training.cpp:332-345), NULL the coarse one (no residuals);
 * the target is dataset sample `sample`. terms = (loss, l1_term, ssim_term);
 * render_grads = the 7 RenderGrads fields [n][w]; layer_gw/gb = DeformGrads in
 * layer_list order (fine only). Any output may be NULL. */
int swr_trainer_gradients(swr_trainer *tr, const float *pos01, int32_t sample, double *terms,
                          float *const render_grads[7], float *const layer_gw[11], float *const layer_gb[11]);
/* train::save_checkpoint (checkpoint.cpp:50-93): WRFC with the config echo,
 * iteration, manifest hash and bbox. */
int swr_trainer_save(swr_trainer *tr, const char *path);

/* ------------------------------------------------------------ beam scan
 * The synthetic-data generator's steering step (sim::build_steering_table,
 * sim::beam_scan, wavesim.cpp:183-252) batched over samples on the GPU, and
 * generate_dataset's target post-processing (dataset.cpp:86-124). The steering
 * table [cells][K] is built once per (array, grid). Arrays: square, K <= 64. */
typedef struct swr_steering swr_steering;
int swr_steering_create(int32_t k_elements, double spacing, double wavelength, int32_t H, int32_t W, int device,
                        swr_steering **out);
void swr_steering_destroy(swr_steering *st);
/* The table (build_steering_table layout: wr/wi [H*W][K], row-major per cell). */
int swr_steering_table(swr_steering *st, double *wr, double *wi);
/* beam_scan for B channels h [B][K][2] (complex double) -> spectra [B][H][W][2]
 * (complex double), bit-identical to the reference without FP contraction. */
int swr_beam_scan(swr_steering *st, const double *channel, int64_t B, double *spectra);
/* Device variant: d_unit = phase-only channels u = h/|h| [B][K][2] already on the
 * device, d_spectra [B][H][W][2] double, ordered on `stream` (a cudaStream_t;
 * NULL = the handle's stream). */
int swr_beam_scan_device(swr_steering *st, const double *d_unit, int64_t B, double *d_spectra, void *stream);
/* Dataset targets for B valid samples: float(|A| / max|A|) with a zero imaginary
 * channel, [B][H][W][2] float; *normalization = max|A| (1 when all zero). */
int swr_beam_scan_targets(swr_steering *st, const double *channel, int64_t B, float *targets, double *normalization);

/* Kernel launches issued by this context since creation (for the bench). */
int64_t swr_launch_count(swr_ctx *ctx);

/* Device time (ms) of the render stages, summed over every chunk rendered while
 * option "stage_timing" is 1 since the last "stage_reset":
 * [0] position prep, [1] MLP, [2] setup, [3] bin (scan+emit+sort), [4] raster, [5] heads.
 * Events are read here (no host sync inside the renders). */
int swr_stage_times(swr_ctx *ctx, double *ms6);

const char *swr_last_error(void);
int swr_version(void);

#ifdef __cplusplus
}
#endif
#endif
