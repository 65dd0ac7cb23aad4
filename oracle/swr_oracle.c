/* Plain-C restatement of the SwiftWRF render path. TEST INFRASTRUCTURE ONLY —
 * see swr_oracle.h. Compiled with -ffp-contract=off so every float operation is
 * the single IEEE operation written here (the GPU kernels use the same
 * explicitly-rounded sequences, so state, bins and cutoff masks compare
 * bit-for-bit). References are to /root/reference/proj. */
#include "swr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define SO_PI 3.141592653589793238462643383279502884
static const float kCholFloor = 1e-4f; /* splat.hpp:36 */

enum { S_EL, S_AZ, S_I00, S_I01, S_I11, S_DELTA, S_RE, S_IM, S_INVL1, S_INVL3, S_L2, S_STRIDE };

static inline float fmaxr(float a, float b) { return (a < b) ? b : a; } /* std::max */
static inline float fminr(float a, float b) { return (b < a) ? b : a; } /* std::min */

/* splat.cpp:60-65 */
void so_materialize_center(float raw_el, float raw_az, float *el, float *az)
{
    *el = (float)(SO_PI / 4) * (tanhf(raw_el) + 1.0f);
    *az = (float)SO_PI * (tanhf(raw_az) + 1.0f);
}

/* deform.cpp:54-70: [v | sin(f_0 v) | cos(f_0 v) | ... ], f_k = float(2^k pi) */
void so_encode(const float *values, int count, int bands, float *out)
{
    float *dst = out;
    for (int i = 0; i < count; i++)
        *dst++ = values[i];
    for (int k = 0; k < bands; k++)
    {
        const float f = (float)ldexp(SO_PI, k);
        for (int i = 0; i < count; i++)
            *dst++ = sinf(f * values[i]);
        for (int i = 0; i < count; i++)
            *dst++ = cosf(f * values[i]);
    }
}

/* training.cpp:178-187 */
void so_normalize_position(const double bmin[3], const double bmax[3], const float pos[3], float out[3])
{
    for (int a = 0; a < 3; a++)
    {
        const double range = bmax[a] - bmin[a];
        out[a] = range > 0.0 ? (float)(((double)pos[a] - bmin[a]) / range) : 0.5f;
    }
}

/* ---------------------------------------------------------------- deform MLP */

/* One dense layer for one row, y = W x + b (deform.cpp:126-137 semantics; the
 * sum runs in column order, then the bias is added as Eigen's y += b does). */
static void dense_f(const float *w, const float *b, int rows, int cols, const float *x, float *y, int relu)
{
    for (int r = 0; r < rows; r++)
    {
        float acc = 0.0f;
        const float *wr = w + (size_t)r * cols;
        for (int c = 0; c < cols; c++)
            acc += wr[c] * x[c];
        acc += b[r];
        y[r] = relu ? (acc > 0.0f ? acc : 0.0f) : acc;
    }
}

static void dense_d(const float *w, const float *b, int rows, int cols, const double *x, double *y, int relu)
{
    for (int r = 0; r < rows; r++)
    {
        double acc = 0.0;
        const float *wr = w + (size_t)r * cols;
        for (int c = 0; c < cols; c++)
            acc += (double)wr[c] * x[c];
        acc += (double)b[r];
        y[r] = relu ? (acc > 0.0 ? acc : 0.0) : acc;
    }
}

/* deform.cpp:140-207: row p = [encode(center_p) | encode(pos)], 8 ReLU trunk
 * layers, encoding re-concatenated at 0-based layers 2/4/6 (deform.cpp:41),
 * heads 2/2/1. Straight-line per row, like test_deform.cpp:34-62. */
int so_predict(const so_net *net, const so_set *set, const float pos01[3], int precise,
               float *d_center, float *d_response, float *d_atten)
{
    const int Wd = net->width;
    const int Dc = 2 * (2 * net->bands_c + 1), Dp = 3 * (2 * net->bands_p + 1), D = Dc + Dp;
    if (set->n < 1 || Wd < 1)
        return 1;
    float *penc = (float *)malloc(sizeof(float) * (size_t)Dp);
    so_encode(pos01, 3, net->bands_p, penc);
    int bad = 0;
#pragma omp parallel
    {
        float *xf = (float *)malloc(sizeof(float) * (size_t)(D + Wd));
        float *hf = (float *)malloc(sizeof(float) * (size_t)(D + Wd));
        float *yf = (float *)malloc(sizeof(float) * (size_t)Wd);
        double *xd = (double *)malloc(sizeof(double) * (size_t)(D + Wd));
        double *hd = (double *)malloc(sizeof(double) * (size_t)(D + Wd));
        double *yd = (double *)malloc(sizeof(double) * (size_t)Wd);
        if (!xf || !hf || !yf || !xd || !hd || !yd)
            bad = 1;
#pragma omp for schedule(static)
        for (int p = 0; p < set->n; p++)
        {
            if (bad)
                continue;
            float ang[2];
            so_materialize_center(set->center_raw[2 * (size_t)p], set->center_raw[2 * (size_t)p + 1], &ang[0], &ang[1]);
            so_encode(ang, 2, net->bands_c, xf);
            memcpy(xf + Dc, penc, sizeof(float) * (size_t)Dp);
            float out[5];
            if (!precise)
            {
                /* layer 0 reads x; skip layers read [h, x] */
                dense_f(net->w[0], net->b[0], Wd, D, xf, yf, 1);
                for (int l = 1; l < 8; l++)
                {
                    const int skip = (l == 2 || l == 4 || l == 6);
                    memcpy(hf, yf, sizeof(float) * (size_t)Wd);
                    if (skip)
                        memcpy(hf + Wd, xf, sizeof(float) * (size_t)D);
                    dense_f(net->w[l], net->b[l], Wd, skip ? Wd + D : Wd, hf, yf, 1);
                }
                dense_f(net->w[8], net->b[8], 2, Wd, yf, out, 0);
                dense_f(net->w[9], net->b[9], 2, Wd, yf, out + 2, 0);
                dense_f(net->w[10], net->b[10], 1, Wd, yf, out + 4, 0);
            }
            else
            {
                double o[5];
                for (int k = 0; k < D; k++)
                    xd[k] = xf[k];
                dense_d(net->w[0], net->b[0], Wd, D, xd, yd, 1);
                for (int l = 1; l < 8; l++)
                {
                    const int skip = (l == 2 || l == 4 || l == 6);
                    memcpy(hd, yd, sizeof(double) * (size_t)Wd);
                    if (skip)
                        memcpy(hd + Wd, xd, sizeof(double) * (size_t)D);
                    dense_d(net->w[l], net->b[l], Wd, skip ? Wd + D : Wd, hd, yd, 1);
                }
                dense_d(net->w[8], net->b[8], 2, Wd, yd, o, 0);
                dense_d(net->w[9], net->b[9], 2, Wd, yd, o + 2, 0);
                dense_d(net->w[10], net->b[10], 1, Wd, yd, o + 4, 0);
                for (int k = 0; k < 5; k++)
                    out[k] = (float)o[k];
            }
            d_center[2 * (size_t)p] = out[0];
            d_center[2 * (size_t)p + 1] = out[1];
            d_response[2 * (size_t)p] = out[2];
            d_response[2 * (size_t)p + 1] = out[3];
            d_atten[p] = out[4];
        }
        free(xf);
        free(hf);
        free(yf);
        free(xd);
        free(hd);
        free(yd);
    }
    free(penc);
    return bad ? 2 : 0;
}

/* ------------------------------------------------------ setup + tile binning */

/* splat.cpp:94-118: deformed, clamp-applied parameters */
static void deform_prim(const so_set *s, const float *dc, const float *dr, const float *da, int p, float pr[9])
{
    float el, az;
    so_materialize_center(s->center_raw[2 * (size_t)p], s->center_raw[2 * (size_t)p + 1], &el, &az);
    float l1 = fmaxr(s->cholesky[3 * (size_t)p], kCholFloor);
    float l2 = s->cholesky[3 * (size_t)p + 1];
    float l3 = fmaxr(s->cholesky[3 * (size_t)p + 2], kCholFloor);
    float delta = 1.0f / (1.0f + expf(-s->atten_logit[p]));
    float re = s->response[2 * (size_t)p], im = s->response[2 * (size_t)p + 1];
    if (dc)
    {
        el += dc[2 * (size_t)p];
        az += dc[2 * (size_t)p + 1];
        re += dr[2 * (size_t)p];
        im += dr[2 * (size_t)p + 1];
        delta = fminr(fmaxr(delta + da[p], 0.0f), 1.0f);
    }
    pr[0] = el; pr[1] = az; pr[2] = l1; pr[3] = l2; pr[4] = l3; pr[5] = delta; pr[6] = re; pr[7] = im;
}

typedef struct { int tile, th, tw; } layout_t;

/* splat.cpp:255-282: tiles of one primitive; the wrapped column interval
 * splits into at most two linear spans, the second deduped against the first */
static int visit_tiles(const layout_t *L, int W, const int *rows, const int *cols, int *out)
{
    if (rows[1] < rows[0])
        return 0;
    int k = 0;
    const int tr0 = rows[0] / L->tile, tr1 = rows[1] / L->tile;
    const int j0 = cols[0], len = cols[1];
    if (len >= W)
    {
        for (int tc = 0; tc < L->tw; tc++)
            for (int tr = tr0; tr <= tr1; tr++)
                out[k++] = tr * L->tw + tc;
        return k;
    }
    const int jend = j0 + len - 1;
    const int e0 = (jend < W - 1 ? jend : W - 1) / L->tile;
    for (int tc = j0 / L->tile; tc <= e0; tc++)
        for (int tr = tr0; tr <= tr1; tr++)
            out[k++] = tr * L->tw + tc;
    if (jend >= W)
    {
        const int a = (jend - W) / L->tile, b = j0 / L->tile - 1;
        const int e1 = a < b ? a : b;
        for (int tc = 0; tc <= e1; tc++)
            for (int tr = tr0; tr <= tr1; tr++)
                out[k++] = tr * L->tw + tc;
    }
    return k;
}

int64_t so_prepare(const so_set *s, const float *dc, const float *dr, const float *da, float cutoff,
                   int tile, float *state, int *rows, int *cols, int *tile_offset, int *tile_prims, int64_t cap)
{
    layout_t L;
    L.tile = tile < 1 ? 16 : tile;
    L.th = (s->H + L.tile - 1) / L.tile;
    L.tw = (s->W + L.tile - 1) / L.tile;
    const int tiles = L.th * L.tw;
    const int cut = cutoff > 0.0f;
    const float radius = cut ? cutoff : 0.0f;
    const double cell_el = (SO_PI / 2.0) / s->H, cell_az = (2.0 * SO_PI) / s->W;

    memset(state, 0, sizeof(float) * (size_t)s->n * S_STRIDE);
    memset(cols, 0, sizeof(int) * (size_t)s->n * 2);
    /* splat.cpp:187-249 */
    for (int p = 0; p < s->n; p++)
    {
        float pr[9];
        deform_prim(s, dc, dr, da, p, pr);
        const float el = pr[0], az = pr[1], l1 = pr[2], l2 = pr[3], l3 = pr[4], delta = pr[5];
        float *st = state + (size_t)p * S_STRIDE;
        int *rw = rows + 2 * (size_t)p, *cl = cols + 2 * (size_t)p;
        rw[0] = 0;
        rw[1] = -1;
        if (delta <= 0.0f)
            continue;
        const float det = l1 * l1 * l3 * l3;
        st[S_EL] = el;
        st[S_AZ] = az;
        st[S_I00] = (l2 * l2 + l3 * l3) / det;
        st[S_I01] = -l2 / (l1 * l3 * l3);
        st[S_I11] = 1.0f / (l3 * l3);
        st[S_DELTA] = delta;
        st[S_RE] = pr[6];
        st[S_IM] = pr[7];
        st[S_INVL1] = 1.0f / l1;
        st[S_INVL3] = 1.0f / l3;
        st[S_L2] = l2;
        if (!cut)
        {
            rw[0] = 0;
            rw[1] = s->H - 1;
            cl[0] = 0;
            cl[1] = s->W;
            continue;
        }
        const double h_el = (double)radius * (double)l1;
        const double h_az = (double)radius * sqrt((double)l2 * l2 + (double)l3 * l3);
        int r0 = (int)floor(((double)el - h_el) / cell_el - 0.5);
        int r1 = (int)ceil(((double)el + h_el) / cell_el - 0.5);
        if (r0 < 0) r0 = 0;
        if (r1 > s->H - 1) r1 = s->H - 1;
        if (r0 > r1)
            continue;
        rw[0] = r0;
        rw[1] = r1;
        if (2.0 * h_az >= (double)s->W * cell_az)
        {
            cl[0] = 0;
            cl[1] = s->W;
        }
        else
        {
            int j0 = (int)floor(((double)az - h_az) / cell_az - 0.5);
            int j1 = (int)ceil(((double)az + h_az) / cell_az - 0.5);
            int len = j1 - j0 + 1;
            if (len > s->W) len = s->W;
            j0 = ((j0 % s->W) + s->W) % s->W;
            cl[0] = j0;
            cl[1] = len;
        }
    }
    /* splat.cpp:251-292: count, exclusive prefix, fill in primitive order */
    int *buf = (int *)malloc(sizeof(int) * (size_t)tiles);
    memset(tile_offset, 0, sizeof(int) * (size_t)(tiles + 1));
    for (int p = 0; p < s->n; p++)
    {
        const int k = visit_tiles(&L, s->W, rows + 2 * (size_t)p, cols + 2 * (size_t)p, buf);
        for (int i = 0; i < k; i++)
            tile_offset[buf[i] + 1]++;
    }
    for (int t = 0; t < tiles; t++)
        tile_offset[t + 1] += tile_offset[t];
    const int64_t total = tile_offset[tiles];
    int *cursor = (int *)malloc(sizeof(int) * (size_t)tiles);
    memcpy(cursor, tile_offset, sizeof(int) * (size_t)tiles);
    for (int p = 0; p < s->n; p++)
    {
        const int k = visit_tiles(&L, s->W, rows + 2 * (size_t)p, cols + 2 * (size_t)p, buf);
        for (int i = 0; i < k; i++)
        {
            const int pos = cursor[buf[i]]++;
            if (tile_prims && pos < cap)
                tile_prims[pos] = p;
        }
    }
    free(cursor);
    free(buf);
    return total;
}

/* splat.cpp:72-82 */
static inline float wrap_pm_pi(float x)
{
    if (x < (float)(-8 * SO_PI) || x > (float)(8 * SO_PI))
        x = fmodf(x, (float)(2 * SO_PI));
    while (x >= (float)SO_PI)
        x -= (float)(2 * SO_PI);
    while (x < (float)(-SO_PI))
        x += (float)(2 * SO_PI);
    return x;
}

/* splat.cpp:312-482. The reference evaluates exp(-Q/2) through a factored
 * row recurrence when its `worst < 160` gate allows (splat.cpp:382-426) and
 * exactly otherwise (:429-447); both mask on the same float q. This
 * restatement always takes the exact branch. */
int so_rasterize(const so_set *s, const float *dc, const float *dr, const float *da, float cutoff,
                 int tile, int precise, float *spectrum)
{
    const int n = s->n, H = s->H, W = s->W;
    layout_t L;
    L.tile = tile < 1 ? 16 : tile;
    L.th = (H + L.tile - 1) / L.tile;
    L.tw = (W + L.tile - 1) / L.tile;
    const int tiles = L.th * L.tw;
    float *state = (float *)malloc(sizeof(float) * (size_t)n * S_STRIDE);
    int *rows = (int *)malloc(sizeof(int) * (size_t)n * 2);
    int *cols = (int *)malloc(sizeof(int) * (size_t)n * 2);
    int *off = (int *)malloc(sizeof(int) * (size_t)(tiles + 1));
    const int64_t pairs = so_prepare(s, dc, dr, da, cutoff, tile, state, rows, cols, off, NULL, 0);
    int *prims = (int *)malloc(sizeof(int) * (size_t)(pairs > 0 ? pairs : 1));
    so_prepare(s, dc, dr, da, cutoff, tile, state, rows, cols, off, prims, pairs);

    float *el_c = (float *)malloc(sizeof(float) * (size_t)H);
    float *az_c = (float *)malloc(sizeof(float) * (size_t)W);
    const double cel = (SO_PI / 2.0) / H, caz = (2.0 * SO_PI) / W;
    for (int r = 0; r < H; r++)
        el_c[r] = (float)((r + 0.5) * cel);
    for (int j = 0; j < W; j++)
        az_c[j] = (float)((j + 0.5) * caz);
    const int cut = cutoff > 0.0f;
    const float cut2 = cut ? cutoff * cutoff : INFINITY;
    double *acc = (double *)calloc((size_t)H * W * 2, sizeof(double));
    float *accf = (float *)calloc((size_t)H * W * 2, sizeof(float));

#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < tiles; t++)
    {
        const int tr = t / L.tw, tc = t % L.tw;
        const int r0 = tr * L.tile, r1 = (r0 + L.tile < H ? r0 + L.tile : H) - 1;
        const int c0 = tc * L.tile, c1 = (c0 + L.tile < W ? c0 + L.tile : W) - 1;
        for (int q_i = off[t]; q_i < off[t + 1]; q_i++)
        {
            const int p = prims[q_i];
            const float *st = state + (size_t)p * S_STRIDE;
            const int pr0 = r0 > rows[2 * p] ? r0 : rows[2 * p];
            const int pr1 = r1 < rows[2 * p + 1] ? r1 : rows[2 * p + 1];
            if (pr1 < pr0)
                continue;
            const float i00 = st[S_I00], i01 = st[S_I01], i11 = st[S_I11];
            const float k_re = st[S_RE] * st[S_DELTA], k_im = st[S_IM] * st[S_DELTA];
            const float inv_l1 = st[S_INVL1];
            int seg[2][2], nseg = 0;
            const int j0 = cols[2 * p], len = cols[2 * p + 1];
            if (len >= W)
            {
                seg[0][0] = c0; seg[0][1] = c1; nseg = 1;
            }
            else
            {
                const int jend = j0 + len - 1;
                const int a0 = c0 > j0 ? c0 : j0;
                int b0 = jend < W - 1 ? jend : W - 1;
                if (c1 < b0) b0 = c1;
                if (a0 <= b0) { seg[nseg][0] = a0; seg[nseg][1] = b0; nseg++; }
                if (jend >= W)
                {
                    const int b1 = c1 < jend - W ? c1 : jend - W;
                    if (c0 <= b1) { seg[nseg][0] = c0; seg[nseg][1] = b1; nseg++; }
                }
            }
            for (int sg = 0; sg < nseg; sg++)
                for (int r = pr0; r <= pr1; r++)
                {
                    const float d_el = el_c[r] - st[S_EL];
                    const float u0 = d_el * inv_l1;
                    if (u0 * u0 > cut2)
                        continue;
                    const float q_c = i00 * d_el * d_el;
                    for (int j = seg[sg][0]; j <= seg[sg][1]; j++)
                    {
                        const float d_az = wrap_pm_pi(az_c[j] - st[S_AZ]);
                        const float w1 = i11 * d_az * d_az;
                        const float w2 = 2.0f * i01 * d_az;
                        const float q = q_c + d_el * w2 + w1;
                        if (!(q <= cut2))
                            continue;
                        const size_t c = (size_t)r * W + j;
                        if (precise)
                        {
                            const double e = exp(-0.5 * (double)q);
                            acc[2 * c] += (double)k_re * e;
                            acc[2 * c + 1] += (double)k_im * e;
                        }
                        else
                        {
                            const float e = expf(-0.5f * q);
                            accf[2 * c] += k_re * e;
                            accf[2 * c + 1] += k_im * e;
                        }
                    }
                }
        }
    }
    for (size_t c = 0; c < (size_t)H * W * 2; c++)
        spectrum[c] = precise ? (float)acc[c] : accf[c];
    free(acc);
    free(accf);
    free(el_c);
    free(az_c);
    free(prims);
    free(off);
    free(cols);
    free(rows);
    free(state);
    return 0;
}

/* spectrum.cpp:136-143 */
void so_magnitude(const float *spectrum, int cells, float *out)
{
    for (int k = 0; k < cells; k++)
        out[k] = (float)hypot((double)spectrum[2 * (size_t)k], (double)spectrum[2 * (size_t)k + 1]);
}

/* tasks.cpp:154-169: strict > keeps the first maximum in row-major order */
int so_aoa(const float *spectrum, int H, int W, int *row, int *col, double *el, double *az)
{
    const int cells = H * W;
    int best = 0;
    float bv = (float)hypot((double)spectrum[0], (double)spectrum[1]);
    for (int k = 1; k < cells; k++)
    {
        const float m = (float)hypot((double)spectrum[2 * (size_t)k], (double)spectrum[2 * (size_t)k + 1]);
        if (m > bv)
        {
            bv = m;
            best = k;
        }
    }
    *row = best / W;
    *col = best % W;
    *el = (*row + 0.5) * ((SO_PI / 2.0) / H);
    *az = (*col + 0.5) * ((2.0 * SO_PI) / W);
    return best;
}

/* tasks.cpp:32-39: mean of float magnitudes, summed in double */
double so_pooled(const float *spectrum, int cells)
{
    double sum = 0.0;
    for (int k = 0; k < cells; k++)
        sum += (float)hypot((double)spectrum[2 * (size_t)k], (double)spectrum[2 * (size_t)k + 1]);
    return sum / (double)cells;
}

/* ------------------------------------------------------------------ metrics
 * spectrum.cpp:145-250: psnr / l1 over all 2*H*W floats in double; SSIM per
 * channel (re, im) with an 11x11 Gaussian window (sigma 1.5, unit sum,
 * spectrum.cpp:51-70), valid-region separable correlation (spectrum.cpp:72-101),
 * statistics in double, mean over windows, average of the two channels.
 * Returns 0, or 1 for a non-finite input (the reference throws domain_error,
 * spectrum.cpp:44-49), 2 for a grid smaller than the window (invalid_argument). */
#define SO_WIN 11

static void so_window_taps(double g[SO_WIN])
{
    double sum = 0.0;
    for (int i = 0; i < SO_WIN; i++)
    {
        const double d = i - SO_WIN / 2;
        g[i] = exp(-0.5 * d * d / (1.5 * 1.5));
        sum += g[i];
    }
    for (int i = 0; i < SO_WIN; i++)
        g[i] /= sum;
}

/* spectrum.cpp:72-101 (src H x W -> dst (H-10) x (W-10)) */
static void so_conv_valid(const double *src, int h, int w, double *tmp, double *dst, const double *g)
{
    const int vw = w - SO_WIN + 1, vh = h - SO_WIN + 1;
    for (size_t k = 0; k < (size_t)h * vw; k++)
        tmp[k] = 0.0;
    for (int i = 0; i < h; i++)
        for (int t = 0; t < SO_WIN; t++)
            for (int j = 0; j < vw; j++)
                tmp[(size_t)i * vw + j] += g[t] * src[(size_t)i * w + j + t];
    for (int i = 0; i < vh; i++)
    {
        double *out = dst + (size_t)i * vw;
        for (int j = 0; j < vw; j++)
            out[j] = 0.0;
        for (int t = 0; t < SO_WIN; t++)
            for (int j = 0; j < vw; j++)
                out[j] += g[t] * tmp[(size_t)(i + t) * vw + j];
    }
}

/* spectrum.cpp:177-238 without the gradient */
static double so_ssim_channel(const float *x, const float *y, int h, int w, int c, double peak)
{
    const int vh = h - SO_WIN + 1, vw = w - SO_WIN + 1;
    const size_t cells = (size_t)h * w, wins = (size_t)vh * vw;
    const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
    double g[SO_WIN];
    so_window_taps(g);
    double *xs = malloc(sizeof(double) * cells), *ys = malloc(sizeof(double) * cells);
    double *prod = malloc(sizeof(double) * cells), *tmp = malloc(sizeof(double) * (size_t)h * vw);
    double *mx = malloc(sizeof(double) * wins), *my = malloc(sizeof(double) * wins);
    double *sxx = malloc(sizeof(double) * wins), *syy = malloc(sizeof(double) * wins);
    double *sxy = malloc(sizeof(double) * wins);
    for (size_t k = 0; k < cells; k++)
    {
        xs[k] = (double)x[2 * k + c];
        ys[k] = (double)y[2 * k + c];
    }
    so_conv_valid(xs, h, w, tmp, mx, g);
    so_conv_valid(ys, h, w, tmp, my, g);
    for (size_t k = 0; k < cells; k++)
        prod[k] = xs[k] * xs[k];
    so_conv_valid(prod, h, w, tmp, sxx, g);
    for (size_t k = 0; k < cells; k++)
        prod[k] = ys[k] * ys[k];
    so_conv_valid(prod, h, w, tmp, syy, g);
    for (size_t k = 0; k < cells; k++)
        prod[k] = xs[k] * ys[k];
    so_conv_valid(prod, h, w, tmp, sxy, g);
    double total = 0.0;
    for (size_t k = 0; k < wins; k++)
    {
        const double ux = mx[k], uy = my[k];
        const double vx = sxx[k] - ux * ux, vy = syy[k] - uy * uy, vxy = sxy[k] - ux * uy;
        const double a1 = 2.0 * ux * uy + c1, a2 = 2.0 * vxy + c2;
        const double b1 = ux * ux + uy * uy + c1, b2 = vx + vy + c2;
        total += (a1 * a2) / (b1 * b2);
    }
    free(xs), free(ys), free(prod), free(tmp), free(mx), free(my), free(sxx), free(syy), free(sxy);
    return total / (double)wins;
}

int so_metrics(const float *a, const float *b, int H, int W, double peak, double *psnr, double *ssim, double *l1)
{
    const size_t n = (size_t)2 * H * W;
    for (size_t k = 0; k < n; k++)
        if (!isfinite((double)a[k]) || !isfinite((double)b[k]))
            return 1;
    double mse = 0.0, sad = 0.0;
    for (size_t k = 0; k < n; k++)
    {
        const double d = (double)a[k] - (double)b[k];
        mse += d * d;
        sad += fabs((double)a[k] - (double)b[k]);
    }
    mse /= (double)n;
    if (psnr)
        *psnr = mse <= 0.0 ? 100.0 : fmin(100.0, 10.0 * log10(peak * peak / mse)); /* spectrum.cpp:145-161 */
    if (l1)
        *l1 = sad / (double)n; /* spectrum.cpp:163-172 */
    if (ssim)
    {
        if (H < SO_WIN || W < SO_WIN)
            return 2;
        *ssim = 0.5 * (so_ssim_channel(a, b, H, W, 0, peak) + so_ssim_channel(a, b, H, W, 1, peak));
    }
    return 0;
}
