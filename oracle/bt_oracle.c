/*
 * bt_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * THIS IS THE CHECKER, NOT THE PRODUCT.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` leg may load it.  The
 * product path (paper_2208_14228_b200/) never links, imports or calls it.
 *
 * It restates, in plain C with binary64 arithmetic and NO floating-point
 * contraction (built with -ffp-contract=off, see oracle/Makefile), the pure-
 * Python reference package `bittrain` 0.1.0 under /root/reference/pkg/src:
 *
 *   prng.py       mix64/splitmix64/unit_float/derive_stream/fnv1a64/
 *                 shuffled_range                         (prng.py:27-93)
 *   reduction.py  reduce_sum Sequential / Tree(f)        (reduction.py:39-62)
 *   model.py      init_random, forward_backward,
 *                 TrackedStat.updated, sgd_step          (model.py:58-213)
 *   buckets.py    build_buckets_initial, rebuild, _pack,
 *                 layout_arrival_perm, allreduce         (buckets.py:47-124)
 *   sampling.py   make_dataset, epoch_indices, worker_rng,
 *                 DataPipeline._produce (jitter)         (sampling.py:24-172)
 *   engine.py     assign_ranks, init_training, run_minibatch (incl. the d0
 *                 bucket rebuild), split_by_rank         (engine.py:169-329)
 *   checkpoint.py restore semantics used by apply_layout (checkpoint.py:204-238)
 *
 * tanh: the reference calls math.tanh (model.py:148) == the host libm tanh;
 * this oracle calls the same libm tanh, so on the same box it is bit-exact
 * with the reference (pinned by the JSON files in tests/golden/, generated from the
 * reference itself by tests/golden/gen_golden.py).
 *
 * Parity is PINNED: tests/test_golden_oracle.py checks every function here
 * against the golden vectors captured from the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>

#define OR_INPUT_DIM 8
#define OR_HIDDEN 16
#define OR_W1 0
#define OR_B1 (OR_INPUT_DIM * OR_HIDDEN)
#define OR_W2 (OR_B1 + OR_HIDDEN)
#define OR_B2 (OR_W2 + OR_HIDDEN)
#define OR_P (OR_B2 + 1) /* 161, model.py:34 */

enum { OR_OK = 0, OR_INPUT = 1, OR_CONFIG = 2, OR_STATE = 3, OR_PROGRESS = 4, OR_NUMERIC = 5,
       OR_CORRUPTION = 6 };

static const uint64_t GAMMA = 0x9E3779B97F4A7C15ull; /* prng.py:14 */
static const uint64_t TAG_DATASET = 0xD5A61C0FFEE5EED5ull;      /* prng.py:20 */
static const uint64_t TAG_MODEL_INIT = 0x1417E5EED0D0CAFEull;   /* prng.py:21 */
static const uint64_t TAG_DROPOUT = 0xD80F0D7A6B15EA5Eull;      /* prng.py:22 */
static const uint64_t TAG_DATA_WORKER = 0xB07C9E11A7756E1Dull;  /* prng.py:23 */
static const uint64_t TAG_BUCKET_ARRIVAL = 0xAC1DB0B5CA77E7E5ull; /* prng.py:24 */

/* ---------------------------------------------------------------- prng.py */
uint64_t or_mix64(uint64_t x) { /* prng.py:27-35 */
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

uint64_t or_splitmix64_next(uint64_t *state) { /* prng.py:38-45 */
    *state += GAMMA;
    return or_mix64(*state);
}

double or_unit_float(uint64_t raw) { return (double)(raw >> 11) * 0x1p-53; } /* prng.py:48-50 */

double or_uniform01(uint64_t *state) { return or_unit_float(or_splitmix64_next(state)); } /* :53-56 */

uint64_t or_derive_stream(const uint64_t *words, int n) { /* prng.py:59-69 */
    uint64_t s = 0x243F6A8885A308D3ull;
    for (int i = 0; i < n; i++) s = or_mix64(s ^ words[i]);
    return s;
}

uint64_t or_fnv1a64(const uint8_t *data, size_t n) { /* prng.py:72-78 */
    uint64_t h = 0xCBF29CE484222325ull;
    for (size_t i = 0; i < n; i++) {
        h ^= data[i];
        h *= 0x100000001B3ull;
    }
    return h;
}

void or_shuffled_range(int n, uint64_t state, int32_t *arr) { /* prng.py:81-93 */
    for (int i = 0; i < n; i++) arr[i] = i;
    for (int t = n - 1; t > 0; t--) {
        uint64_t raw = or_splitmix64_next(&state);
        int k = (int)(raw % (uint64_t)(t + 1));
        int32_t tmp = arr[t];
        arr[t] = arr[k];
        arr[k] = tmp;
    }
}

/* ----------------------------------------------------------- reduction.py */
/* fanin 0 == Sequential.  Tree(f): bottom-up, children folded left to right,
 * each group folded from its FIRST element (no 0.0 seed) -- reduction.py:39-62. */
double or_reduce_sum(const double *values, int n, int fanin) {
    if (n == 0) return 0.0;
    if (fanin == 0) {
        double acc = values[0];
        for (int i = 1; i < n; i++) acc += values[i];
        return acc;
    }
    double buf[64]; /* small: large stack frames pay stack-clash probes on every call */
    double *lvl = buf;
    double *heap = NULL;
    if (n > 64) lvl = heap = (double *)malloc(sizeof(double) * (size_t)n);
    memcpy(lvl, values, sizeof(double) * (size_t)n);
    int len = n;
    while (len > 1) {
        int out = 0;
        for (int i = 0; i < len; i += fanin) {
            int hi = i + fanin < len ? i + fanin : len;
            double acc = lvl[i];
            for (int k = i + 1; k < hi; k++) acc += lvl[k];
            lvl[out++] = acc;
        }
        len = out;
    }
    double r = lvl[0];
    free(heap);
    return r;
}

/* --------------------------------------------------------------- model.py */
void or_init_random(uint64_t seed, double scale, double *out) { /* model.py:58-66 */
    uint64_t w[2] = {TAG_MODEL_INIT, seed};
    uint64_t s = or_derive_stream(w, 2);
    for (int i = 0; i < OR_P; i++) {
        double u = or_uniform01(&s);
        out[i] = (u * 2.0 - 1.0) * scale;
    }
}

/* forward_backward (model.py:107-196); x is [B][8] row-major, y is [B]. */
int or_forward_backward(const double *v, const double *x, const double *y, int nrows, int64_t rank,
                        uint64_t rng, double stat_mean, uint64_t stat_count, int fanin, double rate,
                        double *loss_out, double *grads, uint64_t *rng_out, double *stat_mean_out,
                        uint64_t *stat_count_out) {
    if (nrows <= 0) return OR_INPUT;
    if (nrows > 256) return OR_INPUT;
    double acts[nrows][OR_HIDDEN], masks[nrows][OR_HIDDEN], hid[nrows][OR_HIDDEN]; /* VLAs sized to the batch */
    double dz[nrows][OR_HIDDEN], errs[nrows], gy[nrows], col[nrows > OR_HIDDEN ? nrows : OR_HIDDEN];
    const int d = OR_INPUT_DIM, h = OR_HIDDEN;
    for (int r = 0; r < nrows; r++) {
        const double *xr = x + (size_t)r * d;
        for (int j = 0; j < h; j++) {
            double acc = v[OR_W1 + j] * xr[0];
            for (int i = 1; i < d; i++) acc += v[OR_W1 + i * h + j] * xr[i];
            acts[r][j] = tanh(acc + v[OR_B1 + j]);
        }
    }
    double keep_scale = rate >= 1.0 ? 0.0 : 1.0 / (1.0 - rate);
    for (int r = 0; r < nrows; r++)
        for (int j = 0; j < h; j++) {
            if (rate > 0.0) {
                double u = or_uniform01(&rng);
                masks[r][j] = u < rate ? 0.0 : keep_scale;
            } else {
                masks[r][j] = 1.0;
            }
        }
    for (int r = 0; r < nrows; r++)
        for (int j = 0; j < h; j++) hid[r][j] = acts[r][j] * masks[r][j];
    for (int r = 0; r < nrows; r++) {
        double acc = v[OR_W2] * hid[r][0];
        for (int j = 1; j < h; j++) acc += v[OR_W2 + j] * hid[r][j];
        errs[r] = acc + v[OR_B2] - y[r];
    }
    for (int r = 0; r < nrows; r++) col[r] = errs[r] * errs[r];
    *loss_out = or_reduce_sum(col, nrows, fanin) / nrows;
    for (int r = 0; r < nrows; r++) gy[r] = 2.0 * errs[r] / nrows;
    for (int r = 0; r < nrows; r++)
        for (int j = 0; j < h; j++)
            dz[r][j] = gy[r] * v[OR_W2 + j] * masks[r][j] * (1.0 - acts[r][j] * acts[r][j]);
    for (int i = 0; i < d; i++)
        for (int j = 0; j < h; j++) {
            for (int r = 0; r < nrows; r++) col[r] = dz[r][j] * x[(size_t)r * d + i];
            grads[OR_W1 + i * h + j] = or_reduce_sum(col, nrows, fanin);
        }
    for (int j = 0; j < h; j++) {
        for (int r = 0; r < nrows; r++) col[r] = dz[r][j];
        grads[OR_B1 + j] = or_reduce_sum(col, nrows, fanin);
    }
    for (int j = 0; j < h; j++) {
        for (int r = 0; r < nrows; r++) col[r] = gy[r] * hid[r][j];
        grads[OR_W2 + j] = or_reduce_sum(col, nrows, fanin);
    }
    grads[OR_B2] = or_reduce_sum(gy, nrows, fanin);
    /* TrackedStat (model.py:99-104, 194-196): plain sequential means. */
    for (int r = 0; r < nrows; r++) col[r] = or_reduce_sum(acts[r], h, 0) / h;
    double batch_mean = or_reduce_sum(col, nrows, 0) / nrows;
    double mixed = batch_mean + (double)rank * 0x1p-40;
    *stat_mean_out = stat_mean * 0.9 + 0.1 * mixed;
    *stat_count_out = stat_count + 1;
    *rng_out = rng;
    return OR_OK;
}

/* sgd_step (model.py:199-213).  Returns OR_NUMERIC and the index via *bad. */
int or_sgd_step(const double *params, const double *vel, const double *grads, int n, double lr,
                double mu, double *params_out, double *vel_out, int *bad) {
    for (int p = 0; p < n; p++)
        if (!isfinite(grads[p])) {
            if (bad) *bad = p;
            return OR_NUMERIC;
        }
    for (int p = 0; p < n; p++) {
        double v = mu * vel[p] + grads[p];
        vel_out[p] = v;
        params_out[p] = params[p] - lr * v;
    }
    return OR_OK;
}

/* ------------------------------------------------------------- buckets.py */
/* A bucket map is (nbuckets, sizes[nb], flat indices[P]). */
void or_build_buckets_initial(int nparams, int capacity, int *nb, int32_t *sizes, int32_t *idx) {
    for (int i = 0; i < nparams; i++) idx[i] = nparams - 1 - i; /* buckets.py:47-53 */
    int b = 0;
    for (int i = 0; i < nparams; i += capacity, b++) sizes[b] = (nparams - i) < capacity ? nparams - i : capacity;
    *nb = b;
}

void or_pack(const int32_t *order, int nparams, int capacity, int *nb, int32_t *sizes, int32_t *idx) {
    memcpy(idx, order, sizeof(int32_t) * (size_t)nparams); /* buckets.py:63-67 */
    int b = 0;
    for (int i = 0; i < nparams; i += capacity, b++) sizes[b] = (nparams - i) < capacity ? nparams - i : capacity;
    *nb = b;
}

/* layout_key: nexec pairs (fnv1a64(kind utf-8), threads)  (buckets.py:70-82) */
void or_layout_arrival_perm(int nparams, int nexec, const uint64_t *kind_fnv, const int64_t *threads,
                            int32_t *perm) {
    uint64_t words[2 + 2 * 64];
    int nw = 0;
    words[nw++] = TAG_BUCKET_ARRIVAL;
    words[nw++] = (uint64_t)nexec;
    for (int e = 0; e < nexec; e++) {
        words[nw++] = kind_fnv[e];
        words[nw++] = (uint64_t)threads[e];
    }
    or_shuffled_range(nparams, or_derive_stream(words, nw), perm);
}

/* allreduce (buckets.py:85-124); replicas is [nrep][nparams] by ascending rank. */
int or_allreduce(const double *replicas, int nrep, int nparams, int nb, const int32_t *sizes,
                 const int32_t *idx, int fanin, double *out) {
    if (nrep < 1) return OR_INPUT;
    int covered = 0;
    for (int b = 0; b < nb; b++) covered += sizes[b];
    if (covered != nparams) return OR_INPUT;
    double *contrib = (double *)malloc(sizeof(double) * (size_t)nrep);
    int base = 0;
    for (int b = 0; b < nb; b++) {
        int blen = sizes[b];
        for (int pos = 0; pos < blen; pos++) {
            int p = idx[base + pos];
            if (fanin == 0) {
                for (int k = 0; k < nrep; k++) contrib[k] = replicas[(size_t)k * nparams + p];
            } else {
                int start = (int)(((int64_t)pos * nrep) / blen);
                for (int k = 0; k < nrep; k++) contrib[k] = replicas[(size_t)((start + k) % nrep) * nparams + p];
            }
            out[p] = or_reduce_sum(contrib, nrep, fanin) / nrep;
        }
        base += blen;
    }
    free(contrib);
    return OR_OK;
}

/* ------------------------------------------------------------ sampling.py */
void or_make_dataset(uint64_t seed, int n, int dim, double *out) { /* sampling.py:24-35 */
    uint64_t w[2] = {TAG_DATASET, seed};
    uint64_t s = or_derive_stream(w, 2);
    for (int r = 0; r < n; r++) {
        for (int i = 0; i <= dim; i++) out[(size_t)r * (dim + 1) + i] = or_uniform01(&s) * 2.0 - 1.0;
    }
}

uint64_t or_worker_rng(uint64_t seed, uint64_t epoch, uint64_t local, uint64_t worker) { /* :99-101 */
    uint64_t w[5] = {TAG_DATA_WORKER, seed, epoch, local, worker};
    return or_derive_stream(w, 5);
}

/* epoch_indices (sampling.py:63-82): out is [workers][per_worker], per_worker = spe*micro. */
int or_epoch_indices(uint64_t seed, uint64_t epoch, int n, int workers, int micro, int shuffle, int32_t *out) {
    if (workers < 1 || n < workers) return OR_CONFIG;
    int spe = n / (workers * micro);
    if (spe < 1) return OR_CONFIG;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (shuffle) or_shuffled_range(n, seed ^ epoch, order);
    else for (int i = 0; i < n; i++) order[i] = i;
    int per = spe * micro;
    for (int k = 0; k < workers; k++)
        for (int t = 0; t < per; t++) out[(size_t)k * per + t] = order[(size_t)t * workers + k];
    free(order);
    return OR_OK;
}

/* -------------------------------------------------------------- engine.py */
#define OR_MAX_EXEC 64
typedef struct {
    uint64_t seed;
    int max_workers, micro_batch, dataset_size;
    double lr, momentum, dropout_rate, jitter;
    int bucket_capacity, d0, d1, d2, shuffle;
} or_cfg;

typedef struct {
    int nexec;
    int fanin[OR_MAX_EXEC];     /* executor kernel profile: 0 = Sequential (d2), else Tree(f) */
    uint64_t kind_fnv[OR_MAX_EXEC];
    int first[OR_MAX_EXEC], count[OR_MAX_EXEC];
} or_layout;

typedef struct {
    or_cfg cfg;
    or_layout lay;
    double params[OR_P], vel[OR_P];
    uint64_t *rng, *stat_count;
    double *stat_mean;
    double *dataset;
    int32_t *lists; /* cached [workers][per] lists for cached_epoch */
    int64_t cached_epoch;
    int nb;
    int32_t bsizes[OR_P], bidx[OR_P];
    int rebuild_pending;
    int64_t global_step, epoch;
    int spe;
    double *grads; /* [E][P] */
    /* worker pool (bench cpu baseline / reference arm only) */
    int nthreads;
    struct or_pool *pool;
} or_run;

/* assign_ranks (engine.py:169-199).  threads may be NULL (balanced, larger shares first). */
int or_assign(or_layout *lay, int nexec, const int64_t *threads, int max_workers) {
    if (nexec < 1 || nexec > OR_MAX_EXEC) return OR_CONFIG;
    int counts[OR_MAX_EXEC];
    if (threads) {
        int64_t s = 0;
        for (int e = 0; e < nexec; e++) {
            if (threads[e] < 1) return OR_CONFIG;
            s += threads[e];
            counts[e] = (int)threads[e];
        }
        if (s != max_workers) return OR_CONFIG;
    } else {
        if (nexec > max_workers) return OR_CONFIG;
        int base = max_workers / nexec, extra = max_workers % nexec;
        for (int e = 0; e < nexec; e++) counts[e] = base + (e < extra ? 1 : 0);
    }
    int cur = 0;
    lay->nexec = nexec;
    for (int e = 0; e < nexec; e++) {
        lay->first[e] = cur;
        lay->count[e] = counts[e];
        cur += counts[e];
    }
    return OR_OK;
}

static void or_lists_for_epoch(or_run *R, int64_t epoch) {
    if (R->cached_epoch == epoch) return;
    or_epoch_indices(R->cfg.seed, (uint64_t)epoch, R->cfg.dataset_size, R->cfg.max_workers,
                     R->cfg.micro_batch, R->cfg.shuffle, R->lists);
    R->cached_epoch = epoch;
}

/* Micro-batch rows of (step, worker) per DataPipeline._produce (sampling.py:160-172). */
void or_pipeline_rows(or_run *R, int64_t step, int worker, double *x, double *y) {
    const int B = R->cfg.micro_batch;
    int64_t epoch = step / R->spe, local = step % R->spe;
    or_lists_for_epoch(R, epoch);
    int per = R->spe * B;
    const int32_t *idxs = R->lists + (size_t)worker * per + (size_t)local * B;
    uint64_t rng = or_worker_rng(R->cfg.seed, (uint64_t)epoch, (uint64_t)local, (uint64_t)worker);
    for (int r = 0; r < B; r++) {
        const double *row = R->dataset + (size_t)idxs[r] * (OR_INPUT_DIM + 1);
        if (R->cfg.jitter != 0.0) {
            double u = or_uniform01(&rng);
            for (int i = 0; i < OR_INPUT_DIM; i++) x[r * OR_INPUT_DIM + i] = row[i] + (u - 0.5) * R->cfg.jitter;
        } else {
            for (int i = 0; i < OR_INPUT_DIM; i++) x[r * OR_INPUT_DIM + i] = row[i];
        }
        y[r] = row[OR_INPUT_DIM];
    }
}

/* init_training (engine.py:202-243). kind_fnv/fanins per executor; fanin ignored under d2. */
or_run *or_run_create(const or_cfg *cfg, int nexec, const uint64_t *kind_fnv, const int32_t *fanins,
                      const int64_t *threads) {
    or_run *R = (or_run *)calloc(1, sizeof(or_run));
    R->cfg = *cfg;
    const int E = cfg->max_workers;
    if (or_assign(&R->lay, nexec, threads, E) != OR_OK) { free(R); return NULL; }
    for (int e = 0; e < nexec; e++) {
        R->lay.fanin[e] = cfg->d2 ? 0 : fanins[e];
        R->lay.kind_fnv[e] = kind_fnv[e];
    }
    or_init_random(cfg->seed, 0.5, R->params);
    memset(R->vel, 0, sizeof R->vel);
    R->rng = (uint64_t *)calloc((size_t)E, 8);
    R->stat_count = (uint64_t *)calloc((size_t)E, 8);
    R->stat_mean = (double *)calloc((size_t)E, 8);
    for (int k = 0; k < E; k++) {
        uint64_t w[3] = {TAG_DROPOUT, cfg->seed, (uint64_t)k};
        R->rng[k] = or_derive_stream(w, 3);
    }
    R->dataset = (double *)malloc(sizeof(double) * (size_t)cfg->dataset_size * (OR_INPUT_DIM + 1));
    or_make_dataset(cfg->seed, cfg->dataset_size, OR_INPUT_DIM, R->dataset);
    R->spe = cfg->dataset_size / (E * cfg->micro_batch);
    if (R->spe < 1) { free(R); return NULL; }
    R->lists = (int32_t *)malloc(sizeof(int32_t) * (size_t)R->spe * cfg->micro_batch * E);
    R->cached_epoch = -1;
    or_build_buckets_initial(OR_P, cfg->bucket_capacity, &R->nb, R->bsizes, R->bidx);
    R->rebuild_pending = !cfg->d1;
    R->grads = (double *)malloc(sizeof(double) * (size_t)E * OR_P);
    return R;
}

static void or_pool_stop(or_run *R);
void or_run_free(or_run *R) {
    if (!R) return;
    or_pool_stop(R);
    free(R->rng); free(R->stat_count); free(R->stat_mean); free(R->dataset); free(R->lists); free(R->grads);
    free(R);
}

/* apply_layout == checkpoint_save + checkpoint_restore (engine.py:332-336, checkpoint.py:204-238):
 * contexts/params/opt unchanged; ESTs redistributed contiguously; bucket map kept iff d1,
 * otherwise reset to the initial map with the arrival-order rebuild pending again. */
int or_run_relayout(or_run *R, int nexec, const uint64_t *kind_fnv, const int32_t *fanins, const int64_t *threads) {
    or_layout lay;
    int st = or_assign(&lay, nexec, threads, R->cfg.max_workers);
    if (st) return st;
    for (int e = 0; e < nexec; e++) {
        lay.fanin[e] = R->cfg.d2 ? 0 : fanins[e];
        lay.kind_fnv[e] = kind_fnv[e];
    }
    R->lay = lay;
    if (!R->cfg.d1) {
        or_build_buckets_initial(OR_P, R->cfg.bucket_capacity, &R->nb, R->bsizes, R->bidx);
        R->rebuild_pending = 1;
    }
    return OR_OK;
}

static int or_fanin_of_rank(const or_run *R, int rank) {
    for (int e = 0; e < R->lay.nexec; e++)
        if (rank >= R->lay.first[e] && rank < R->lay.first[e] + R->lay.count[e]) return R->lay.fanin[e];
    return 0;
}

/* ---- optional worker pool: ESTs are independent inside a step, so the
 * bench's CPU baseline fans forward_backward out over host threads (results
 * are identical: each EST writes only its own slots). ---- */
typedef struct {
    or_run *R;
    const double *gx, *gy; /* explicit global batch or NULL */
    double *losses;
    int lo, hi;
    int status;
} or_job;

static void or_est_range(or_job *J) {
    or_run *R = J->R;
    const int B = R->cfg.micro_batch, E = R->cfg.max_workers;
    double x[R->cfg.micro_batch * OR_INPUT_DIM], y[R->cfg.micro_batch];
    for (int k = J->lo; k < J->hi; k++) {
        if (J->gx) {
            for (int r = 0; r < B; r++) { /* split_by_rank: rows t::E (engine.py:261-268) */
                memcpy(x + r * OR_INPUT_DIM, J->gx + (size_t)(r * E + k) * OR_INPUT_DIM, sizeof(double) * OR_INPUT_DIM);
                y[r] = J->gy[(size_t)r * E + k];
            }
        } else {
            or_pipeline_rows(R, R->global_step, k, x, y);
        }
        uint64_t rng2, cnt2;
        double mean2;
        int st = or_forward_backward(R->params, x, y, B, k, R->rng[k], R->stat_mean[k], R->stat_count[k],
                                     or_fanin_of_rank(R, k), R->cfg.dropout_rate, &J->losses[k],
                                     R->grads + (size_t)k * OR_P, &rng2, &mean2, &cnt2);
        if (st) { J->status = st; return; }
        R->rng[k] = rng2;
        R->stat_mean[k] = mean2;
        R->stat_count[k] = cnt2;
    }
}

static void *or_thread_main(void *arg) {
    or_est_range((or_job *)arg);
    return NULL;
}

/* Persistent spinning workers (the per-step cost of pthread_create would exceed a mini-batch's
 * work): the main thread publishes a generation, each worker runs its EST range and counts in. */
typedef struct or_pool {
    int n; /* workers besides the main thread */
    pthread_t th[64];
    or_job jobs[64];
    atomic_int gen, done, quit;
    struct or_worker { struct or_pool *pool; int id; } w[64];
} or_pool;

static inline void or_relax(void) {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}

static void *or_pool_main(void *arg) {
    struct or_worker *w = (struct or_worker *)arg;
    or_pool *P = w->pool;
    int seen = 0;
    for (;;) {
        int g;
        while ((g = atomic_load(&P->gen)) == seen && !atomic_load(&P->quit)) or_relax();
        if (atomic_load(&P->quit)) return NULL;
        seen = g;
        or_est_range(&P->jobs[w->id]);
        atomic_fetch_add(&P->done, 1);
    }
}

static void or_pool_stop(or_run *R) {
    or_pool *P = R->pool;
    if (!P) return;
    atomic_store(&P->quit, 1);
    for (int t = 1; t <= P->n; t++) pthread_join(P->th[t], NULL);
    free(P);
    R->pool = NULL;
}

static void or_pool_start(or_run *R, int n) {
    or_pool_stop(R);
    if (n < 1) return;
    or_pool *P = (or_pool *)calloc(1, sizeof(or_pool));
    P->n = n;
    atomic_init(&P->gen, 0);
    atomic_init(&P->done, 0);
    atomic_init(&P->quit, 0);
    for (int t = 1; t <= n; t++) {
        P->w[t] = (struct or_worker){P, t};
        pthread_create(&P->th[t], NULL, or_pool_main, &P->w[t]);
    }
    R->pool = P;
}

/* run_minibatch (engine.py:271-329).  gx/gy: optional explicit global batch
 * ([E*B][8], [E*B]); losses_out: [E]. */
int or_run_step(or_run *R, const double *gx, const double *gy, double *losses_out) {
    const int E = R->cfg.max_workers;
    if (gx == NULL) { /* pipeline epoch lists must exist before threads read them */
        or_lists_for_epoch(R, R->global_step / R->spe);
    }
    int nt = R->nthreads > 1 ? R->nthreads : 1;
    if (nt > E) nt = E;
    if (nt > 64) nt = 64;
    or_job jobs[64];
    pthread_t th[64];
    or_pool *P = R->pool;
    if (P && P->n + 1 == nt) { /* persistent workers */
        for (int t = 0; t < nt; t++) P->jobs[t] = (or_job){R, gx, gy, losses_out, (E * t) / nt, (E * (t + 1)) / nt, 0};
        atomic_store(&P->done, 0);
        atomic_fetch_add(&P->gen, 1);
        or_est_range(&P->jobs[0]);
        while (atomic_load(&P->done) != P->n) or_relax();
        for (int t = 0; t < nt; t++) jobs[t] = P->jobs[t];
    } else {
        for (int t = 0; t < nt; t++) {
            jobs[t] = (or_job){R, gx, gy, losses_out, (E * t) / nt, (E * (t + 1)) / nt, 0};
        }
        if (nt == 1) {
            or_est_range(&jobs[0]);
        } else {
            for (int t = 1; t < nt; t++) pthread_create(&th[t], NULL, or_thread_main, &jobs[t]);
            or_est_range(&jobs[0]);
            for (int t = 1; t < nt; t++) pthread_join(th[t], NULL);
        }
    }
    for (int t = 0; t < nt; t++) if (jobs[t].status) return jobs[t].status;
    double synced[OR_P], np[OR_P], nv[OR_P];
    int comm_fanin = R->lay.fanin[0]; /* executor 0's profile (engine.py:309) */
    or_allreduce(R->grads, E, OR_P, R->nb, R->bsizes, R->bidx, comm_fanin, synced);
    int bad = -1;
    int st = or_sgd_step(R->params, R->vel, synced, OR_P, R->cfg.lr, R->cfg.momentum, np, nv, &bad);
    if (st) return st;
    memcpy(R->params, np, sizeof np);
    memcpy(R->vel, nv, sizeof nv);
    R->global_step += 1;
    R->epoch = R->global_step / R->spe;
    if (R->rebuild_pending) { /* engine.py:323-328 */
        int32_t perm[OR_P];
        int64_t thr[OR_MAX_EXEC];
        for (int e = 0; e < R->lay.nexec; e++) thr[e] = R->lay.count[e];
        or_layout_arrival_perm(OR_P, R->lay.nexec, R->lay.kind_fnv, thr, perm);
        or_pack(perm, OR_P, R->cfg.bucket_capacity, &R->nb, R->bsizes, R->bidx);
        R->rebuild_pending = 0;
    }
    return OR_OK;
}

void or_run_set_threads(or_run *R, int n) {
    R->nthreads = n;
    const int nt = n > R->cfg.max_workers ? R->cfg.max_workers : n;
    or_pool_start(R, nt > 1 ? (nt > 64 ? 63 : nt - 1) : 0);
}

/* n pipeline-fed steps in C (the bench's reference arm: no per-step interpreter overhead) */
int or_run_steps(or_run *R, int64_t n, double *losses_out) {
    for (int64_t i = 0; i < n; i++) {
        int st = or_run_step(R, NULL, NULL, losses_out);
        if (st) return st;
    }
    return OR_OK;
}

void or_run_get_state(const or_run *R, double *params, double *vel, double *stat_mean, uint64_t *stat_count,
                      uint64_t *rng, int64_t *global_step, int64_t *epoch) {
    const int E = R->cfg.max_workers;
    if (params) memcpy(params, R->params, sizeof R->params);
    if (vel) memcpy(vel, R->vel, sizeof R->vel);
    if (stat_mean) memcpy(stat_mean, R->stat_mean, 8 * (size_t)E);
    if (stat_count) memcpy(stat_count, R->stat_count, 8 * (size_t)E);
    if (rng) memcpy(rng, R->rng, 8 * (size_t)E);
    if (global_step) *global_step = R->global_step;
    if (epoch) *epoch = R->epoch;
}

int or_run_get_buckets(const or_run *R, int32_t *sizes, int32_t *idx) {
    if (sizes) memcpy(sizes, R->bsizes, sizeof(int32_t) * (size_t)R->nb);
    if (idx) memcpy(idx, R->bidx, sizeof R->bidx);
    return R->nb;
}

/* Generic (large-P) reducer restatement for the C5 sweep checker: the
 * reference allreduce + sgd_step composed, on a float32 or float64 buffer, with
 * the per-parameter rotation start precomputed (rot may be NULL = no rotation).
 * Mirrors buckets.py:115-123 (fold order) and model.py:206-212 (update). */
#define OR_REDUCE_UPDATE(T, NAME)                                                                       \
    int NAME(const T *grads, int E, int64_t n, const int32_t *rot, int fanin, const T *params,          \
             const T *vel, T lr, T mu, T *params_out, T *vel_out) {                                     \
        T contrib[1024];                                                                                \
        if (E < 1 || E > 1024) return OR_INPUT;                                                         \
        for (int64_t p = 0; p < n; p++) {                                                               \
            int start = rot ? rot[p] : 0;                                                               \
            for (int k = 0; k < E; k++) contrib[k] = grads[(size_t)((start + k) % E) * (size_t)n + p];  \
            T acc;                                                                                      \
            if (fanin == 0) {                                                                           \
                acc = contrib[0];                                                                       \
                for (int k = 1; k < E; k++) acc += contrib[k];                                          \
            } else {                                                                                    \
                int len = E;                                                                            \
                while (len > 1) {                                                                       \
                    int out = 0;                                                                        \
                    for (int i = 0; i < len; i += fanin) {                                              \
                        int hi = i + fanin < len ? i + fanin : len;                                     \
                        T a = contrib[i];                                                               \
                        for (int k = i + 1; k < hi; k++) a += contrib[k];                               \
                        contrib[out++] = a;                                                             \
                    }                                                                                   \
                    len = out;                                                                          \
                }                                                                                       \
                acc = contrib[0];                                                                       \
            }                                                                                           \
            T g = acc / (T)E;                                                                           \
            if (!isfinite(g)) return OR_NUMERIC;                                                        \
            T v = mu * vel[p] + g;                                                                      \
            vel_out[p] = v;                                                                             \
            params_out[p] = params[p] - lr * v;                                                         \
        }                                                                                               \
        return OR_OK;                                                                                   \
    }
OR_REDUCE_UPDATE(double, or_reduce_update_f64)
OR_REDUCE_UPDATE(float, or_reduce_update_f32)

/* Rank-ordered fold of E f32 buffers for the bench's large-S cpu baseline,
 * split over host threads by parameter range (each element's fold order is
 * unchanged, so threading does not change bits). */
typedef struct {
    const float *grads; int E; int64_t n, lo, hi; const float *params, *vel; float lr, mu;
    float *po, *vo; int st;
} or_red_job;
static void *or_red_main(void *a) {
    or_red_job *J = (or_red_job *)a;
    for (int64_t p = J->lo; p < J->hi; p++) {
        float acc = J->grads[p];
        for (int k = 1; k < J->E; k++) acc += J->grads[(size_t)k * (size_t)J->n + p];
        float g = acc / (float)J->E;
        if (!isfinite(g)) { J->st = OR_NUMERIC; return NULL; }
        float v = J->mu * J->vel[p] + g;
        J->vo[p] = v;
        J->po[p] = J->params[p] - J->lr * v;
    }
    return NULL;
}
int or_reduce_update_seq_f32_mt(const float *grads, int E, int64_t n, const float *params, const float *vel,
                                float lr, float mu, float *po, float *vo, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 64) nthreads = 64;
    or_red_job jobs[64];
    pthread_t th[64];
    for (int t = 0; t < nthreads; t++)
        jobs[t] = (or_red_job){grads, E, n, n * t / nthreads, n * (t + 1) / nthreads, params, vel, lr, mu, po, vo, 0};
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, or_red_main, &jobs[t]);
    or_red_main(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; t++) if (jobs[t].st) return jobs[t].st;
    return OR_OK;
}

/* The reference's math.tanh is this host's libm tanh (model.py:148): a batch
 * form for checking the device tanh on many inputs. */
void or_libm_tanh_array(const double *x, int64_t n, double *out) {
    for (int64_t i = 0; i < n; i++) out[i] = tanh(x[i]);
}
