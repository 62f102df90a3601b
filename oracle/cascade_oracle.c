/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference planner's
 * plan-search hot path, written from the reference's behaviour (file:line
 * citations relative to /root/reference/proj).  It is the checker for the
 * GPU engine in tests/ and smoke(); its own parity is pinned against the
 * compiled, unmodified reference (oracle/_ref) in tests/test_oracle.py.
 * Single-threaded, no FMA contraction (-ffp-contract=off), glibc libm.
 *
 * Return codes: -1 = ok, otherwise the cascade::Errc value
 * (include/cascade/errors.hpp:10-18).
 */
#include "cascade_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OK (-1)
#define E_INVALID 0
#define E_EMPTY 2
#define E_NODEPLOY 3
#define E_INFEASIBLE 4
#define E_INFEASIBLE_PROBLEM 5
#define MAXS 32

/* ---------------- std::mt19937_64 (util.hpp:16-54) */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    uint64_t x;
    if (s->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        for (; i < 311; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[x & 1ULL];
        s->mti = 0;
    }
    x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
static double exponential_mean(mt64* s, double mean) {
    double u = uniform01(s);
    return -mean * log1p(-u);
}

/* ---------------- util (util.cpp:11-29) */
static int cmp_dbl(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) ? -1 : (x > y) ? 1 : 0;
}

static double quantile_sorted(const double* v, int64_t n, double q) {
    double nn = (double)n;
    int64_t rank = (int64_t)ceil(q * nn);
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return v[rank - 1];
}

static double mean_of(const double* v, int64_t n) {
    if (n == 0) return 0.0;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i];
    return s / (double)n;
}

static double overall_rate(const double* arrival, int64_t n) {
    if (n < 2) return 0.0;
    double span = arrival[n - 1] - arrival[0];
    if (span <= 0.0) return 0.0;
    return (double)n / span;
}

/* ---------------- routing (routing.cpp:19-93) */
static void stats_over(const int64_t* idx, int64_t cnt, const double* in_tok, const double* out_col, double rate,
                       double* w) {
    w[0] = rate;
    w[1] = w[2] = w[3] = w[4] = 0.0;
    if (cnt == 0) return;
    double* a = (double*)malloc(sizeof(double) * cnt);
    double* b = (double*)malloc(sizeof(double) * cnt);
    for (int64_t k = 0; k < cnt; ++k) {
        a[k] = in_tok[idx[k]];
        b[k] = out_col[idx[k]];
    }
    w[1] = mean_of(a, cnt);
    w[2] = mean_of(b, cnt);
    qsort(a, cnt, sizeof(double), cmp_dbl);
    qsort(b, cnt, sizeof(double), cmp_dbl);
    w[3] = quantile_sorted(a, cnt, 0.95);
    w[4] = quantile_sorted(b, cnt, 0.95);
    free(a);
    free(b);
}

int co_route(const double* arrival, const double* in_tok, const double* out_tok, const double* scores, int64_t n,
             int c, const double* h, const int* deployed, double* ratios, double* workloads, double* quality,
             int* accept_stage) {
    if (n == 0) return E_EMPTY;
    int last = -1;
    for (int i = c - 1; i >= 0; --i)
        if (deployed[i]) {
            last = i;
            break;
        }
    if (last < 0) return E_NODEPLOY;
    int64_t** reached = (int64_t**)calloc(c, sizeof(int64_t*));
    int64_t* cnt = (int64_t*)calloc(c, sizeof(int64_t));
    for (int i = 0; i < c; ++i) reached[i] = (int64_t*)malloc(sizeof(int64_t) * n);
    double score_sum = 0.0;
    for (int64_t r = 0; r < n; ++r) {
        int accept = last;
        for (int i = 0; i < c; ++i) {
            if (!deployed[i]) continue;
            reached[i][cnt[i]++] = r;
            if (i == last) {
                accept = last;
                break;
            }
            if (scores[(int64_t)i * n + r] >= h[i]) {
                accept = i;
                break;
            }
        }
        score_sum += scores[(int64_t)accept * n + r];
        if (accept_stage) accept_stage[r] = accept + 1;
    }
    const double nn = (double)n;
    const double rate = overall_rate(arrival, n);
    for (int i = 0; i < c; ++i) {
        ratios[i] = (double)cnt[i] / nn;
        stats_over(reached[i], cnt[i], in_tok, out_tok + (int64_t)i * n, rate * ratios[i], workloads + 5 * i);
        free(reached[i]);
    }
    free(reached);
    free(cnt);
    *quality = score_sum / nn;
    return OK;
}

/* ---------------- cost model (costmodel.cpp:79-414) */
static int mem_feasible(int tp, int pp, const co_model* m, const co_hw* hw, const co_params* p, double kv_tokens) {
    const double gpus = tp * pp;
    const double weights = m->param_count * m->bytes_per_param;
    if (weights / gpus > hw->mem_cap) return 0;
    const double kv_budget = p->kv_frac * (gpus * hw->mem_cap - weights);
    return kv_budget >= m->kv_bytes_per_token * kv_tokens;
}

static int legal_shapes(const co_model* m, const co_hw* hw, const co_params* p, int* tp, int* pp) {
    int ct[64], cp[64], k = 0;
    for (int t = 1; t <= hw->gpus_per_node && k < 64; t *= 2)
        for (int q = 1; q <= 8; ++q) {
            ct[k] = t;
            cp[k] = q;
            ++k;
        }
    /* canonical order: gpus desc, tp desc (insertion sort, unique keys) */
    for (int i = 1; i < k; ++i) {
        int a = ct[i], b = cp[i], j = i - 1;
        while (j >= 0 && (ct[j] * cp[j] < a * b || (ct[j] * cp[j] == a * b && ct[j] < a))) {
            ct[j + 1] = ct[j];
            cp[j + 1] = cp[j];
            --j;
        }
        ct[j + 1] = a;
        cp[j + 1] = b;
    }
    int s = 0;
    for (int i = 0; i < k; ++i)
        if (mem_feasible(ct[i], cp[i], m, hw, p, 1.0) && s < MAXS) {
            tp[s] = ct[i];
            pp[s] = cp[i];
            ++s;
        }
    return s;
}

typedef struct {
    int S, N, n_req;
    int tp[MAXS], pp[MAXS];
    char ok[MAXS];
    double prefill[MAXS], decode[MAXS], ms[MAXS];
    double rate;
    const double *arr, *outs;
    double* fifo;   /* [dp][n_req] */
    int64_t *head, *size;
    double *avail, *soj;
    int* rep_shape;
    double* best_lat;   /* [N+1] */
    int* best_counts;   /* [(N+1)*MAXS] */
    char* has_best;
    int64_t* best_idx;  /* [N+1] enumeration index of the best plan */
    int64_t counter, lo, hi;  /* plan-index shard [lo, hi) */
} rowctx;

static int parts_less(const int* A, const int* B, int S) {
    for (int s = 0; s < S; ++s) {
        if (A[s] == B[s]) continue;
        if (A[s] > 0 && B[s] > 0) return A[s] < B[s];
        if (A[s] == 0) {
            for (int t = s + 1; t < S; ++t)
                if (A[t]) return 0;
            return 1;
        }
        for (int t = s + 1; t < S; ++t)
            if (B[t]) return 1;
        return 0;
    }
    return 0;
}

/* simulate_plan_p95 (costmodel.cpp:248-292) */
static double simulate(rowctx* x, int dp) {
    const int64_t n = x->n_req;
    for (int j = 0; j < dp; ++j) {
        x->avail[j] = 0.0;
        x->head[j] = 0;
        x->size[j] = 0;
    }
    for (int64_t k = 0; k < n; ++k) {
        const double t = x->arr[k];
        int best = 0;
        int64_t best_len = INT64_MAX;
        for (int j = 0; j < dp; ++j) {
            double* q = x->fifo + (int64_t)j * n;
            int64_t h = x->head[j];
            while (h < x->size[j] && q[h] <= t) ++h;
            x->head[j] = h;
            const int64_t len = x->size[j] - h;
            if (len < best_len) {
                best_len = len;
                best = j;
                if (len == 0) break;
            }
        }
        const int s = x->rep_shape[best];
        const double start = (t < x->avail[best]) ? x->avail[best] : t;
        const double fin = start + x->prefill[s] + x->outs[k] * x->decode[s];
        x->avail[best] = fin;
        x->fifo[(int64_t)best * n + x->size[best]++] = fin;
        x->soj[k] = fin - t;
    }
    double r = ceil(0.95 * (double)n);
    int64_t rank = (int64_t)r;
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    qsort(x->soj, n, sizeof(double), cmp_dbl);
    return x->soj[rank - 1];
}

static void visit_plan(rowctx* x, const int* counts, int used) {
    const int64_t pidx = x->counter++;
    if (pidx < x->lo || pidx >= x->hi) return;
    int ok = 1, dp = 0;
    double capacity = 0.0;
    for (int s = 0; s < x->S; ++s) {
        if (!counts[s]) continue;
        if (!x->ok[s]) {
            ok = 0;
            break;
        }
        capacity += counts[s] / x->ms[s];
        for (int r = 0; r < counts[s]; ++r) x->rep_shape[dp++] = s;
    }
    if (!ok || x->rate >= capacity) return;
    const double lat = simulate(x, dp);
    int* slot = x->best_counts + (int64_t)used * MAXS;
    if (!x->has_best[used] || lat < x->best_lat[used] ||
        (lat == x->best_lat[used] && parts_less(counts, slot, x->S))) {
        x->has_best[used] = 1;
        x->best_lat[used] = lat;
        if (x->best_idx) x->best_idx[used] = pidx;
        memcpy(slot, counts, sizeof(int) * MAXS);
    }
}

static void enum_rec(rowctx* x, int idx, int* counts, int used) {
    if (idx == x->S) {
        if (used > 0) visit_plan(x, counts, used);
        return;
    }
    const int size = x->tp[idx] * x->pp[idx];
    for (int k = 0; used + k * size <= x->N; ++k) {
        counts[idx] = k;
        enum_rec(x, idx + 1, counts, used + k * size);
    }
    counts[idx] = 0;
}

static int workload_invalid(const double* w) {
    return w[0] < 0 || w[1] < 0 || w[2] < 0 || w[3] < 0 || w[4] < 0 || w[3] < w[1] || w[4] < w[2];
}

static int co_row_impl(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
                       double* latency, int* plan_counts, int* num_shapes, int* shapes, int64_t lo, int64_t hi,
                       double* shard_lat, int64_t* shard_idx, int64_t* total_plans) {
    if (workload_invalid(w)) return E_INVALID;
    for (int f = 0; f <= max_budget; ++f) latency[f] = INFINITY;
    if (plan_counts) memset(plan_counts, 0, sizeof(int) * (size_t)(max_budget + 1) * MAXS);
    rowctx x;
    memset(&x, 0, sizeof(x));
    x.S = legal_shapes(m, hw, p, x.tp, x.pp);
    if (num_shapes) *num_shapes = x.S;
    if (shapes)
        for (int s = 0; s < x.S; ++s) {
            shapes[2 * s] = x.tp[s];
            shapes[2 * s + 1] = x.pp[s];
        }
    if (w[0] == 0.0) {
        for (int f = 0; f <= max_budget; ++f) latency[f] = 0.0;
        return OK;
    }
    if (max_budget < 1 || x.S == 0) return OK;
    x.N = max_budget;
    x.n_req = p->n_req;
    x.rate = w[0];
    const double kv_tokens = w[3] + w[4];
    const double clamped = w[2] * 0.98168436111126578;
    for (int s = 0; s < x.S; ++s) {
        if (!mem_feasible(x.tp[s], x.pp[s], m, hw, p, kv_tokens)) continue;
        x.ok[s] = 1;
        const double gpus = x.tp[s] * x.pp[s];
        const double bubble = 1.0 + p->bubble * (x.pp[s] - 1);
        x.prefill[s] = (2.0 * m->param_count * w[1] / (gpus * hw->flops * p->prefill_eff) + x.pp[s] * p->comm) * bubble;
        x.decode[s] = m->param_count * m->bytes_per_param / (x.tp[s] * hw->mem_bw * p->decode_eff) + x.pp[s] * p->comm;
        x.ms[s] = x.prefill[s] + clamped * x.decode[s];
    }
    const int64_t n = p->n_req;
    double* arr = (double*)malloc(sizeof(double) * n);
    double* outs = (double*)malloc(sizeof(double) * n);
    mt64 rng;
    mt64_seed(&rng, p->seed);
    double t = 0.0;
    const double cap = 4.0 * w[2];
    for (int64_t k = 0; k < n; ++k) {
        t += exponential_mean(&rng, 1.0) / w[0];
        arr[k] = t;
        double o = exponential_mean(&rng, w[2]);
        outs[k] = (cap < o) ? cap : o;
    }
    x.arr = arr;
    x.outs = outs;
    const int maxdp = max_budget;
    x.fifo = (double*)malloc(sizeof(double) * (size_t)maxdp * n);
    x.head = (int64_t*)malloc(sizeof(int64_t) * maxdp);
    x.size = (int64_t*)malloc(sizeof(int64_t) * maxdp);
    x.avail = (double*)malloc(sizeof(double) * maxdp);
    x.soj = (double*)malloc(sizeof(double) * n);
    x.rep_shape = (int*)malloc(sizeof(int) * maxdp);
    x.best_lat = (double*)malloc(sizeof(double) * (max_budget + 1));
    x.best_counts = (int*)calloc((size_t)(max_budget + 1) * MAXS, sizeof(int));
    x.has_best = (char*)calloc(max_budget + 1, 1);
    x.best_idx = (int64_t*)malloc(sizeof(int64_t) * (max_budget + 1));
    x.counter = 0;
    x.lo = lo;
    x.hi = hi;
    int counts[MAXS];
    memset(counts, 0, sizeof(counts));
    enum_rec(&x, 0, counts, 0);
    if (total_plans) *total_plans = x.counter;
    if (shard_lat)
        for (int g = 0; g <= max_budget; ++g) {
            shard_lat[g] = x.has_best[g] ? x.best_lat[g] : INFINITY;
            shard_idx[g] = x.has_best[g] ? x.best_idx[g] : -1;
        }
    /* prefix minimum, strict '<' (costmodel.cpp:398-412) */
    double running = INFINITY;
    int have = 0, run_g = 0;
    for (int f = 1; f <= max_budget; ++f) {
        if (x.has_best[f] && x.best_lat[f] < running) {
            running = x.best_lat[f];
            run_g = f;
            have = 1;
        }
        if (have) {
            latency[f] = running;
            if (plan_counts) memcpy(plan_counts + (int64_t)f * MAXS, x.best_counts + (int64_t)run_g * MAXS, sizeof(int) * MAXS);
        }
    }
    free(arr);
    free(outs);
    free(x.fifo);
    free(x.head);
    free(x.size);
    free(x.avail);
    free(x.soj);
    free(x.rep_shape);
    free(x.best_lat);
    free(x.best_counts);
    free(x.has_best);
    free(x.best_idx);
    return OK;
}

int co_row(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget, double* latency,
           int* plan_counts, int* num_shapes, int* shapes) {
    return co_row_impl(m, w, hw, p, max_budget, latency, plan_counts, num_shapes, shapes, 0, INT64_MAX, NULL, NULL,
                       NULL);
}

int co_row_shard(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
                 int64_t plan_lo, int64_t plan_hi, double* best_lat, int64_t* best_idx, int64_t* total_plans) {
    double* lat = (double*)malloc(sizeof(double) * (max_budget + 1));
    int rc = co_row_impl(m, w, hw, p, max_budget, lat, NULL, NULL, NULL, plan_lo, plan_hi, best_lat, best_idx,
                         total_plans);
    free(lat);
    return rc;
}

/* ---------------- inner min-max (innerplan.cpp:58-194) */
static int min_budget_within(const double* row, int len, double limit) {
    for (int f = 0; f < len; ++f)
        if (!isinf(row[f]) && row[f] <= limit) return f;
    return -1;
}

int co_solve(const double* entries, int stages, int gpu_budget, int total_gpus, int* alloc, double* objective) {
    const int n = gpu_budget;
    if (n < 0 || stages <= 0) return E_INVALID;
    for (int i = 0; i < stages; ++i) {
        int seen = 0;
        double prev = INFINITY;
        for (int f = 0; f <= n; ++f) {
            double cell = entries[(int64_t)i * (n + 1) + f];
            if (isinf(cell)) {
                if (seen && f > 0) return E_INVALID;
                continue;
            }
            if (cell < 0.0) return E_INVALID;
            if (seen && cell > prev) return E_INVALID;
            seen = 1;
            prev = cell;
        }
    }
    if (total_gpus < 0 || total_gpus > gpu_budget) return E_INVALID;
    double* cand = (double*)malloc(sizeof(double) * (size_t)stages * (total_gpus + 1) + 8);
    int nc = 0;
    for (int i = 0; i < stages; ++i)
        for (int f = 0; f <= total_gpus; ++f) {
            double v = entries[(int64_t)i * (n + 1) + f];
            if (!isinf(v)) cand[nc++] = v;
        }
    qsort(cand, nc, sizeof(double), cmp_dbl);
    int u = 0;
    for (int k = 0; k < nc; ++k)
        if (u == 0 || cand[k] != cand[u - 1]) cand[u++] = cand[k];
    int lo = 0, hi = u - 1, found = -1;
    while (lo <= hi) {
        int mid = lo + (hi - lo) / 2;
        long long need = 0;
        int feas = 1;
        for (int i = 0; i < stages; ++i) {
            int t = min_budget_within(entries + (int64_t)i * (n + 1), n + 1, cand[mid]);
            if (t < 0) {
                feas = 0;
                break;
            }
            need += t;
        }
        if (feas && need <= total_gpus) {
            found = mid;
            hi = mid - 1;
        } else {
            lo = mid + 1;
        }
    }
    if (found < 0) {
        free(cand);
        return E_INFEASIBLE_PROBLEM;
    }
    const double obj = cand[found];
    free(cand);
    int used = 0;
    for (int i = 0; i < stages; ++i) {
        alloc[i] = min_budget_within(entries + (int64_t)i * (n + 1), n + 1, obj);
        used += alloc[i];
    }
    alloc[stages - 1] += total_gpus - used;
    double L = 0.0;
    for (int i = 0; i < stages; ++i) {
        double v = entries[(int64_t)i * (n + 1) + alloc[i]];
        L = (L < v) ? v : L;
    }
    *objective = L;
    return OK;
}

/* ---------------- outer sweep (outerplan.cpp:93-319) */
typedef struct {
    int stage;
    double w[5];
    double* lat;  /* [N+1] */
    int* plans;   /* [(N+1)*MAXS] */
} rowent;

typedef struct {
    rowent* v;
    int n, cap, N;
} rowcache;

static rowent* cache_get(rowcache* rc, int stage, const double* w, const co_model* m, const co_hw* hw,
                         const co_params* p, int* err) {
    for (int i = 0; i < rc->n; ++i)
        if (rc->v[i].stage == stage && memcmp(rc->v[i].w, w, sizeof(double) * 5) == 0) return &rc->v[i];
    if (rc->n == rc->cap) {
        rc->cap = rc->cap ? rc->cap * 2 : 64;
        rc->v = (rowent*)realloc(rc->v, sizeof(rowent) * rc->cap);
    }
    rowent* e = &rc->v[rc->n];
    e->stage = stage;
    memcpy(e->w, w, sizeof(double) * 5);
    e->lat = (double*)malloc(sizeof(double) * (rc->N + 1));
    e->plans = (int*)malloc(sizeof(int) * (size_t)(rc->N + 1) * MAXS);
    int rc2 = co_row(m, w, hw, p, rc->N, e->lat, e->plans, NULL, NULL);
    if (rc2 != OK) {
        free(e->lat);
        free(e->plans);
        *err = rc2;
        return NULL;
    }
    rc->n++;
    return e;
}

static const double* g_L;
static const double* g_Q;
static int cmp_pareto(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    if (g_L[x] != g_L[y]) return g_L[x] < g_L[y] ? -1 : 1;
    if (g_Q[x] != g_Q[y]) return g_Q[x] > g_Q[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int co_sweep(const double* arrival, const double* in_tok, const double* out_tok, const double* scores, int64_t n,
             int c, const co_model* models, const co_hw* hw, const co_params* p, int total_gpus, int grid_dims,
             const int64_t* grid_sizes, const double* grid_values, double wmin, double wmax, int wcount,
             int64_t* eval_cand, double* eval_L, double* eval_Q, int* eval_alloc, int* eval_plan_counts,
             double* weights, int* sel, int64_t* front, int64_t* skipped, int64_t* counts, double* z) {
    if (n == 0) return E_EMPTY;
    if (c <= 0) return E_INVALID;
    for (int i = 0; i < c; ++i) {
        const co_model* m = &models[i];
        if (m->param_count < 0 || m->bytes_per_param < 0 || m->kv_bytes_per_token < 0 || m->min_gpus < 1 ||
            m->stage_index != i + 1 || (i > 0 && m->param_count < models[i - 1].param_count))
            return E_INVALID;
    }
    if (overall_rate(arrival, n) <= 0.0) return E_INVALID;
    const int D = c - 1;
    int gsz[8];
    double* gv[8];
    if (grid_dims == 0) {
        double* tmp = (double*)malloc(sizeof(double) * n);
        for (int d = 0; d < D; ++d) {
            memcpy(tmp, scores + (int64_t)d * n, sizeof(double) * n);
            qsort(tmp, n, sizeof(double), cmp_dbl);
            double vals[11];
            int k = 0;
            vals[k++] = 0.0;
            vals[k++] = 101.0;
            for (int q = 1; q <= 9; ++q) vals[k++] = quantile_sorted(tmp, n, q / 10.0);
            qsort(vals, k, sizeof(double), cmp_dbl);
            int u = 0;
            for (int i = 0; i < k; ++i)
                if (u == 0 || vals[i] != vals[u - 1]) vals[u++] = vals[i];
            gv[d] = (double*)malloc(sizeof(double) * u);
            memcpy(gv[d], vals, sizeof(double) * u);
            gsz[d] = u;
        }
        free(tmp);
    } else {
        if (grid_dims != D) return E_INVALID;
        int64_t off = 0;
        for (int d = 0; d < D; ++d) {
            if (grid_sizes[d] == 0) return E_INVALID;
            gsz[d] = (int)grid_sizes[d];
            gv[d] = (double*)malloc(sizeof(double) * gsz[d]);
            memcpy(gv[d], grid_values + off, sizeof(double) * gsz[d]);
            off += grid_sizes[d];
        }
    }
    if (hw->gpu_count <= 0 || hw->flops <= 0 || hw->mem_bw <= 0 || hw->mem_cap <= 0 || hw->intra_bw <= 0 ||
        hw->inter_bw <= 0 || hw->gpus_per_node <= 0)
        return E_INVALID;
    if (!(p->prefill_eff > 0 && p->prefill_eff <= 1) || !(p->decode_eff > 0 && p->decode_eff <= 1) ||
        !(p->kv_frac > 0 && p->kv_frac <= 1) || p->bubble < 0 || p->comm < 0 || p->n_req <= 0)
        return E_INVALID;

    const int N = total_gpus;
    rowcache rc = {NULL, 0, 0, N};
    int err = OK;
    int* dep = (int*)malloc(sizeof(int) * c);
    for (int i = 0; i < c; ++i) dep[i] = 1;
    double* h = (double*)malloc(sizeof(double) * (c > 1 ? c : 1));
    double* ratios = (double*)malloc(sizeof(double) * c);
    double* wl = (double*)malloc(sizeof(double) * 5 * c);
    double q;
    /* utopia */
    for (int d = 0; d < D; ++d) h[d] = 0.0;
    co_route(arrival, in_tok, out_tok, scores, n, c, h, dep, ratios, wl, &q, NULL);
    rowent* r0 = cache_get(&rc, 0, wl, &models[0], hw, p, &err);
    if (!r0) return err;
    if (isinf(r0->lat[N])) return E_INFEASIBLE;
    z[0] = r0->lat[N];
    for (int d = 0; d < D; ++d) h[d] = 101.0;
    co_route(arrival, in_tok, out_tok, scores, n, c, h, dep, ratios, wl, &q, NULL);
    z[1] = q;

    int64_t ncand = 1;
    for (int d = 0; d < D; ++d) ncand *= gsz[d];
    int64_t E = 0, S = 0;
    double* table = (double*)malloc(sizeof(double) * (size_t)c * (N + 1));
    int* live = (int*)malloc(sizeof(int) * c);
    rowent** lrows = (rowent**)malloc(sizeof(rowent*) * c);
    int* al = (int*)malloc(sizeof(int) * c);
    for (int64_t cand = 0; cand < ncand; ++cand) {
        int64_t rem = cand;
        for (int d = D - 1; d >= 0; --d) {
            h[d] = gv[d][rem % gsz[d]];
            rem /= gsz[d];
        }
        co_route(arrival, in_tok, out_tok, scores, n, c, h, dep, ratios, wl, &q, NULL);
        int nl = 0;
        for (int i = 0; i < c; ++i)
            if (ratios[i] > 0.0) live[nl++] = i;
        for (int k = 0; k < nl; ++k) {
            rowent* e = cache_get(&rc, live[k], wl + 5 * live[k], &models[live[k]], hw, p, &err);
            if (!e) return err;
            lrows[k] = e;
            memcpy(table + (int64_t)k * (N + 1), e->lat, sizeof(double) * (N + 1));
            table[(int64_t)k * (N + 1)] = INFINITY;
        }
        double L;
        int rcode = co_solve(table, nl, N, N, al, &L);
        if (rcode == E_INFEASIBLE_PROBLEM) {
            skipped[S++] = cand;
            continue;
        }
        if (rcode != OK) return rcode;
        eval_cand[E] = cand;
        eval_L[E] = L;
        eval_Q[E] = q;
        for (int i = 0; i < c; ++i) eval_alloc[E * c + i] = 0;
        memset(eval_plan_counts + E * c * MAXS, 0, sizeof(int) * c * MAXS);
        for (int k = 0; k < nl; ++k) {
            eval_alloc[E * c + live[k]] = al[k];
            if (al[k] > 0)
                memcpy(eval_plan_counts + (E * c + live[k]) * MAXS, lrows[k]->plans + (int64_t)al[k] * MAXS,
                       sizeof(int) * MAXS);
        }
        ++E;
    }
    if (E == 0) return E_INFEASIBLE_PROBLEM;
    if (wcount < 1 || wmin <= 0 || wmax < wmin) return E_INVALID;
    for (int k = 0; k < wcount; ++k) {
        double t = wcount == 1 ? 0.0 : (double)k / (wcount - 1);
        double ratio = wmin * pow(wmax / wmin, t);
        weights[2 * k] = ratio / (1.0 + ratio);
        weights[2 * k + 1] = 1.0 / (1.0 + ratio);
        int best = -1;
        double bt = 0.0;
        for (int64_t i = 0; i < E; ++i) {
            double a1 = weights[2 * k] * (eval_L[i] - z[0]);
            double a2 = weights[2 * k + 1] * (z[1] - eval_Q[i]);
            double tt = (a1 < a2) ? a2 : a1;
            int take = best < 0 || tt < bt ||
                       (tt == bt && (eval_L[i] < eval_L[best] || (eval_L[i] == eval_L[best] && eval_Q[i] > eval_Q[best])));
            if (take) {
                best = (int)i;
                bt = tt;
            }
        }
        sel[k] = best;
    }
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * E);
    for (int64_t i = 0; i < E; ++i) order[i] = i;
    g_L = eval_L;
    g_Q = eval_Q;
    qsort(order, E, sizeof(int64_t), cmp_pareto);
    int64_t F = 0;
    double bq = -INFINITY;
    for (int64_t i = 0; i < E; ++i)
        if (eval_Q[order[i]] > bq) {
            front[F++] = order[i];
            bq = eval_Q[order[i]];
        }
    counts[0] = E;
    counts[1] = F;
    counts[2] = S;
    counts[3] = wcount;
    free(order);
    free(table);
    free(live);
    free(lrows);
    free(al);
    free(dep);
    free(h);
    free(ratios);
    free(wl);
    for (int i = 0; i < rc.n; ++i) {
        free(rc.v[i].lat);
        free(rc.v[i].plans);
    }
    free(rc.v);
    for (int d = 0; d < D; ++d) free(gv[d]);
    return OK;
}

/* ---------------- plan census (bench.py's CPU-baseline extrapolation only)
 *
 * For one row (model, workload, budget N): the number of plans the reference
 * enumerates (enumerate_multisets, costmodel.cpp:132-146), and how many of
 * them pass the stability test of StageEvaluator::row (costmodel.cpp:366-376:
 * every part's shape memory-feasible at the p95 sequence length, and
 * rate < sum over parts in shape order of cnt / mean_service[s]) -- i.e. how
 * many queueing simulations the reference runs for that row -- binned by the
 * replica count dp (bins: dp <= 4, 8, 16, 32, 64, 128, 256, > 256) together
 * with the sum of dp per bin.  No simulation is run.  Threaded over prefixes
 * of the enumeration (pthreads, dynamic task claiming). */
#include <pthread.h>

#define CENSUS_BINS 8

typedef struct {
    int S, N, L;
    int size[MAXS];
    char ok[MAXS];
    double ms[MAXS];
    double rate;
    /* task prefixes: counts of shapes [0, L) */
    int* prefix;
    int64_t ntasks;
    int64_t next;
    pthread_mutex_t mu;
    int64_t plans, stable, bin_n[CENSUS_BINS], bin_dp[CENSUS_BINS];
} census_ctx;

typedef struct {
    int64_t plans, stable, bin_n[CENSUS_BINS], bin_dp[CENSUS_BINS];
} census_acc;

static int census_bin(int dp) {
    int b = 0;
    for (int lim = 4; b < CENSUS_BINS - 1 && dp > lim; lim *= 2) ++b;
    return b;
}

/* level idx onward; cap = capacity of the parts so far (shape order), bad =
 * some nonzero part is memory-infeasible */
static void census_rec(const census_ctx* x, census_acc* a, int idx, int used, int dp, double cap, int bad) {
    if (idx == x->S) {
        if (used == 0) return;
        a->plans++;
        if (bad || x->rate >= cap) return;
        a->stable++;
        const int b = census_bin(dp);
        a->bin_n[b]++;
        a->bin_dp[b] += dp;
        return;
    }
    const int size = x->size[idx];
    for (int k = 0; used + k * size <= x->N; ++k) {
        const double c2 = k > 0 ? cap + (double)k / x->ms[idx] : cap;
        census_rec(x, a, idx + 1, used + k * size, dp + k, c2, bad || (k > 0 && !x->ok[idx]));
    }
}

static int64_t census_prefixes(const census_ctx* x, int L, int* out) {
    /* all count vectors of shapes [0, L) with sum of gpus <= N, recursion order */
    int64_t n = 0;
    int c[MAXS];
    memset(c, 0, sizeof(c));
    int used = 0, lvl = 0;
    /* iterative odometer over levels [0, L) */
    for (;;) {
        if (lvl == L) {
            if (out) memcpy(out + n * L, c, sizeof(int) * L);
            ++n;
            /* advance */
            --lvl;
            while (lvl >= 0) {
                if (used + x->size[lvl] <= x->N) {
                    c[lvl]++;
                    used += x->size[lvl];
                    ++lvl;
                    break;
                }
                used -= c[lvl] * x->size[lvl];
                c[lvl] = 0;
                --lvl;
            }
            if (lvl < 0) break;
            continue;
        }
        ++lvl;
    }
    return n;
}

static void* census_worker(void* arg) {
    census_ctx* x = (census_ctx*)arg;
    census_acc a;
    memset(&a, 0, sizeof(a));
    for (;;) {
        pthread_mutex_lock(&x->mu);
        const int64_t t = x->next++;
        pthread_mutex_unlock(&x->mu);
        if (t >= x->ntasks) break;
        const int* c = x->prefix + t * x->L;
        int used = 0, dp = 0, bad = 0;
        double cap = 0.0;
        for (int s = 0; s < x->L; ++s) {
            used += c[s] * x->size[s];
            dp += c[s];
            if (c[s] > 0) {
                cap = cap + (double)c[s] / x->ms[s];
                bad = bad || !x->ok[s];
            }
        }
        census_rec(x, &a, x->L, used, dp, cap, bad);
    }
    pthread_mutex_lock(&x->mu);
    x->plans += a.plans;
    x->stable += a.stable;
    for (int b = 0; b < CENSUS_BINS; ++b) {
        x->bin_n[b] += a.bin_n[b];
        x->bin_dp[b] += a.bin_dp[b];
    }
    pthread_mutex_unlock(&x->mu);
    return NULL;
}

/* out[0] = plans, out[1] = stable plans, out[2 + b] = stable plans in dp bin b,
 * out[2 + CENSUS_BINS + b] = sum of dp over them. */
int co_row_census(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
                  int threads, int64_t* out) {
    memset(out, 0, sizeof(int64_t) * (2 + 2 * CENSUS_BINS));
    if (workload_invalid(w)) return E_INVALID;
    census_ctx x;
    memset(&x, 0, sizeof(x));
    int tp[MAXS], pp[MAXS];
    x.S = legal_shapes(m, hw, p, tp, pp);
    if (max_budget < 1 || x.S == 0) return OK;
    x.N = max_budget;
    x.rate = w[0];
    const double kv_tokens = w[3] + w[4];
    const double clamped = w[2] * 0.98168436111126578;
    for (int s = 0; s < x.S; ++s) {
        x.size[s] = tp[s] * pp[s];
        if (!mem_feasible(tp[s], pp[s], m, hw, p, kv_tokens)) continue;
        x.ok[s] = 1;
        const double gpus = tp[s] * pp[s];
        const double bubble = 1.0 + p->bubble * (pp[s] - 1);
        const double prefill = (2.0 * m->param_count * w[1] / (gpus * hw->flops * p->prefill_eff) + pp[s] * p->comm) * bubble;
        const double decode = m->param_count * m->bytes_per_param / (tp[s] * hw->mem_bw * p->decode_eff) + pp[s] * p->comm;
        x.ms[s] = prefill + clamped * decode;
    }
    if (w[0] == 0.0) { /* the reference returns an all-zero row without enumerating */
        return OK;
    }
    if (threads < 1) threads = 1;
    /* prefix depth: enough tasks to balance the threads */
    int L = 0;
    int64_t nt = 1;
    while (L < x.S && nt < 256 * (int64_t)threads) {
        ++L;
        nt = census_prefixes(&x, L, NULL);
    }
    x.L = L;
    x.ntasks = nt;
    x.prefix = (int*)malloc(sizeof(int) * (size_t)(nt * (L > 0 ? L : 1)));
    census_prefixes(&x, L, x.prefix);
    pthread_mutex_init(&x.mu, NULL);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, census_worker, &x);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&x.mu);
    free(th);
    free(x.prefix);
    out[0] = x.plans;
    out[1] = x.stable;
    for (int b = 0; b < CENSUS_BINS; ++b) {
        out[2 + b] = x.bin_n[b];
        out[2 + CENSUS_BINS + b] = x.bin_dp[b];
    }
    return OK;
}
