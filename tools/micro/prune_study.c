/*
 * Development study (not product, not a test): how many JSQ request-steps the
 * K4 prune rules need per row, on the CPU, with the row's exact final bounds
 * (the ub_oracle situation).  Includes the C oracle for its row tables.
 *
 * Rules, checked every `every` steps after request k-1 was dispatched:
 *   A  (K4 today) exceedances so far + future requests whose service lower
 *      bound exceeds U on every shape of the plan >= K
 *   B  A, where a future request j also counts when the earliest replica
 *      release time bounds its wait: max(0, Amin - t_j) + svcmin_j > U
 *      (start_j >= avail_b(now) >= Amin for whichever replica b JSQ picks)
 */
#include "../../oracle/cascade_oracle.c"

#include <stdio.h>

typedef struct {
    int64_t plans, stable, steps_full, steps_a, steps_b, pruned_a, pruned_b, first_a, first_b;
    int64_t hist[12], hsteps[12];  /* rule A prune step k by log2 bucket: count, steps */
} co_study;

static int64_t run_rule(rowctx* x, int dp, double U, int K, int every, int rule, int* pruned_at_first) {
    const int64_t n = x->n_req;
    double smin_p = INFINITY, smin_d = INFINITY;
    for (int j = 0; j < dp; ++j) {
        const int s = x->rep_shape[j];
        if (x->prefill[s] < smin_p) smin_p = x->prefill[s];
        if (x->decode[s] < smin_d) smin_d = x->decode[s];
    }
    for (int j = 0; j < dp; ++j) {
        x->avail[j] = 0.0;
        x->head[j] = 0;
        x->size[j] = 0;
    }
    int ab = 0;
    for (int64_t k = 0; k < n; ++k) {
        if (k > 0 && k % every == 0) {
            double amin = INFINITY;
            for (int j = 0; j < dp; ++j) amin = x->avail[j] < amin ? x->avail[j] : amin;
            int fut = 0;
            if (rule == 2) {
                /* K4 today: the exact count rounded down to blocks of 32 in output
                   rank order, and k rounded up to a multiple of 32 */
                int cex = 0;
                for (int64_t j = 0; j < n; ++j) {
                    double svc = INFINITY;
                    for (int r = 0; r < dp; ++r) {
                        const int s = x->rep_shape[r];
                        const double v = x->prefill[s] + x->outs[j] * x->decode[s];
                        svc = v < svc ? v : svc;
                    }
                    if (svc * (1.0 - 1e-12) - 1e-12 * x->arr[n - 1] > U) ++cex;
                }
                const int c32 = cex / 32 * 32;
                /* requests of output rank < c32 arriving at j >= 32*ceil(k/32):
                   rank by output descending, ties by index */
                const int64_t k32 = (k + 31) / 32 * 32;
                for (int64_t j = k32; j < n; ++j) {
                    int rank = 0;
                    for (int64_t i = 0; i < n; ++i)
                        rank += (x->outs[i] > x->outs[j]) || (x->outs[i] == x->outs[j] && i < j);
                    if (rank < c32) ++fut;
                }
            } else
            for (int64_t j = k; j < n; ++j) {
                double svc = INFINITY;
                for (int r = 0; r < dp; ++r) {
                    const int s = x->rep_shape[r];
                    const double v = x->prefill[s] + x->outs[j] * x->decode[s];
                    svc = v < svc ? v : svc;
                }
                double lb = svc * (1.0 - 1e-12) - 1e-12 * x->arr[n - 1];
                if (rule == 1 && amin > x->arr[j]) {
                    /* B': per replica, the wait until its current release plus its own service */
                    double b2 = INFINITY;
                    for (int r = 0; r < dp; ++r) {
                        const int s = x->rep_shape[r];
                        const double wv = x->avail[r] > x->arr[j] ? x->avail[r] - x->arr[j] : 0.0;
                        const double v = wv + x->prefill[s] + x->outs[j] * x->decode[s];
                        b2 = v < b2 ? v : b2;
                    }
                    b2 = b2 * (1.0 - 1e-12) - 1e-12 * x->arr[n - 1];
                    lb = b2 > lb ? b2 : lb;
                }
                if (lb > U) ++fut;
            }
            if (ab + fut >= K) {
                if (pruned_at_first) *pruned_at_first = (k == every);
                return k;
            }
        }
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
        if (fin - t > U) ++ab;
    }
    return -n;  /* completed */
}

typedef struct {
    rowctx* x;
    const double* U;  /* final row latency per budget */
    int K, every;
    co_study* st;
} studyctx;

static void study_rec(studyctx* c, int idx, int* counts, int used) {
    rowctx* x = c->x;
    if (idx == x->S) {
        if (used == 0) return;
        c->st->plans++;
        int dp = 0;
        double capacity = 0.0;
        for (int s = 0; s < x->S; ++s) {
            if (!counts[s]) continue;
            if (!x->ok[s]) return;
            capacity += counts[s] / x->ms[s];
            for (int r = 0; r < counts[s]; ++r) x->rep_shape[dp++] = s;
        }
        if (x->rate >= capacity) return;
        c->st->stable++;
        const double U = c->U[used];
        int fa = 0, fb = 0;
        int64_t a = run_rule(x, dp, U, c->K, c->every, 0, &fa);
        int64_t b = run_rule(x, dp, U, c->K, c->every, 2, &fb);
        if (a < 0) c->st->steps_full += -a; else { c->st->steps_a += a; c->st->pruned_a++; c->st->first_a += fa; }
        {
            int64_t kk = a < 0 ? -a : a;
            int bkt = 0;
            while ((4ll << bkt) < kk && bkt < 11) ++bkt;
            c->st->hist[bkt]++;
            c->st->hsteps[bkt] += kk;
        }
        if (b < 0) c->st->steps_full += 0; else { c->st->steps_b += b; c->st->pruned_b++; c->st->first_b += fb; }
        if (b < 0) c->st->steps_b += -b;
        if (a < 0) c->st->steps_a += -a;
        return;
    }
    const int size = x->tp[idx] * x->pp[idx];
    for (int k = 0; used + k * size <= x->N; ++k) {
        counts[idx] = k;
        study_rec(c, idx + 1, counts, used + k * size);
    }
    counts[idx] = 0;
}

int co_prune_study(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int N, int every,
                   int64_t plan_limit, int64_t* out) {
    double* lat = (double*)malloc(sizeof(double) * (N + 1));
    int rc = co_row_impl(m, w, hw, p, N, lat, NULL, NULL, NULL, 0, INT64_MAX, NULL, NULL, NULL);
    if (rc != OK) return rc;
    /* rebuild the row context (co_row_impl frees its own) */
    rowctx x;
    memset(&x, 0, sizeof(x));
    x.S = legal_shapes(m, hw, p, x.tp, x.pp);
    x.N = N;
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
    x.fifo = (double*)malloc(sizeof(double) * (size_t)N * n);
    x.head = (int64_t*)malloc(sizeof(int64_t) * N);
    x.size = (int64_t*)malloc(sizeof(int64_t) * N);
    x.avail = (double*)malloc(sizeof(double) * N);
    x.rep_shape = (int*)malloc(sizeof(int) * N);
    co_study st;
    memset(&st, 0, sizeof(st));
    /* the row's final bound at each budget: the prefix minimum */
    studyctx c = {&x, lat, (int)(n - (int64_t)ceil(0.95 * (double)n) + 1), every, &st};
    (void)plan_limit;
    int counts[MAXS];
    memset(counts, 0, sizeof(counts));
    study_rec(&c, 0, counts, 0);
    out[0] = st.plans;
    out[1] = st.stable;
    out[2] = st.steps_a;
    out[3] = st.steps_b;
    out[4] = st.pruned_a;
    out[5] = st.pruned_b;
    out[6] = st.first_a;
    out[7] = st.first_b;
    for (int i = 0; i < 12; ++i) {
        out[8 + i] = st.hist[i];
        out[20 + i] = st.hsteps[i];
    }
    free(arr);
    free(outs);
    free(x.fifo);
    free(x.head);
    free(x.size);
    free(x.avail);
    free(x.rep_shape);
    free(lat);
    return OK;
}
