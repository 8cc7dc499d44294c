/*
 * slora_oracle.c -- CPU fp64 ORACLE (TEST INFRASTRUCTURE ONLY; see header).
 *
 * Plain, slow, obviously correct loops.  No blocking, no fusion, no
 * reordering beyond the definition written in slora_oracle.h:
 *   Eq. (lora_factored):  out_i = y_in_i + scale_a * (x_i A_a) B_a
 * Compile with -ffp-contract=off so that every a*b+c is two roundings in the
 * order written here.
 */
#include "slora_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t t0, t1, h, d;
    const double *x, *y_in, *A_all, *B_all, *scale;
    const int64_t *rank, *A_off, *B_off, *slot;
    double* out;
    int64_t flops;
    int64_t r_pad; /* 0 = unpadded; else every adapter padded to r_pad */
} job_t;

/* One token range.  For token i with adapter a:
 *   v[j]   = sum_k x[i,k] A_a[k,j]          (shrink, k ascending)
 *   dl[c]  = sum_j v[j] B_a[j,c]            (expand, j ascending)
 *   out[i] = y_in[i] + scale_a * dl          (R6)
 * With r_pad > 0 the loops run to r_pad and read zero for j >= r_a (the
 * padded baseline of P:193-195): the extra terms are exact zeros. */
static void* run_range(void* arg) {
    job_t* jb = (job_t*)arg;
    const int64_t h = jb->h, d = jb->d;
    int64_t flops = 0;
    for (int64_t i = jb->t0; i < jb->t1; ++i) {
        const double* xi = jb->x + i * h;
        double* oi = jb->out + i * d;
        const double* yi = jb->y_in + i * d;
        int64_t a = jb->slot[i];
        if (a < 0) { /* no adapter: base output untouched (R7) */
            for (int64_t c = 0; c < d; ++c) oi[c] = yi[c];
            continue;
        }
        const int64_t r = jb->rank[a];
        const int64_t rl = jb->r_pad > 0 ? jb->r_pad : r; /* loop bound */
        const double* A = jb->A_all + jb->A_off[a]; /* h x r, row-major */
        const double* B = jb->B_all + jb->B_off[a]; /* r x d, row-major */
        double* v = (double*)malloc(sizeof(double) * (size_t)rl);
        double* dl = (double*)malloc(sizeof(double) * (size_t)d);
        /* shrink: v = x_i A */
        for (int64_t j = 0; j < rl; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < h; ++k) {
                double akj = (j < r) ? A[k * r + j] : 0.0; /* zero padding */
                acc = acc + xi[k] * akj;
                flops += 2;
            }
            v[j] = acc;
        }
        /* expand: dl = v B */
        for (int64_t c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int64_t j = 0; j < rl; ++j) {
                double bjc = (j < r) ? B[j * d + c] : 0.0; /* zero padding */
                acc = acc + v[j] * bjc;
                flops += 2;
            }
            dl[c] = acc;
        }
        const double s = jb->scale[a];
        for (int64_t c = 0; c < d; ++c) oi[c] = yi[c] + s * dl[c];
        free(v);
        free(dl);
    }
    jb->flops = flops;
    return NULL;
}

static int check_args(int64_t T, int64_t h, int64_t d, int64_t n_adapters,
                      const int64_t* rank, const int64_t* slot) {
    if (T < 0 || h < 1 || d < 1 || n_adapters < 0) return -1;
    for (int64_t a = 0; a < n_adapters; ++a)
        if (rank[a] < 1) return -1;
    for (int64_t i = 0; i < T; ++i)
        if (slot[i] < -1 || slot[i] >= n_adapters) return -1;
    return 0;
}

static int run_jobs(job_t proto, int64_t T, int nthreads, int64_t* flops_out) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > T && T > 0) nthreads = (int)T;
    if (T == 0) nthreads = 1;
    job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (T + nthreads - 1) / (nthreads > 0 ? nthreads : 1);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].t0 = t * per < T ? t * per : T;
        jobs[t].t1 = (t + 1) * per < T ? (t + 1) * per : T;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_range, &jobs[t]);
    run_range(&jobs[0]);
    int64_t flops = jobs[0].flops;
    for (int t = 1; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        flops += jobs[t].flops;
    }
    if (flops_out) *flops_out = flops;
    free(jobs);
    free(th);
    return 0;
}

int oracle_lora_apply(int64_t T, int64_t h, int64_t d, const double* x,
                      const double* y_in, int64_t n_adapters,
                      const int64_t* rank, const double* scale,
                      const int64_t* A_off, const int64_t* B_off,
                      const double* A_all, const double* B_all,
                      const int64_t* slot, double* out, int nthreads,
                      int64_t* flops_out) {
    if (check_args(T, h, d, n_adapters, rank, slot)) return -1;
    job_t p;
    memset(&p, 0, sizeof(p));
    p.h = h; p.d = d; p.x = x; p.y_in = y_in; p.A_all = A_all; p.B_all = B_all;
    p.scale = scale; p.rank = rank; p.A_off = A_off; p.B_off = B_off;
    p.slot = slot; p.out = out; p.r_pad = 0;
    return run_jobs(p, T, nthreads, flops_out);
}

int oracle_padded_apply(int64_t T, int64_t h, int64_t d, const double* x,
                        const double* y_in, int64_t n_adapters,
                        const int64_t* rank, const double* scale,
                        const int64_t* A_off, const int64_t* B_off,
                        const double* A_all, const double* B_all,
                        const int64_t* slot, double* out, int64_t* flops_out) {
    if (check_args(T, h, d, n_adapters, rank, slot)) return -1;
    int64_t r_max = 0; /* max rank over adapters used in this batch */
    for (int64_t i = 0; i < T; ++i)
        if (slot[i] >= 0 && rank[slot[i]] > r_max) r_max = rank[slot[i]];
    job_t p;
    memset(&p, 0, sizeof(p));
    p.h = h; p.d = d; p.x = x; p.y_in = y_in; p.A_all = A_all; p.B_all = B_all;
    p.scale = scale; p.rank = rank; p.A_off = A_off; p.B_off = B_off;
    p.slot = slot; p.out = out; p.r_pad = r_max > 0 ? r_max : 1;
    return run_jobs(p, T, 1, flops_out);
}

typedef struct {
    int64_t t0, t1, h, d;
    const double *x, *W;
    double* out;
} base_job_t;

static void* run_base(void* arg) {
    base_job_t* jb = (base_job_t*)arg;
    for (int64_t i = jb->t0; i < jb->t1; ++i)
        for (int64_t c = 0; c < jb->d; ++c) {
            double acc = 0.0;
            for (int64_t k = 0; k < jb->h; ++k) acc = acc + jb->x[i * jb->h + k] * jb->W[k * jb->d + c];
            jb->out[i * jb->d + c] = acc;
        }
    return NULL;
}

int oracle_base_forward(int64_t T, int64_t h, int64_t d, const double* x,
                        const double* W, double* out, int nthreads) {
    if (T < 0 || h < 1 || d < 1) return -1;
    if (nthreads < 1) nthreads = 1;
    if (T > 0 && nthreads > T) nthreads = (int)T;
    base_job_t* jobs = (base_job_t*)calloc((size_t)nthreads, sizeof(base_job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t per = (T + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].h = h; jobs[t].d = d; jobs[t].x = x; jobs[t].W = W; jobs[t].out = out;
        jobs[t].t0 = t * per < T ? t * per : T;
        jobs[t].t1 = (t + 1) * per < T ? (t + 1) * per : T;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run_base, &jobs[t]);
    run_base(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}
