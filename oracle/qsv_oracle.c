/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Never called by the product
 * (paper_2512_18995_b200/), only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg, and there only as the checker.
 *
 * A plain-C restatement of the reference's qubit hot path (quasar::qubit,
 * /root/reference/proj/include/quasar). Each function cites the reference
 * lines it restates. Pinned against the reference itself: tests/test_oracle.py
 * checks it against oracle/_ref/libquasar_ref.so (the unmodified reference
 * headers compiled here) and against tests/golden/*.json, which
 * tests/golden/make_golden.py generated from that library.
 *
 * Conventions (reference): wire 0 is the MOST significant bit of a basis index
 * (state.hpp:21-24); 2^k x 2^k gate matrices index wires[0] as their MSB
 * (gate.hpp:30, state.hpp:96-105); amplitudes are interleaved (re, im) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- Rng ---- */
/* rng.hpp:29-103: splitmix64 on a keyed counter, fnv1a stream labels,
 * Box-Muller normal with a cached spare. */
typedef struct {
    uint64_t key, counter;
    double spare;
    int have_spare;
} qo_rng;

static uint64_t qo_mix(uint64_t z) { /* rng.hpp:83-88 */
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static uint64_t qo_fnv1a(const char *s) { /* rng.hpp:90-97 */
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 0x100000001b3ull;
    }
    return h;
}

void qo_rng_init(qo_rng *r, uint64_t seed, const char *label) { /* rng.hpp:31-33 */
    if (label) seed ^= qo_fnv1a(label);
    r->key = qo_mix(seed ^ 0x9e3779b97f4a7c15ull);
    r->counter = 0;
    r->spare = 0.0;
    r->have_spare = 0;
}

uint64_t qo_rng_next_u64(qo_rng *r) { return qo_mix(r->key + 0x9e3779b97f4a7c15ull * ++r->counter); } /* :43 */

double qo_rng_uniform(qo_rng *r) { return (double)(qo_rng_next_u64(r) >> 11) * 0x1.0p-53; } /* :46-48 */

double qo_rng_normal(qo_rng *r) { /* rng.hpp:53-65 */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = 0.0;
    while (u1 == 0.0) u1 = qo_rng_uniform(r);
    double u2 = qo_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    r->spare = rad * sin(2.0 * 3.141592653589793 * u2);
    r->have_spare = 1;
    return rad * cos(2.0 * 3.141592653589793 * u2);
}

uint64_t qo_rng_next_below(qo_rng *r, uint64_t n) { return n ? qo_rng_next_u64(r) % n : 0; } /* :80 */

size_t qo_rng_sizeof(void) { return sizeof(qo_rng); }

/* Bulk draws (kind: 0 u64, 1 uniform, 2 normal, 3 next_below(arg)); returns
 * the generator state afterwards so callers can continue the stream. */
void qo_rng_draw(qo_rng *r, int kind, uint64_t arg, int64_t count, void *out) {
    for (int64_t i = 0; i < count; ++i) {
        switch (kind) {
        case 0: ((uint64_t *)out)[i] = qo_rng_next_u64(r); break;
        case 1: ((double *)out)[i] = qo_rng_uniform(r); break;
        case 2: ((double *)out)[i] = qo_rng_normal(r); break;
        default: ((uint64_t *)out)[i] = qo_rng_next_below(r, arg); break;
        }
    }
}

/* ------------------------------------------------------------- gates ---- */
/* Gate record; same field meaning as quasar::qubit::Gate (gate.hpp:28-38). */
typedef struct {
    char name[16];
    int32_t nwires;
    int32_t wires[2];
    int32_t ncontrols;
    int32_t controls[6];
    int32_t nparams;
    double params[3];
    int32_t trainable;
    int32_t encode;
    const double *custom;
} qo_gate;

#define CSET(m, d, r, c, re, im)                                                                                       \
    do {                                                                                                               \
        (m)[2 * ((r) * (d) + (c))] = (re);                                                                             \
        (m)[2 * ((r) * (d) + (c)) + 1] = (im);                                                                         \
    } while (0)

/* rot(G, theta) = cos(theta/2) I - i sin(theta/2) G (gate.hpp:63-68); G is
 * given as a real-or-imaginary d x d matrix in (re,im) layout. */
static void qo_rot(const double *G, int d, double theta, double *out) {
    const double c = cos(theta / 2), s = sin(theta / 2);
    for (int r = 0; r < d; ++r)
        for (int k = 0; k < d; ++k) {
            const double gre = G[2 * (r * d + k)], gim = G[2 * (r * d + k) + 1];
            /* c*delta - (0,s)*(gre,gim) = c*delta - (-s*gim, s*gre) */
            CSET(out, d, r, k, (r == k ? c : 0.0) + s * gim, -s * gre);
        }
}

static void qo_kron2(const double *a, const double *b, double *out) { /* gate.hpp:78-84 */
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            for (int k = 0; k < 2; ++k)
                for (int l = 0; l < 2; ++l) {
                    const double ar = a[2 * (i * 2 + j)], ai = a[2 * (i * 2 + j) + 1];
                    const double br = b[2 * (k * 2 + l)], bi = b[2 * (k * 2 + l) + 1];
                    CSET(out, 4, i * 2 + k, j * 2 + l, ar * br - ai * bi, ar * bi + ai * br);
                }
}

static const double QO_X[8] = {0, 0, 1, 0, 1, 0, 0, 0};
static const double QO_Y[8] = {0, 0, 0, -1, 0, 1, 0, 0};
static const double QO_Z[8] = {1, 0, 0, 0, 0, 0, -1, 0};

/* gate_matrix (gate.hpp:89-154). Returns k (1 or 2) or -1 for an unknown
 * name / wrong parameter count (the reference throws invalid_input). */
int qo_gate_matrix(const qo_gate *g, double *m) {
    const char *nm = g->name;
    const double *p = g->params;
    const double kpi = 3.141592653589793238462643383279502884;
    memset(m, 0, sizeof(double) * 32);
#define NEED(k)                                                                                                        \
    if (g->nparams != (k)) return -1
    if (!strcmp(nm, "x")) { memcpy(m, QO_X, sizeof QO_X); return 1; }
    if (!strcmp(nm, "y")) { memcpy(m, QO_Y, sizeof QO_Y); return 1; }
    if (!strcmp(nm, "z")) { memcpy(m, QO_Z, sizeof QO_Z); return 1; }
    if (!strcmp(nm, "h")) {
        const double r = 1.0 / sqrt(2.0);
        CSET(m, 2, 0, 0, r, 0); CSET(m, 2, 0, 1, r, 0); CSET(m, 2, 1, 0, r, 0); CSET(m, 2, 1, 1, -r, 0);
        return 1;
    }
    if (!strcmp(nm, "s")) { CSET(m, 2, 0, 0, 1, 0); CSET(m, 2, 1, 1, 0, 1); return 1; }
    if (!strcmp(nm, "t")) { CSET(m, 2, 0, 0, 1, 0); CSET(m, 2, 1, 1, cos(kpi / 4), sin(kpi / 4)); return 1; }
    if (!strcmp(nm, "rx")) { NEED(1); qo_rot(QO_X, 2, p[0], m); return 1; }
    if (!strcmp(nm, "ry")) { NEED(1); qo_rot(QO_Y, 2, p[0], m); return 1; }
    if (!strcmp(nm, "rz")) { NEED(1); qo_rot(QO_Z, 2, p[0], m); return 1; }
    if (!strcmp(nm, "p")) { NEED(1); CSET(m, 2, 0, 0, 1, 0); CSET(m, 2, 1, 1, cos(p[0]), sin(p[0])); return 1; }
    if (!strcmp(nm, "u3")) { /* gate.hpp:70-76 */
        NEED(3);
        const double c = cos(p[0] / 2), s = sin(p[0] / 2);
        CSET(m, 2, 0, 0, c, 0);
        CSET(m, 2, 0, 1, -cos(p[2]) * s, -sin(p[2]) * s);
        CSET(m, 2, 1, 0, cos(p[1]) * s, sin(p[1]) * s);
        CSET(m, 2, 1, 1, cos(p[1] + p[2]) * c, sin(p[1] + p[2]) * c);
        return 1;
    }
    if (!strcmp(nm, "swap")) {
        CSET(m, 4, 0, 0, 1, 0); CSET(m, 4, 3, 3, 1, 0); CSET(m, 4, 1, 2, 1, 0); CSET(m, 4, 2, 1, 1, 0);
        return 2;
    }
    if (!strcmp(nm, "rxx") || !strcmp(nm, "ryy") || !strcmp(nm, "rzz")) {
        NEED(1);
        const double *P = nm[1] == 'x' ? QO_X : nm[1] == 'y' ? QO_Y : QO_Z;
        double G[32];
        qo_kron2(P, P, G);
        qo_rot(G, 4, p[0], m);
        return 2;
    }
    if (!strcmp(nm, "custom")) {
        if (!g->custom) return -1;
        const int d = 1 << g->nwires;
        memcpy(m, g->custom, sizeof(double) * 2 * d * d);
        return g->nwires;
    }
    return -1;
#undef NEED
}

/* ---------------------------------------------------- strided kernel ---- */
/* detail::apply_matrix_strided (state.hpp:111-143): in place, psi <- M psi on
 * the target wires for every group base with no target bit set and every
 * control bit set; zero_off_control zeroes the off-control groups. */
int qo_apply_matrix(double *psi, int n, const double *m, int k, const int32_t *wires, int nctl,
                    const int32_t *ctls, int zero_off_control) {
    if (k < 1 || k > 5) return -1;
    for (int i = 0; i < k; ++i)
        if (wires[i] < 0 || wires[i] >= n) return -1;
    for (int i = 0; i < nctl; ++i)
        if (ctls[i] < 0 || ctls[i] >= n) return -1;
    uint64_t tmask = 0, cmask = 0, off[32];
    for (int i = 0; i < k; ++i) tmask |= 1ull << (n - 1 - wires[i]);
    for (int i = 0; i < nctl; ++i) cmask |= 1ull << (n - 1 - ctls[i]);
    const int gs = 1 << k;
    for (int j = 0; j < gs; ++j) { /* group_offsets, state.hpp:96-105 */
        off[j] = 0;
        for (int i = 0; i < k; ++i)
            if ((j >> (k - 1 - i)) & 1) off[j] |= 1ull << (n - 1 - wires[i]);
    }
    const uint64_t dim = 1ull << n;
    double sre[32], sim[32];
    for (uint64_t base = 0; base < dim; ++base) {
        if (base & tmask) continue;
        if ((base & cmask) != cmask) {
            if (zero_off_control)
                for (int j = 0; j < gs; ++j) psi[2 * (base + off[j])] = psi[2 * (base + off[j]) + 1] = 0.0;
            continue;
        }
        for (int j = 0; j < gs; ++j) {
            sre[j] = psi[2 * (base + off[j])];
            sim[j] = psi[2 * (base + off[j]) + 1];
        }
        for (int r = 0; r < gs; ++r) {
            double are = 0.0, aim = 0.0;
            for (int c = 0; c < gs; ++c) {
                const double mr = m[2 * (r * gs + c)], mi = m[2 * (r * gs + c) + 1];
                are += mr * sre[c] - mi * sim[c];
                aim += mr * sim[c] + mi * sre[c];
            }
            psi[2 * (base + off[r])] = are;
            psi[2 * (base + off[r]) + 1] = aim;
        }
    }
    return 0;
}

/* apply_gate (state.hpp:149-156) on one pure state, in place. */
int qo_apply_gate(double *psi, int n, const qo_gate *g) {
    double m[32];
    const int k = qo_gate_matrix(g, m);
    if (k < 0 || k != g->nwires) return -1;
    return qo_apply_matrix(psi, n, m, k, g->wires, g->ncontrols, g->controls, 0);
}

/* Circuit::forward (circuit.hpp:121-153). out holds max(rows,1) states. With
 * rows > 0 each row binds encode slots in circuit order from data. */
int qo_forward(int n, const qo_gate *gates, int ngates, const double *init, const double *data, int rows, int slots,
               double *out) {
    const uint64_t dim = 1ull << n;
    int enc = 0;
    for (int i = 0; i < ngates; ++i)
        if (gates[i].encode) enc += gates[i].nparams;
    if (rows == 0 && enc != 0) return -2;
    if (rows > 0 && slots != enc) return -2;
    const int nrows = rows > 0 ? rows : 1;
    for (int r = 0; r < nrows; ++r) {
        double *psi = out + (size_t)r * 2 * dim;
        if (init) memcpy(psi, init, sizeof(double) * 2 * dim);
        else {
            memset(psi, 0, sizeof(double) * 2 * dim);
            psi[0] = 1.0;
        }
        int cursor = 0;
        for (int i = 0; i < ngates; ++i) {
            qo_gate g = gates[i];
            if (g.encode && rows > 0)
                for (int p = 0; p < g.nparams; ++p) g.params[p] = data[(size_t)r * slots + cursor++];
            int rc = qo_apply_gate(psi, n, &g);
            if (rc) return rc;
        }
    }
    return 0;
}

/* expectation_one (circuit.hpp:248-262): <psi| P |psi> with P applied
 * wire by wire through the strided kernel, then the conjugate-linear dot. */
int qo_expectation(int n, const double *psi, int nw, const int32_t *wires, const char *basis, double *out,
                   double *imag_out) {
    const uint64_t dim = 1ull << n;
    double *phi = (double *)malloc(sizeof(double) * 2 * dim);
    if (!phi) return -3;
    memcpy(phi, psi, sizeof(double) * 2 * dim);
    for (int i = 0; i < nw; ++i) {
        const double *P = basis[i] == 'x' ? QO_X : basis[i] == 'y' ? QO_Y : QO_Z;
        qo_apply_matrix(phi, n, P, 1, &wires[i], 0, NULL, 0);
    }
    double re = 0.0, im = 0.0;
    for (uint64_t j = 0; j < dim; ++j) { /* conj(psi_j) * phi_j */
        re += psi[2 * j] * phi[2 * j] + psi[2 * j + 1] * phi[2 * j + 1];
        im += psi[2 * j] * phi[2 * j + 1] - psi[2 * j + 1] * phi[2 * j];
    }
    free(phi);
    *out = re;
    if (imag_out) *imag_out = im;
    return fabs(im) < 1e-10 ? 0 : -4; /* circuit.hpp:261 */
}

/* marginal_probabilities (circuit.hpp:182-198), pure states. */
int qo_marginal_probabilities(int n, const double *psi, int k, const int32_t *wires, double *probs) {
    const uint64_t dim = 1ull << n;
    memset(probs, 0, sizeof(double) * ((size_t)1 << k));
    for (uint64_t idx = 0; idx < dim; ++idx) {
        uint64_t o = 0;
        for (int i = 0; i < k; ++i) o = (o << 1) | ((idx >> (n - 1 - wires[i])) & 1ull);
        probs[o] += psi[2 * idx] * psi[2 * idx] + psi[2 * idx + 1] * psi[2 * idx + 1];
    }
    return 0;
}

/* measure (circuit.hpp:217-236): CDF sampling with rng.uniform() * total and
 * lower_bound; counts indexed by outcome. */
int qo_measure_counts(const double *probs, int k, int shots, qo_rng *rng, uint64_t *counts) {
    const size_t np = (size_t)1 << k;
    double *cdf = (double *)malloc(sizeof(double) * np);
    if (!cdf) return -3;
    double acc = 0.0;
    for (size_t i = 0; i < np; ++i) {
        acc += probs[i];
        cdf[i] = acc;
    }
    memset(counts, 0, sizeof(uint64_t) * np);
    for (int s = 0; s < shots; ++s) {
        const double u = qo_rng_uniform(rng) * acc;
        size_t lo = 0, hi = np; /* lower_bound: first cdf[i] >= u */
        while (lo < hi) {
            size_t mid = (lo + hi) / 2;
            if (cdf[mid] < u) lo = mid + 1;
            else hi = mid;
        }
        counts[lo < np ? lo : np - 1] += 1;
    }
    free(cdf);
    return 0;
}

/* ||psi||^2 (FP64, sequential). */
double qo_norm2(int n, const double *psi) {
    const uint64_t dim = 1ull << n;
    double s = 0.0;
    for (uint64_t j = 0; j < 2 * dim; ++j) s += psi[j] * psi[j];
    return s;
}

size_t qo_gate_sizeof(void) { return sizeof(qo_gate); }

/* ------------------------------------------ threaded helpers (test infra) */
/* Full-size parity fixtures (tests/golden/make_fullsize.py) and the bench's
 * reference arm need the oracle at 30 qubits: the same arithmetic as above,
 * with the independent work split over host threads. Pinned against the
 * single-threaded restatement and oracle/_ref in tests/test_oracle.py. */
#include <pthread.h>

typedef struct {
    void (*fn)(void *arg, uint64_t b, uint64_t e);
    void *arg;
    uint64_t b, e;
} qo_job;

static void *qo_job_run(void *p) {
    qo_job *j = (qo_job *)p;
    j->fn(j->arg, j->b, j->e);
    return NULL;
}

/* runs fn over [0, total) split into nthreads contiguous ranges (multiples of
 * `grain`) */
static void qo_parallel(uint64_t total, uint64_t grain, int nthreads, void (*fn)(void *, uint64_t, uint64_t),
                        void *arg) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    uint64_t units = (total + grain - 1) / grain;
    if ((uint64_t)nthreads > units) nthreads = units ? (int)units : 1;
    if (nthreads == 1) {
        fn(arg, 0, total);
        return;
    }
    pthread_t th[256];
    qo_job jobs[256];
    const uint64_t per = (units + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        uint64_t b = (uint64_t)t * per * grain, e = b + per * grain;
        if (b > total) b = total;
        if (e > total) e = total;
        jobs[t] = (qo_job){fn, arg, b, e};
        pthread_create(&th[t], NULL, qo_job_run, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Rng(seed, label).normal() draws [offset, offset + count) (offset even):
 * counter-based like rng.hpp:43 -- pair j uses counters 2j+1, 2j+2 -- so
 * threads reproduce the sequential stream; returns 1 if the u1 == 0
 * rejection of rng.hpp:59 (p = 2^-53 per pair) was met, in which case the
 * caller must fall back to qo_rng_draw. */
typedef struct {
    uint64_t key, c0, count;
    double *out;
    int rejected;
} qo_fill_arg;

static void qo_fill_normal_part(void *p, uint64_t b, uint64_t e) {
    qo_fill_arg *a = (qo_fill_arg *)p;
    for (uint64_t j = b; j < e; ++j) {
        const double u1 = (double)(qo_mix(a->key + 0x9e3779b97f4a7c15ull * (a->c0 + 2 * j + 1)) >> 11) * 0x1.0p-53;
        const double u2 = (double)(qo_mix(a->key + 0x9e3779b97f4a7c15ull * (a->c0 + 2 * j + 2)) >> 11) * 0x1.0p-53;
        if (u1 == 0.0) {
            a->rejected = 1;
            return;
        }
        const double rad = sqrt(-2.0 * log(u1));
        a->out[2 * j] = rad * cos(2.0 * 3.141592653589793 * u2);
        if (2 * j + 1 < a->count) a->out[2 * j + 1] = rad * sin(2.0 * 3.141592653589793 * u2);
    }
}

int qo_rng_fill_normal(uint64_t seed, const char *label, uint64_t offset, uint64_t count, double *out, int nthreads) {
    if (offset % 2) return -1;
    qo_rng r;
    qo_rng_init(&r, seed, label);
    qo_fill_arg a = {r.key, offset, count, out, 0};
    qo_parallel((count + 1) / 2, 1 << 14, nthreads, qo_fill_normal_part, &a);
    return a.rejected;
}

/* apply_matrix_strided (state.hpp:111-143) with the group bases split over
 * threads: every base belongs to one thread, so the groups stay disjoint. */
typedef struct {
    double *psi;
    const double *m;
    int gs;
    uint64_t tmask, cmask, off[32];
    int zoc;
} qo_apply_arg;

static void qo_apply_part(void *p, uint64_t b0, uint64_t b1) {
    qo_apply_arg *a = (qo_apply_arg *)p;
    double sre[32], sim[32];
    const int gs = a->gs;
    for (uint64_t base = b0; base < b1; ++base) {
        if (base & a->tmask) continue;
        if ((base & a->cmask) != a->cmask) {
            if (a->zoc)
                for (int j = 0; j < gs; ++j) a->psi[2 * (base + a->off[j])] = a->psi[2 * (base + a->off[j]) + 1] = 0.0;
            continue;
        }
        for (int j = 0; j < gs; ++j) {
            sre[j] = a->psi[2 * (base + a->off[j])];
            sim[j] = a->psi[2 * (base + a->off[j]) + 1];
        }
        for (int r = 0; r < gs; ++r) {
            double are = 0.0, aim = 0.0;
            for (int c = 0; c < gs; ++c) {
                const double mr = a->m[2 * (r * gs + c)], mi = a->m[2 * (r * gs + c) + 1];
                are += mr * sre[c] - mi * sim[c];
                aim += mr * sim[c] + mi * sre[c];
            }
            a->psi[2 * (base + a->off[r])] = are;
            a->psi[2 * (base + a->off[r]) + 1] = aim;
        }
    }
}

int qo_apply_matrix_mt(double *psi, int n, const double *m, int k, const int32_t *wires, int nctl,
                       const int32_t *ctls, int zero_off_control, int nthreads) {
    if (k < 1 || k > 5) return -1;
    for (int i = 0; i < k; ++i)
        if (wires[i] < 0 || wires[i] >= n) return -1;
    for (int i = 0; i < nctl; ++i)
        if (ctls[i] < 0 || ctls[i] >= n) return -1;
    qo_apply_arg a;
    memset(&a, 0, sizeof a);
    a.psi = psi;
    a.m = m;
    a.gs = 1 << k;
    a.zoc = zero_off_control;
    for (int i = 0; i < k; ++i) a.tmask |= 1ull << (n - 1 - wires[i]);
    for (int i = 0; i < nctl; ++i) a.cmask |= 1ull << (n - 1 - ctls[i]);
    for (int j = 0; j < a.gs; ++j)
        for (int i = 0; i < k; ++i)
            if ((j >> (k - 1 - i)) & 1) a.off[j] |= 1ull << (n - 1 - wires[i]);
    qo_parallel(1ull << n, 1 << 12, nthreads, qo_apply_part, &a);
    return 0;
}

/* Circuit::forward without data (circuit.hpp:124-128) on psi, in place. */
int qo_forward_mt(int n, const qo_gate *gates, int ngates, double *psi, int nthreads) {
    for (int i = 0; i < ngates; ++i) {
        double m[32];
        const int k = qo_gate_matrix(&gates[i], m);
        if (k < 0 || k != gates[i].nwires) return -1;
        int rc = qo_apply_matrix_mt(psi, n, m, k, gates[i].wires, gates[i].ncontrols, gates[i].controls, 0, nthreads);
        if (rc) return rc;
    }
    return 0;
}

/* Full-state digest (tests/golden/make_fullsize.py, tests/test_gpu_fullsize.py):
 * the 2^n amplitudes in `nblocks` equal contiguous blocks; per block
 * out[3b] = sum |a|^2 and out[3b+1], out[3b+2] = sum a_i w_i (re, im) with
 * pseudo-random weights w_i = (+-1) + i(+-1) from the top two bits of
 * i * 0x9e3779b97f4a7c15 (i = the GLOBAL index); z[0] = sum |a|^2,
 * z[1 + w] = sum |a|^2 (-1)^{bit of wire w} (wire 0 = MSB), z[n + 1] = the
 * same for Z_0 Z_{n-1}. Sequential FP64 sums inside each block. */
typedef struct {
    const double *psi;
    int n;
    uint64_t bsize;
    double *out;
} qo_digest_arg;

static void qo_digest_part(void *p, uint64_t b0, uint64_t b1) {
    qo_digest_arg *a = (qo_digest_arg *)p;
    for (uint64_t b = b0; b < b1; ++b) {
        double s2 = 0, wr = 0, wi = 0;
        for (uint64_t i = b * a->bsize; i < (b + 1) * a->bsize; ++i) {
            const double re = a->psi[2 * i], im = a->psi[2 * i + 1];
            const uint64_t h = i * 0x9e3779b97f4a7c15ull;
            const double sr = (h >> 63) ? -1.0 : 1.0, si = ((h >> 62) & 1) ? -1.0 : 1.0;
            s2 += re * re + im * im;
            /* (re + i im)(sr + i si) */
            wr += re * sr - im * si;
            wi += re * si + im * sr;
        }
        a->out[3 * b] = s2;
        a->out[3 * b + 1] = wr;
        a->out[3 * b + 2] = wi;
    }
}

typedef struct {
    const double *psi;
    int n;
    double *acc; /* [thread-chunk][n + 2] */
    uint64_t chunk;
} qo_z_arg;

static void qo_z_part(void *p, uint64_t c0, uint64_t c1) {
    qo_z_arg *a = (qo_z_arg *)p;
    const int n = a->n;
    for (uint64_t c = c0; c < c1; ++c) {
        double *z = a->acc + c * (n + 2);
        for (int k = 0; k < n + 2; ++k) z[k] = 0;
        for (uint64_t i = c * a->chunk; i < (c + 1) * a->chunk; ++i) {
            const double p2 = a->psi[2 * i] * a->psi[2 * i] + a->psi[2 * i + 1] * a->psi[2 * i + 1];
            z[0] += p2;
            for (int w = 0; w < n; ++w) z[1 + w] += ((i >> (n - 1 - w)) & 1) ? -p2 : p2;
            z[n + 1] += (((i >> (n - 1)) ^ i) & 1) ? -p2 : p2;
        }
    }
}

int qo_digest(int n, const double *psi, int nblocks, double *blocks, double *z, int nthreads) {
    const uint64_t dim = 1ull << n;
    if (nblocks < 1 || dim % (uint64_t)nblocks) return -1;
    qo_digest_arg a = {psi, n, dim / (uint64_t)nblocks, blocks};
    qo_parallel((uint64_t)nblocks, 1, nthreads, qo_digest_part, &a);
    const uint64_t nch = dim >= 4096 ? 4096 : 1;
    double *acc = (double *)malloc(sizeof(double) * nch * (n + 2));
    if (!acc) return -3;
    qo_z_arg za = {psi, n, acc, dim / nch};
    qo_parallel(nch, 1, nthreads, qo_z_part, &za);
    for (int k = 0; k < n + 2; ++k) {
        double s = 0;
        for (uint64_t c = 0; c < nch; ++c) s += acc[c * (n + 2) + k];
        z[k] = s;
    }
    free(acc);
    return 0;
}
