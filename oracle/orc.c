/* orc.c -- CPU ORACLE for the halo feature pipeline of arXiv 2410.22697.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code with
 * the CUDA library.  See orc.h for the API and DESIGN.md §Readings for every
 * reading R#n of a point the paper leaves open.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no -ffast-math: fp32 must stay IEEE round-to-nearest with denormals, R#12).
 */
#include "orc.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- Philox */
/* Philox4x32-10, Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 * easy as 1, 2, 3", SC'11: 10 rounds of
 *   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 *   c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0),  key += (W0, W1) between rounds. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void seed_key(uint64_t seed, uint32_t key[2]) {
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32);
}

/* Feature stream (R#4): ctr = (node, col/4, 0, 3), key = feat_seed;
 * value = ((out[col%4] >> 8) - 2^23) * 2^-23, exact in fp32, in [-1, 1). */
void orc_feature_row(int64_t node, int32_t dim, uint64_t feat_seed, float* out) {
    uint32_t key[2];
    seed_key(feat_seed, key);
    for (int32_t c = 0; c < dim; c++) {
        uint32_t ctr[4] = {(uint32_t)node, (uint32_t)(c / 4), 0u, 3u}, o[4];
        orc_philox4x32_10(ctr, key, o);
        int32_t q = (int32_t)(o[c % 4] >> 8) - (1 << 23);
        out[c] = (float)q * (1.0f / 8388608.0f);
    }
}

/* R#5: r = floor(u * (t+1) / 2^32), a value in [0, t]. */
uint32_t orc_range(uint32_t u, uint32_t t_plus_1) {
    return (uint32_t)(((uint64_t)u * (uint64_t)t_plus_1) >> 32);
}

/* R#6, Floyd's algorithm for a k-subset of {0..d-1}:
 *   for j = 0..k-1: t = d-k+j; draw r in [0, t];
 *                   pos_j = (r already chosen) ? t : r.                  */
void orc_floyd(int64_t d, int32_t k, const uint32_t* r, int64_t* pos) {
    for (int32_t j = 0; j < k; j++) {
        int64_t t = d - k + j;
        int64_t cand = (int64_t)r[j];
        int seen = 0;
        for (int32_t i = 0; i < j; i++)
            if (pos[i] == cand) seen = 1;
        pos[j] = seen ? t : cand;
    }
}

/* Eq.1 with initial S_E = 1 (R#13): alpha = ((1*g)*g)...*g, Delta times, in fp32. */
float orc_alpha_default(float gamma, int32_t delta) {
    float a = 1.0f;
    for (int32_t i = 0; i < delta; i++) a = a * gamma;
    return a;
}

/* ---------------------------------------------------------------- types */
struct orc_world {
    int32_t dense;     /* NEXT-1 dense S_A: every non-local node is scorable (set before the partitions) */
    int32_t P;
    int64_t n_global;
    int64_t* bounds;   /* P+1 */
    int32_t D;
    uint64_t feat_seed;
    orc_part** parts;  /* registered by orc_part_new */
};

struct orc_part {
    orc_world* w;
    int32_t p;
    int64_t lo, hi, n_local;
    int64_t* indptr;   /* n_local+1 */
    int32_t* cols;     /* global ids */
    int32_t* train;
    int64_t n_train;
    int32_t* halo;     /* V_p^h sorted ascending */
    int32_t* deg_in;
    int64_t n_h;
    int64_t n_h_true;  /* |V_p^h| (halo nodes with deg_in > 0): the basis of |BUF| even when dense */
    float* table;      /* local KVStore: n_local x D */
    /* prefetcher */
    int ready;
    float gamma, alpha, theta_r;
    int32_t delta;
    int64_t cap;
    int32_t* node_of_slot;
    float* se;
    float* sa;
    int32_t* slot_of;
    float* rows;       /* cap x D */
    uint8_t* hitflag;  /* cap */
    /* epoch order cache */
    int64_t perm_epoch;
    int32_t* perm;
    /* last step */
    int32_t L;
    int64_t hop_size[9];
    int64_t* hop_off[8];
    int32_t* hop_cols[8];
    int64_t hop_edges[8];
    int32_t* F;
    int64_t F_cap;
    float* X;
    int64_t X_rows;
    int8_t* cls;
    int64_t counts[ORC_C_N];
    int64_t totals[4];
    int32_t expand_remote;  /* non-local frontier nodes sampled from their owner's CSR */
};

/* ---------------------------------------------------------------- helpers */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static int64_t bsearch_i32(const int32_t* arr, int64_t n, int32_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (arr[mid] < v) lo = mid + 1; else hi = mid;
    }
    return (lo < n && arr[lo] == v) ? lo : -1;
}

static int32_t owner_of(const orc_world* w, int64_t v) {
    for (int32_t q = 0; q < w->P; q++)
        if (v >= w->bounds[q] && v < w->bounds[q + 1]) return q;
    return -1;
}

/* KVStore / RPC: the feature row of node v, read from its owner's table. */
static void kv_fetch(const orc_world* w, int64_t v, float* out) {
    int32_t q = owner_of(w, v);
    const orc_part* o = w->parts[q];
    memcpy(out, o->table + (size_t)(v - o->lo) * (size_t)w->D, sizeof(float) * (size_t)w->D);
}

/* ---------------------------------------------------------------- world */
orc_world* orc_world_new(int32_t n_parts, int64_t n_global, const int64_t* bounds, int32_t feat_dim,
                         uint64_t feat_seed) {
    if (n_parts < 1 || n_global < 0 || n_global >= ((int64_t)1 << 31) || feat_dim < 0) return NULL;
    if (bounds[0] != 0 || bounds[n_parts] != n_global) return NULL;
    for (int32_t q = 0; q < n_parts; q++)
        if (bounds[q + 1] < bounds[q]) return NULL;
    orc_world* w = calloc(1, sizeof(*w));
    w->P = n_parts;
    w->n_global = n_global;
    w->bounds = malloc(sizeof(int64_t) * (size_t)(n_parts + 1));
    memcpy(w->bounds, bounds, sizeof(int64_t) * (size_t)(n_parts + 1));
    w->D = feat_dim;
    w->feat_seed = feat_seed;
    w->parts = calloc((size_t)n_parts, sizeof(orc_part*));
    return w;
}

void orc_world_free(orc_world* w) {
    if (!w) return;
    free(w->bounds);
    free(w->parts);
    free(w);
}

/* ---------------------------------------------------------------- partition (O1) */
orc_part* orc_part_new(orc_world* w, int32_t part_id, const int64_t* indptr, const int32_t* cols,
                       const int32_t* train_ids, int64_t n_train) {
    if (!w || part_id < 0 || part_id >= w->P || w->parts[part_id]) return NULL;
    int64_t lo = w->bounds[part_id], hi = w->bounds[part_id + 1], nl = hi - lo;
    if (indptr[0] != 0) return NULL;
    for (int64_t r = 0; r < nl; r++) {
        if (indptr[r + 1] < indptr[r]) return NULL;
        for (int64_t e = indptr[r]; e < indptr[r + 1]; e++) {
            int32_t c = cols[e];
            if (c < 0 || c >= w->n_global || c == lo + r) return NULL;       /* simple graph */
            if (e > indptr[r] && cols[e - 1] >= c) return NULL;             /* rows ascending, no dups */
        }
    }
    for (int64_t i = 0; i < n_train; i++) {
        if (train_ids[i] < lo || train_ids[i] >= hi) return NULL;
        if (i > 0 && train_ids[i - 1] >= train_ids[i]) return NULL;
    }
    orc_part* p = calloc(1, sizeof(*p));
    p->w = w;
    p->p = part_id;
    p->lo = lo;
    p->hi = hi;
    p->n_local = nl;
    int64_t nnz = indptr[nl];
    p->indptr = malloc(sizeof(int64_t) * (size_t)(nl + 1));
    memcpy(p->indptr, indptr, sizeof(int64_t) * (size_t)(nl + 1));
    p->cols = malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
    memcpy(p->cols, cols, sizeof(int32_t) * (size_t)nnz);
    p->n_train = n_train;
    p->train = malloc(sizeof(int32_t) * (size_t)(n_train ? n_train : 1));
    memcpy(p->train, train_ids, sizeof(int32_t) * (size_t)n_train);

    /* V_p^h = {v not in V_p^l : v in N(u), u in V_p^l} (R#9), sorted.  Dense scores
       (NEXT-1, P:228's O(|V|) S_A): the scorable set is every non-local node. */
    int64_t m = 0, nh = 0;
    int32_t* tmp;
    if (w->dense) {
        tmp = malloc(sizeof(int32_t) * (size_t)(w->n_global - nl ? w->n_global - nl : 1));
        for (int64_t v = 0; v < w->n_global; v++)
            if (v < lo || v >= hi) tmp[nh++] = (int32_t)v;
    } else {
        tmp = malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
        for (int64_t e = 0; e < nnz; e++)
            if (cols[e] < lo || cols[e] >= hi) tmp[m++] = cols[e];
        qsort(tmp, (size_t)m, sizeof(int32_t), cmp_i32);
        for (int64_t i = 0; i < m; i++)
            if (i == 0 || tmp[i] != tmp[i - 1]) tmp[nh++] = tmp[i];
    }
    p->n_h = nh;
    p->halo = malloc(sizeof(int32_t) * (size_t)(nh ? nh : 1));
    memcpy(p->halo, tmp, sizeof(int32_t) * (size_t)nh);
    free(tmp);
    /* deg_in[h] = |N(h) ∩ V_p^l| = occurrences of h among local rows (R#10). */
    p->deg_in = calloc((size_t)(nh ? nh : 1), sizeof(int32_t));
    for (int64_t e = 0; e < nnz; e++)
        if (cols[e] < lo || cols[e] >= hi) p->deg_in[bsearch_i32(p->halo, nh, cols[e])]++;
    p->n_h_true = 0;
    for (int64_t h = 0; h < nh; h++) p->n_h_true += p->deg_in[h] > 0;

    /* local KVStore */
    int32_t D = w->D;
    p->table = malloc(sizeof(float) * (size_t)(nl ? nl : 1) * (size_t)(D ? D : 1));
    for (int64_t r = 0; r < nl; r++) orc_feature_row(lo + r, D, w->feat_seed, p->table + (size_t)r * (size_t)D);
    p->perm_epoch = -1;
    w->parts[part_id] = p;
    return p;
}

static void free_step(orc_part* p) {
    for (int i = 0; i < 8; i++) {
        free(p->hop_off[i]);
        free(p->hop_cols[i]);
        p->hop_off[i] = NULL;
        p->hop_cols[i] = NULL;
    }
}

void orc_part_free(orc_part* p) {
    if (!p) return;
    if (p->w && p->w->parts[p->p] == p) p->w->parts[p->p] = NULL;
    free(p->indptr); free(p->cols); free(p->train); free(p->halo); free(p->deg_in); free(p->table);
    free(p->node_of_slot); free(p->se); free(p->sa); free(p->slot_of); free(p->rows); free(p->hitflag);
    free(p->perm); free(p->F); free(p->X); free(p->cls);
    free_step(p);
    free(p);
}

int64_t orc_n_local(const orc_part* p) { return p->n_local; }
int64_t orc_n_halo(const orc_part* p) { return p->n_h; }
int64_t orc_capacity(const orc_part* p) { return p->cap; }

void orc_halo(const orc_part* p, int32_t* halo_ids, int32_t* deg_in) {
    if (halo_ids) memcpy(halo_ids, p->halo, sizeof(int32_t) * (size_t)p->n_h);
    if (deg_in) memcpy(deg_in, p->deg_in, sizeof(int32_t) * (size_t)p->n_h);
}

/* ---------------------------------------------------------------- INITIALIZE_PREFETCHER (O3) */
typedef struct { int32_t deg, id; int64_t h; } rank_item;

static int cmp_rank(const void* a, const void* b) {
    const rank_item* x = a; const rank_item* y = b;
    if (x->deg != y->deg) return x->deg > y->deg ? -1 : 1;       /* degree desc */
    return (x->id > y->id) - (x->id < y->id);                    /* id asc */
}

int orc_buffer_init(orc_part* p, float gamma, float alpha, float theta_r, int32_t delta, uint32_t f_bp) {
    if (!(gamma > 0.0f && gamma <= 1.0f) || !(alpha >= 0.0f) || isinf(alpha) || isnan(theta_r) ||
        delta < 0 || f_bp > 10000u)
        return -1;
    for (int32_t q = 0; q < p->w->P; q++)
        if (!p->w->parts[q]) return -1;   /* every owner's KVStore must exist for the init RPC */
    p->gamma = gamma; p->alpha = alpha; p->theta_r = theta_r; p->delta = delta;
    /* |BUF| = ceil(f * |V_p^h|) in integer basis points (R#11); the true halo, also when dense */
    int64_t nh = p->n_h;
    p->cap = ((int64_t)f_bp * p->n_h_true + 9999) / 10000;
    free(p->node_of_slot); free(p->se); free(p->sa); free(p->slot_of); free(p->rows); free(p->hitflag);
    int64_t cap = p->cap, D = p->w->D;
    p->node_of_slot = malloc(sizeof(int32_t) * (size_t)(cap ? cap : 1));
    p->se = malloc(sizeof(float) * (size_t)(cap ? cap : 1));
    p->hitflag = calloc((size_t)(cap ? cap : 1), 1);
    p->rows = malloc(sizeof(float) * (size_t)(cap ? cap : 1) * (size_t)(D ? D : 1));
    p->sa = malloc(sizeof(float) * (size_t)(nh ? nh : 1));
    p->slot_of = malloc(sizeof(int32_t) * (size_t)(nh ? nh : 1));
    /* top-f halo nodes by degree (R#10): order (deg_in desc, id asc) */
    rank_item* it = malloc(sizeof(rank_item) * (size_t)(nh ? nh : 1));
    for (int64_t h = 0; h < nh; h++) { it[h].deg = p->deg_in[h]; it[h].id = p->halo[h]; it[h].h = h; }
    qsort(it, (size_t)nh, sizeof(rank_item), cmp_rank);
    /* S_A[m] = 0 for non-buffered halo nodes */
    for (int64_t h = 0; h < nh; h++) { p->sa[h] = 0.0f; p->slot_of[h] = -1; }
    for (int64_t s = 0; s < cap; s++) {
        int64_t h = it[s].h;
        p->node_of_slot[s] = p->halo[h];
        p->slot_of[h] = (int32_t)s;
        p->se[s] = 1.0f;      /* S_E[n] = 1 */
        p->sa[h] = -1.0f;     /* S_A[n] = -1 */
        kv_fetch(p->w, p->halo[h], p->rows + (size_t)s * (size_t)D);   /* "RPC" */
    }
    free(it);
    memset(p->totals, 0, sizeof(p->totals));
    p->totals[3] = cap;
    p->ready = 1;
    return 0;
}

/* ---------------------------------------------------------------- epoch order (O5, R#8) */
typedef struct { uint64_t key; int32_t id; } perm_item;

static int cmp_perm(const void* a, const void* b) {
    const perm_item* x = a; const perm_item* y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

void orc_epoch_perm(const orc_part* p, uint64_t run_seed, uint64_t epoch, int32_t* out) {
    uint32_t key[2];
    seed_key(run_seed, key);
    perm_item* it = malloc(sizeof(perm_item) * (size_t)(p->n_train ? p->n_train : 1));
    for (int64_t i = 0; i < p->n_train; i++) {
        uint32_t ctr[4] = {(uint32_t)p->train[i], (uint32_t)epoch, 0u, ((uint32_t)p->p << 8) | 2u}, o[4];
        orc_philox4x32_10(ctr, key, o);
        it[i].key = ((uint64_t)o[0] << 32) | o[1];
        it[i].id = p->train[i];
    }
    qsort(it, (size_t)p->n_train, sizeof(perm_item), cmp_perm);
    for (int64_t i = 0; i < p->n_train; i++) out[i] = it[i].id;
    free(it);
}

/* ---------------------------------------------------------------- EVICT_AND_REPLACE helpers (O12) */
typedef struct { float se; int32_t id; int64_t s; } ev_item;
typedef struct { float sa; int32_t deg; int32_t id; int64_t h; } rp_item;

static int cmp_ev(const void* a, const void* b) {             /* (S_E asc, id asc) */
    const ev_item* x = a; const ev_item* y = b;
    if (x->se != y->se) return x->se < y->se ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int cmp_rp(const void* a, const void* b) {             /* (S_A desc, deg_in desc, id asc) */
    const rp_item* x = a; const rp_item* y = b;
    if (x->sa != y->sa) return x->sa > y->sa ? -1 : 1;
    if (x->deg != y->deg) return x->deg > y->deg ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* EVICT_AND_REPLACE (Alg.2 l.25-34) with the swap of P:224:
 *   E = buffered slots with S_E < alpha, by (S_E asc, id asc)          (R#16)
 *   R = halo nodes not buffered with S_A >= theta_r,
 *       by (S_A desc, deg_in desc, id asc)                              (R#17, R#18)
 *   k = min(|E|, |R|)  -- "exactly equal ... constant buffer size"     (R#19)
 *   pair i: s = E[i], e = node in s, r = R[i]:
 *       S_A[e] <- S_E[s]; BUF[s] <- r; S_E[s] <- S_A[r]; S_A[r] <- -1   (R#20, R#21)
 * Returns k; the pair lists (node ids / slots) are written if non-NULL. */
int64_t orc_evict_and_replace(int64_t cap, int64_t n_h, int32_t* node_of_slot, float* se, float* sa,
                              int32_t* slot_of, const int32_t* halo, const int32_t* deg_in, float alpha,
                              float theta_r, int32_t* evicted_out, int32_t* replaced_out, int32_t* slots_out) {
    ev_item* E = malloc(sizeof(ev_item) * (size_t)(cap ? cap : 1));
    int64_t nE = 0;
    for (int64_t s = 0; s < cap; s++)
        if (se[s] < alpha) {                         /* S_E[n] < alpha */
            E[nE].se = se[s]; E[nE].id = node_of_slot[s]; E[nE].s = s; nE++;
        }
    rp_item* R = malloc(sizeof(rp_item) * (size_t)(n_h ? n_h : 1));
    int64_t nR = 0;
    for (int64_t h = 0; h < n_h; h++)
        if (slot_of[h] < 0 && sa[h] >= theta_r) {    /* "m = max(S_A) is not empty" */
            R[nR].sa = sa[h]; R[nR].deg = deg_in[h]; R[nR].id = halo[h]; R[nR].h = h; nR++;
        }
    qsort(E, (size_t)nE, sizeof(ev_item), cmp_ev);
    qsort(R, (size_t)nR, sizeof(rp_item), cmp_rp);
    int64_t k = nE < nR ? nE : nR;
    for (int64_t i = 0; i < k; i++) {
        int64_t s = E[i].s, r = R[i].h;
        int64_t e = bsearch_i32(halo, n_h, node_of_slot[s]);
        float se_old = se[s], sa_old_r = sa[r];
        if (evicted_out) evicted_out[i] = node_of_slot[s];
        if (replaced_out) replaced_out[i] = halo[r];
        if (slots_out) slots_out[i] = (int32_t)s;
        sa[e] = se_old;              /* evicted: S_A <- last S_E */
        slot_of[e] = -1;
        node_of_slot[s] = halo[r];   /* BUF[V^{h|e}] = V^{h|r} */
        slot_of[r] = (int32_t)s;
        se[s] = sa_old_r;            /* replacement: S_E <- last S_A */
        sa[r] = -1.0f;               /* S_A[m] = -1 */
    }
    free(E);
    free(R);
    return k;
}

static void ensure_F(orc_part* p, int64_t n) {
    if (n <= p->F_cap) return;
    int64_t c = p->F_cap ? p->F_cap : 1024;
    while (c < n) c *= 2;
    p->F = realloc(p->F, sizeof(int32_t) * (size_t)c);
    p->F_cap = c;
}

/* ---------------------------------------------------------------- PREFETCH_WITH_EVICTION */
int orc_step(orc_part* p, uint64_t run_seed, uint64_t step, const int32_t* fanouts, int32_t n_layers,
             int32_t batch, const int32_t* seeds, int32_t n_seeds) {
    if (!p->ready || step < 1 || n_layers < 1 || n_layers > 8) return -1;
    int32_t k_max = 1;
    for (int32_t l = 0; l < n_layers; l++) {
        if (fanouts[l] < 1) return -1;
        if (fanouts[l] > k_max) k_max = fanouts[l];
    }
    orc_world* w = p->w;
    const int32_t D = w->D;
    free_step(p);
    p->L = n_layers;

    /* seeds = this step's slice of the epoch order (R#8), or the given ids */
    int64_t n0;
    if (seeds) {
        if (n_seeds < 1) return -1;
        for (int32_t i = 0; i < n_seeds; i++)
            if (seeds[i] < p->lo || seeds[i] >= p->hi) return -1;
        ensure_F(p, n_seeds);
        memcpy(p->F, seeds, sizeof(int32_t) * (size_t)n_seeds);
        n0 = n_seeds;
    } else {
        if (batch < 1 || p->n_train < 1) return -1;
        int64_t nb = (p->n_train + batch - 1) / batch;
        int64_t e = (int64_t)((step - 1) / (uint64_t)nb), b = (int64_t)((step - 1) % (uint64_t)nb);
        if (p->perm_epoch != e) {
            free(p->perm);
            p->perm = malloc(sizeof(int32_t) * (size_t)p->n_train);
            orc_epoch_perm(p, run_seed, (uint64_t)e, p->perm);
            p->perm_epoch = e;
        }
        int64_t s0 = b * batch, s1 = s0 + batch < p->n_train ? s0 + batch : p->n_train;
        n0 = s1 - s0;
        ensure_F(p, n0);
        memcpy(p->F, p->perm + s0, sizeof(int32_t) * (size_t)n0);
    }
    /* seeds must be distinct */
    {
        int32_t* t = malloc(sizeof(int32_t) * (size_t)n0);
        memcpy(t, p->F, sizeof(int32_t) * (size_t)n0);
        qsort(t, (size_t)n0, sizeof(int32_t), cmp_i32);
        for (int64_t i = 1; i < n0; i++)
            if (t[i] == t[i - 1]) { free(t); return -1; }
        free(t);
    }

    /* Alg.2 l.1: NeighborSampler (R#1-#7).  Hop i draws k_i = fanouts[L-1-i]. */
    uint32_t key[2];
    seed_key(run_seed, key);
    int64_t nF = n0;
    p->hop_size[0] = nF;
    for (int32_t i = 0; i < n_layers; i++) {
        int32_t k = fanouts[n_layers - 1 - i];
        int64_t nFi = nF;
        int64_t* off = malloc(sizeof(int64_t) * (size_t)(nFi + 1));
        int64_t ecap = nFi * k + 1;
        int32_t* col = malloc(sizeof(int32_t) * (size_t)ecap);
        int64_t ne = 0;
        off[0] = 0;
        for (int64_t f = 0; f < nFi; f++) {
            int32_t x = p->F[f];
            /* the CSR row of x: local rows; with expand_remote (NEXT-1, DistDGL's sampling through the
               owner) also every other node, from the owning partition's rows */
            const orc_part* src = NULL;
            if (x >= p->lo && x < p->hi) src = p;     /* halo frontier nodes are leaves (R#1) */
            else if (p->expand_remote) src = w->parts[owner_of(w, x)];
            if (src) {
                int64_t row = x - src->lo, b0 = src->indptr[row], d = src->indptr[row + 1] - b0;
                if (d <= k) {                          /* d <= k: whole neighbourhood (R#3) */
                    for (int64_t j = 0; j < d; j++) col[ne++] = src->cols[b0 + j];
                } else {                               /* any fanout (the GPU library caps it at 32) */
                    uint32_t* r = malloc(sizeof(uint32_t) * (size_t)k_max);
                    int64_t* pos = malloc(sizeof(int64_t) * (size_t)k_max);
                    for (int32_t j = 0; j < k; j++) {
                        uint32_t ctr[4] = {(uint32_t)x, ((uint32_t)i << 16) | (uint32_t)j, (uint32_t)step,
                                           ((uint32_t)p->p << 8) | 1u}, o[4];
                        orc_philox4x32_10(ctr, key, o);
                        r[j] = orc_range(o[0], (uint32_t)(d - k + j + 1));
                    }
                    orc_floyd(d, k, r, pos);
                    for (int32_t j = 0; j < k; j++) col[ne++] = src->cols[b0 + pos[j]];
                    free(r);
                    free(pos);
                }
            }
            off[f + 1] = ne;
        }
        p->hop_off[i] = off;
        p->hop_cols[i] = col;
        p->hop_edges[i] = ne;
        /* F_{i+1} = F_i ++ (sorted unique(cols_i) \ F_i)   (R#7) */
        int32_t* u = malloc(sizeof(int32_t) * (size_t)(ne ? ne : 1));
        memcpy(u, col, sizeof(int32_t) * (size_t)ne);
        qsort(u, (size_t)ne, sizeof(int32_t), cmp_i32);
        int32_t* fs = malloc(sizeof(int32_t) * (size_t)(nFi ? nFi : 1));
        memcpy(fs, p->F, sizeof(int32_t) * (size_t)nFi);
        qsort(fs, (size_t)nFi, sizeof(int32_t), cmp_i32);
        ensure_F(p, nFi + ne);
        for (int64_t j = 0; j < ne; j++) {
            if (j > 0 && u[j] == u[j - 1]) continue;
            if (bsearch_i32(fs, nFi, u[j]) >= 0) continue;
            p->F[nF++] = u[j];
        }
        free(u);
        free(fs);
        p->hop_size[i + 1] = nF;
    }

    /* Alg.2 l.2-5: local / halo split, Hits = V^{h|s} ∩ BUF, Misses = V^{h|s} \ BUF. */
    free(p->cls);
    p->cls = malloc((size_t)(nF ? nF : 1));
    int64_t* miss_h = malloc(sizeof(int64_t) * (size_t)(nF ? nF : 1));
    int64_t n_local = 0, n_hit = 0, n_miss = 0, n_far = 0;
    memset(p->hitflag, 0, (size_t)(p->cap ? p->cap : 1));
    for (int64_t f = 0; f < nF; f++) {
        int32_t u = p->F[f];
        if (u >= p->lo && u < p->hi) { p->cls[f] = 0; n_local++; continue; }
        int64_t h = bsearch_i32(p->halo, p->n_h, u);     /* binary search into sorted V_p^h */
        if (h < 0) {
            if (!p->expand_remote) { free(miss_h); return -1; }   /* cannot happen: partition-local sampling */
            p->cls[f] = 3;          /* a remote node outside V_p^h: a miss, fetched, never buffered or scored */
            n_far++;
            continue;
        }
        int32_t s = p->slot_of[h];
        if (s >= 0) { p->cls[f] = 1; n_hit++; p->hitflag[s] = 1; }
        else { p->cls[f] = 2; miss_h[n_miss++] = h; }
    }

    /* Alg.2 l.6-9: S_E[n] = S_E[n] * gamma for every n in BUF not sampled. */
    for (int64_t s = 0; s < p->cap; s++)
        if (!p->hitflag[s]) p->se[s] = p->se[s] * p->gamma;

    /* Alg.2 l.10-11: B^l <- local rows; B^h <- BUF[Hits] (read before any refill). */
    if (nF > p->X_rows) {
        free(p->X);
        p->X = malloc(sizeof(float) * (size_t)nF * (size_t)(D ? D : 1));
        p->X_rows = nF;
    }
    for (int64_t f = 0; f < nF; f++) {
        int32_t u = p->F[f];
        float* dst = p->X + (size_t)f * (size_t)D;
        if (p->cls[f] == 0) memcpy(dst, p->table + (size_t)(u - p->lo) * (size_t)D, sizeof(float) * (size_t)D);
        else if (p->cls[f] == 1) {
            int32_t s = p->slot_of[bsearch_i32(p->halo, p->n_h, u)];
            memcpy(dst, p->rows + (size_t)s * (size_t)D, sizeof(float) * (size_t)D);
        }
    }

    /* Alg.2 l.21: S_A[n] = S_A[n] + 1 for every miss (every step, before eviction: R#15). */
    for (int64_t i = 0; i < n_miss; i++) p->sa[miss_h[i]] = p->sa[miss_h[i]] + 1.0f;

    /* Alg.2 l.12-19: every Delta steps (R#14) EVICT_AND_REPLACE (l.25-34) + combined fetch. */
    int64_t k = 0;
    if (p->delta > 0 && step % (uint64_t)p->delta == 0) {
        int64_t m = p->cap < p->n_h ? p->cap : p->n_h;
        int32_t* slots = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
        int32_t* repl = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
        k = orc_evict_and_replace(p->cap, p->n_h, p->node_of_slot, p->se, p->sa, p->slot_of, p->halo,
                                  p->deg_in, p->alpha, p->theta_r, NULL, repl, slots);
        for (int64_t i = 0; i < k; i++)   /* Update BUF with F[V^{h|r}] */
            kv_fetch(w, repl[i], p->rows + (size_t)slots[i] * (size_t)D);
        free(slots);
        free(repl);
    }

    /* Alg.2 l.22 / l.18: B^h <- fetched features of Misses. */
    for (int64_t f = 0; f < nF; f++)
        if (p->cls[f] >= 2) kv_fetch(w, p->F[f], p->X + (size_t)f * (size_t)D);
    free(miss_h);

    p->counts[ORC_C_NODES] = nF;
    p->counts[ORC_C_LOCAL] = n_local;
    p->counts[ORC_C_HIT] = n_hit;
    p->counts[ORC_C_MISS] = n_miss + n_far;
    p->counts[ORC_C_EVICTED] = k;
    p->counts[ORC_C_REFILLED] = k;
    p->counts[ORC_C_ROWS_FETCHED] = n_miss + n_far + k;
    p->totals[0] += n_hit;
    p->totals[1] += n_miss + n_far;
    p->totals[2] += k;
    return 0;
}

void orc_set_expand_remote(orc_part* p, int32_t on) { p->expand_remote = on ? 1 : 0; }
void orc_world_set_dense(orc_world* w, int32_t on) { w->dense = on ? 1 : 0; }

/* ---------------------------------------------------------------- getters */
void orc_counts(const orc_part* p, int64_t* out) { memcpy(out, p->counts, sizeof(p->counts)); }
int64_t orc_hop_size(const orc_part* p, int32_t hop) { return (hop >= 0 && hop <= p->L) ? p->hop_size[hop] : -1; }
int64_t orc_hop_edges(const orc_part* p, int32_t hop) { return (hop >= 0 && hop < p->L) ? p->hop_edges[hop] : -1; }
void orc_frontier(const orc_part* p, int32_t* out) { memcpy(out, p->F, sizeof(int32_t) * (size_t)p->hop_size[p->L]); }

void orc_hop_block(const orc_part* p, int32_t hop, int64_t* offsets, int32_t* cols) {
    if (offsets) memcpy(offsets, p->hop_off[hop], sizeof(int64_t) * (size_t)(p->hop_size[hop] + 1));
    if (cols) memcpy(cols, p->hop_cols[hop], sizeof(int32_t) * (size_t)p->hop_edges[hop]);
}

void orc_features_out(const orc_part* p, float* out) {
    memcpy(out, p->X, sizeof(float) * (size_t)p->hop_size[p->L] * (size_t)p->w->D);
}

void orc_classes(const orc_part* p, int8_t* out) { memcpy(out, p->cls, (size_t)p->hop_size[p->L]); }

void orc_buffer_state(const orc_part* p, int32_t* node_of_slot, float* se, float* sa, int32_t* slot_of, float* rows) {
    if (node_of_slot) memcpy(node_of_slot, p->node_of_slot, sizeof(int32_t) * (size_t)p->cap);
    if (se) memcpy(se, p->se, sizeof(float) * (size_t)p->cap);
    if (sa) memcpy(sa, p->sa, sizeof(float) * (size_t)p->n_h);
    if (slot_of) memcpy(slot_of, p->slot_of, sizeof(int32_t) * (size_t)p->n_h);
    if (rows) memcpy(rows, p->rows, sizeof(float) * (size_t)p->cap * (size_t)p->w->D);
}

void orc_totals(const orc_part* p, int64_t* out4) { memcpy(out4, p->totals, sizeof(p->totals)); }
