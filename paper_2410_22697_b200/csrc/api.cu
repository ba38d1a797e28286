// api.cu -- the C ABI of include/mgnn.h: context, partition load, buffer
// init, window arenas and the three per-window calls.  Host code only
// marshals sizes/pointers and launches the kernels of sample.cu, gather.cu,
// score.cu, sort.cu and load.cu; every step of the path runs on the GPU.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mgnn.h"
#include "ctx.h"
#include "launch.h"

namespace mgnn {
static std::atomic<long long> g_launches{0};
static const bool g_debug_sync = [] {
    const char* e = getenv("MGNN_DEBUG_SYNC");
    return e && e[0] == '1';
}();
struct ProfRec {
    const char* who;
    cudaEvent_t a, b;
    cudaStream_t s;
};
static bool g_kprof = false;
static std::vector<ProfRec> g_kprof_recs;
static std::vector<std::pair<cudaStream_t, cudaEvent_t>> g_kprof_last;

void count_launches(long long n, const char* who, cudaStream_t s) {
    g_launches.fetch_add(n, std::memory_order_relaxed);
    if (g_debug_sync) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) fprintf(stderr, "[mgnn] %s failed: %s\n", who, cudaGetErrorString(e));
    }
    if (g_kprof) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, s);
        for (auto& pl : g_kprof_last)
            if (pl.first == s) {
                g_kprof_recs.push_back(ProfRec{who, pl.second, e, s});
                pl.second = e;
                return;
            }
        g_kprof_last.emplace_back(s, e);
    }
}
long long launches_total() { return g_launches.load(); }

extern thread_local int t_sm_limit;          // partition.cu: set while a call runs on an SM partition
int num_sms() {
    if (t_sm_limit > 0) return t_sm_limit;
    static std::atomic<int> cache[64];            // 0 = not yet queried
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
    if (dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
    if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

cudaError_t ensure_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> have;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    int& cur = have[{dev, func}];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("MGNN_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace mgnn


using namespace mgnn;
using namespace mgnn::host;

namespace mgnn {
namespace host {

mgnn_status fail(mgnn_ctx c, mgnn_status st, const std::string& msg) {
    if (c) {
        c->err = msg;
        if (st == MGNN_ECUDA) c->sticky = st;
    }
    return st;
}

void fill_partdev(const mgnn_ctx_s* c, const Part& p, PartDev* d) {
    memset(d, 0, sizeof(*d));
    d->part_id = p.part_id;
    d->lo = p.lo;
    d->n_local = p.n_local;
    d->n_h = p.n_h;
    d->h_below = p.h_below;
    d->vp = p.n_local + p.n_h;
    d->n_train = p.n_train;
    d->cap = p.cap;
    d->nbatch = p.nbatch;
    d->perm_slots = p.perm_slots;
    d->indptr = p.indptr;
    d->cols_rank = p.cols_rank;
    d->halo_ids = p.halo;
    d->deg_in = p.deg_in;
    d->train_ids = p.train;
    d->table = p.table;
    d->rows = p.rows;
    d->se = p.se;
    d->sa = p.sa;
    d->slot_of = p.slot_of;
    d->slot_h = p.slot_h;
    d->hitmask = p.hitmask;
    d->rank_deg = p.rank_deg;
    d->deg_order = p.deg_order;
    d->perm = p.perm;
    d->halo_map = p.halo_map;
    (void)c;
}

mgnn_status upload_parts(mgnn_ctx ctx) {
    std::vector<PartDev> h(ctx->parts.size());
    for (size_t i = 0; i < ctx->parts.size(); ++i) fill_partdev(ctx, ctx->parts[i], &h[i]);
    dfree(ctx->d_parts);
    CK(dalloc(&ctx->d_parts, h.size()));
    CK(cudaMemcpy(ctx->d_parts, h.data(), h.size() * sizeof(PartDev), cudaMemcpyHostToDevice));
    return MGNN_OK;
}

mgnn_status upload_tables(mgnn_ctx ctx) {
    CK(cudaMemcpy((void*)ctx->d_tables, ctx->tables.data(), ctx->P * sizeof(float*), cudaMemcpyHostToDevice));
    std::vector<uint8_t> peer(ctx->P);
    for (int q = 0; q < ctx->P; ++q) peer[q] = (ctx->tables[q] && ctx->lp_of[q] < 0) ? 1 : 0;
    CK(cudaMemcpy(ctx->d_on_peer, peer.data(), ctx->P, cudaMemcpyHostToDevice));
    std::vector<int8_t> lpo(ctx->P);
    for (int q = 0; q < ctx->P; ++q) lpo[q] = (int8_t)(ctx->lp_of[q] < 128 ? ctx->lp_of[q] : -1);
    CK(cudaMemcpy(ctx->d_lp_of, lpo.data(), ctx->P, cudaMemcpyHostToDevice));
    return MGNN_OK;
}

WorldDev world_of(mgnn_ctx ctx) {
    WorldDev w;
    w.n_parts = ctx->P;
    w.pitch = ctx->pitch;
    w.bounds = ctx->d_bounds;
    w.tables = ctx->d_tables;
    w.on_peer = ctx->d_on_peer;
    w.lp_of = ctx->d_lp_of;
    return w;
}

void free_win(Win& w) {
    dfree(w.fr_rank);
    dfree(w.fr_gid);
    dfree(w.hop_size);
    for (int i = 0; i < kMaxLayers; ++i) {
        dfree(w.off[i]);
        dfree(w.cols[i]);
    }
    if (!w.x_user) dfree(w.X);              // a caller-owned X stays the caller's
    w.X = nullptr;
    dfree(w.zero);
    dfree(w.ext_seeds);
    dfree(w.ext_counts);
    w = Win();
}

void free_buffer(Part& p) {
    dfree(p.rows); dfree(p.se); dfree(p.sa); dfree(p.slot_of); dfree(p.slot_h); dfree(p.hitmask); dfree(p.rank_deg); dfree(p.deg_order);
    dfree(p.ek); dfree(p.ekt); dfree(p.ev); dfree(p.evt); dfree(p.rk); dfree(p.rkt); dfree(p.rv); dfree(p.rvt);
}

void free_perm(Part& p) {
    dfree(p.perm); dfree(p.pk); dfree(p.pkt); dfree(p.pvt);
    p.chunk_loaded[0] = p.chunk_loaded[1] = -1;
    p.perm_slots = 0;
}

mgnn_status ensure_scratch(mgnn_ctx ctx, void** p, size_t* have, size_t bytes) {
    if (bytes <= *have) return MGNN_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    CK(cudaMalloc(p, bytes));
    *have = bytes;
    return MGNN_OK;
}

WinDev win_dev(mgnn_ctx ctx, Win& w) {
    WinDev d;
    memset(&d, 0, sizeof(d));
    d.n_steps = w.n_steps;
    d.n_inst = (int32_t)ctx->parts.size() * w.n_steps;
    d.L = ctx->L;
    d.batch = ctx->batch;
    d.pitch = ctx->pitch;
    d.feat_dim = ctx->D;
    d.step0 = w.step0;
    d.seed_lo = (uint32_t)ctx->run_seed;
    d.seed_hi = (uint32_t)(ctx->run_seed >> 32);
    for (int i = 0; i < ctx->L; ++i) {
        d.k_hop[i] = ctx->k_hop[i];
        d.off_stride[i] = ctx->fcap[i] + 1;
        d.col_stride[i] = ctx->ecap[i];
        d.off[i] = w.off[i];
        d.cols[i] = w.cols[i];
    }
    d.ucap = ctx->ucap;
    d.seed_hmask = ctx->seed_h - 1;
    d.bm_words = ctx->bm_words;
    d.fr_rank = w.fr_rank;
    d.fr_gid = w.fr_gid;
    d.hop_size = w.hop_size;
    d.X = w.X;
    d.counts = w.counts;
    d.gctr = w.gctr;
    d.seedpos = w.seedpos;
    d.ovf = ctx->d_ovf;
    d.fb = w.fb;
    d.fbp = w.fbp;
    d.nb = w.nb;
    d.parts = ctx->d_parts;
    d.err = ctx->d_err;
    d.gathered_rows = ctx->d_gathered;
    d.sampled_units = ctx->prof ? ctx->d_sampled : nullptr;
    d.prof_hm = ctx->prof ? ctx->d_sampled + 3 : nullptr;
    d.remote = ctx->remote ? 1 : 0;
    d.n_global = ctx->n_global;
    d.g_indptr = ctx->g_indptr;
    d.g_cols = ctx->g_cols;
    int64_t nnz_max = ctx->remote ? ctx->g_nnz : 0;
    if (!ctx->remote)
        for (auto& p : ctx->parts) nnz_max = std::max(nnz_max, p.nnz);
    d.idx32 = nnz_max < ((int64_t)1 << 32) ? 1 : 0;
    return d;
}

}  // namespace host
}  // namespace mgnn

// =====================================================================================
extern "C" {

float mgnn_alpha_default(float gamma, int32_t delta) {
    float a = 1.0f;
    for (int32_t i = 0; i < delta; ++i) a = a * gamma;   // Eq.1, iterated fp32 (R#13)
    return a;
}

mgnn_status mgnn_ctx_create(int32_t device, int32_t n_parts, int64_t n_global, const int64_t* bounds,
                            int32_t feat_dim, uint64_t feat_seed, mgnn_ctx* out) {
    if (!out || !bounds || n_parts < 1 || n_global < 0 || n_global >= (1ll << 31) || feat_dim < 0) return MGNN_EINVAL;
    if (bounds[0] != 0 || bounds[n_parts] != n_global) return MGNN_EINVAL;
    for (int q = 0; q < n_parts; ++q)
        if (bounds[q + 1] < bounds[q]) return MGNN_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return MGNN_ECUDA;
    if (cudaSetDevice(device) != cudaSuccess) return MGNN_ECUDA;
    mgnn_ctx ctx = new mgnn_ctx_s();
    ctx->device = device;
    ctx->P = n_parts;
    ctx->n_global = n_global;
    ctx->bounds.assign(bounds, bounds + n_parts + 1);
    ctx->D = feat_dim;
    ctx->pitch = ((feat_dim + 3) / 4) * 4;
    if (ctx->pitch == 0) ctx->pitch = 4;
    ctx->feat_seed = feat_seed;
    ctx->lp_of.assign(n_parts, -1);
    {
        const char* e = getenv("MGNN_EVICT_SORT");
        ctx->force_sort_path = e && (e[0] == '1' || e[0] == '2');
        ctx->sort_full_lists = e && e[0] == '2';
        const char* e2 = getenv("MGNN_EV_SELECT");
        ctx->ev_scan = e2 && e2[0] == '0';
        const char* e3 = getenv("MGNN_FUSED_DECAY");
        ctx->no_fused_decay = e3 && e3[0] == '0';
    }
    ctx->tables.assign(n_parts, nullptr);
    mgnn_status st = MGNN_OK;
    auto chk = [&](cudaError_t e) { if (e != cudaSuccess && st == MGNN_OK) st = MGNN_ECUDA; };
    chk(dalloc(&ctx->d_bounds, n_parts + 1));
    chk(cudaMemcpy(ctx->d_bounds, bounds, (n_parts + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    chk(dalloc((float***)&ctx->d_tables, n_parts));
    chk(cudaMemset((void*)ctx->d_tables, 0, n_parts * sizeof(float*)));
    chk(dalloc(&ctx->d_on_peer, n_parts));
    chk(cudaMemset(ctx->d_on_peer, 0, n_parts));
    chk(dalloc(&ctx->d_lp_of, n_parts));
    chk(cudaMemset(ctx->d_lp_of, 0xFF, n_parts));
    chk(dalloc(&ctx->d_err, 1));
    chk(cudaMemset(ctx->d_err, 0, sizeof(int32_t)));
    chk(dalloc(&ctx->d_ovf, 1));
    chk(cudaMemset(ctx->d_ovf, 0xFF, sizeof(unsigned long long)));
    chk(dalloc(&ctx->d_gathered, 1));
    chk(cudaMemset(ctx->d_gathered, 0, sizeof(long long)));
    chk(dalloc(&ctx->d_sampled, 6));
    chk(cudaMemset(ctx->d_sampled, 0, 6 * sizeof(long long)));
    if (st != MGNN_OK) {
        mgnn_destroy(ctx);
        return st;
    }
    *out = ctx;
    return MGNN_OK;
}

void mgnn_destroy(mgnn_ctx ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    partition_free(ctx);
    for (auto& w : ctx->win) free_win(w);
    free_sage(ctx);
    for (auto& p : ctx->parts) {
        free_buffer(p);
        free_perm(p);
        dfree(p.indptr); dfree(p.cols_rank); dfree(p.halo); dfree(p.deg_in); dfree(p.train); dfree(p.table);
    }
    for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    for (auto& v : ctx->prof_ev)
        for (auto& e : v) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    dfree(ctx->d_sampled);
    dfree(ctx->d_bounds);
    dfree(ctx->d_tables);
    dfree(ctx->d_on_peer);
    dfree(ctx->d_lp_of);
    dfree(ctx->d_parts);
    dfree(ctx->d_err);
    dfree(ctx->d_ovf);
    dfree(ctx->d_gathered);
    dfree(ctx->d_evsegs);
    dfree(ctx->d_candsegs);
    dfree(ctx->d_candsegs_hi);
    dfree(ctx->d_initsegs);
    dfree(ctx->d_sel_n);
    dfree(ctx->ev_zero);
    if (ctx->sort_scr) cudaFree(ctx->sort_scr);
    if (ctx->perm_scr) cudaFree(ctx->perm_scr);
    dfree(ctx->d_permsegs);
    dfree(ctx->d_perm_n);
    dfree(ctx->g_indptr);
    dfree(ctx->g_cols);
    for (auto& p : ctx->parts) dfree(p.halo_map);
    delete ctx;
}

const char* mgnn_last_error(mgnn_ctx ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

mgnn_status mgnn_next_step(mgnn_ctx ctx, uint64_t* next_step) {
    if (!ctx || !next_step) return MGNN_EINVAL;
    *next_step = ctx->seq_started ? ctx->next_step : 1;
    return MGNN_OK;
}

int64_t mgnn_launch_count(mgnn_ctx ctx) {
    (void)ctx;
    return launches_total();
}

// ------------------------------------------------------------------ partition load (A1)
mgnn_status mgnn_partition_load(mgnn_ctx ctx, const mgnn_partition_desc* d, int32_t* local_index) {
    GUARD();
    if (!d || d->part_id < 0 || d->part_id >= ctx->P) return fail(ctx, MGNN_EINVAL, "bad part_id");
    if (ctx->lp_of[d->part_id] >= 0) return fail(ctx, MGNN_EINVAL, "partition already loaded");
    if (ctx->configured || ctx->buffer_ready) return fail(ctx, MGNN_ESTATE, "load after buffer_init/sampler_config");
    const int64_t lo = ctx->bounds[d->part_id], hi = ctx->bounds[d->part_id + 1], nl = hi - lo;
    if (!d->indptr || (nl > 0 && d->indptr[0] != 0)) return fail(ctx, MGNN_EINVAL, "indptr[0] != 0");
    for (int64_t r = 0; r < nl; ++r) {
        if (d->indptr[r + 1] < d->indptr[r]) return fail(ctx, MGNN_EINVAL, "indptr not monotone");
        for (int64_t e = d->indptr[r]; e < d->indptr[r + 1]; ++e) {
            const int32_t c = d->cols[e];
            if (c < 0 || c >= ctx->n_global) return fail(ctx, MGNN_EINVAL, "column out of range");
            if (c == lo + r) return fail(ctx, MGNN_EINVAL, "self loop");
            if (e > d->indptr[r] && d->cols[e - 1] >= c) return fail(ctx, MGNN_EINVAL, "row not strictly ascending");
        }
    }
    if (d->n_train < 0 || (d->n_train > 0 && !d->train_ids)) return fail(ctx, MGNN_EINVAL, "train ids");
    for (int64_t i = 0; i < d->n_train; ++i) {
        if (d->train_ids[i] < lo || d->train_ids[i] >= hi) return fail(ctx, MGNN_EINVAL, "train id not local");
        if (i > 0 && d->train_ids[i - 1] >= d->train_ids[i]) return fail(ctx, MGNN_EINVAL, "train ids not sorted");
    }
    const int64_t nnz = nl > 0 ? d->indptr[nl] : 0;
    Part p;
    p.part_id = d->part_id;
    p.lo = lo;
    p.n_local = nl;
    p.nnz = nnz;
    p.n_train = d->n_train;
    cudaStream_t s = 0;
    int32_t* cols_g = nullptr;
    uint32_t* bm = nullptr;
    int32_t* gmap = nullptr;
    unsigned long long* status = nullptr;
    long long* d_n = nullptr;
    const int64_t words = (ctx->n_global + 31) / 32;
    const int64_t halo_max = std::min<int64_t>(nnz, ctx->n_global - nl);
    const int64_t tiles = (words + 1023) / 1024 + 1;
    CK(dalloc(&p.indptr, nl + 1));
    CK(cudaMemcpy(p.indptr, d->indptr, (nl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(dalloc(&cols_g, nnz));
    if (nnz) CK(cudaMemcpy(cols_g, d->cols, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(dalloc(&bm, words));
    CK(cudaMemset(bm, 0, std::max<int64_t>(words, 1) * sizeof(uint32_t)));
    CK(dalloc(&status, tiles + 1));
    CK(cudaMemset(status, 0, (tiles + 1) * sizeof(unsigned long long)));
    CK(dalloc(&d_n, 2));
    CK(cudaMemset(d_n, 0, 2 * sizeof(long long)));
    const int64_t halo_cap = ctx->dense ? std::max<int64_t>(ctx->n_global - nl, 1) : halo_max;
    CK(dalloc(&p.halo, halo_cap));
    if (ctx->dense) {       // NEXT-1 dense S_A: the scorable set is every non-local node
        std::vector<uint32_t> hb((size_t)words, 0u);
        for (int64_t v = 0; v < ctx->n_global; ++v)
            if (v < lo || v >= hi) hb[(size_t)(v >> 5)] |= 1u << (v & 31);
        if (words) CK(cudaMemcpy(bm, hb.data(), words * sizeof(uint32_t), cudaMemcpyHostToDevice));
    } else {
        launch_mark_halo(cols_g, nnz, lo, hi, bm, s);
    }
    Scratch sc{status + 1, (int32_t*)status};
    launch_bitmap_to_ids(bm, words, p.halo, d_n, sc, s);
    CKL();
    long long nh = 0;
    CK(cudaMemcpy(&nh, d_n, sizeof(long long), cudaMemcpyDeviceToHost));
    p.n_h = nh;
    launch_lower_bound(p.halo, nh, lo, d_n + 1, s);
    long long hb = 0;
    CK(cudaMemcpy(&hb, d_n + 1, sizeof(long long), cudaMemcpyDeviceToHost));
    p.h_below = hb;
    CK(dalloc(&gmap, ctx->n_global));
    launch_halo_index(p.halo, nh, gmap, s);
    CK(dalloc(&p.deg_in, nh));
    CK(cudaMemset(p.deg_in, 0, std::max<int64_t>(nh, 1) * sizeof(int32_t)));
    CK(dalloc(&p.cols_rank, nnz));
    launch_deg_rank(cols_g, nnz, lo, nl, hb, gmap, p.deg_in, p.cols_rank, s);
    {   // max in-partition degree: sets the number of degree digits the replacement sort needs
        std::vector<int32_t> deg(nh);
        if (nh) CK(cudaMemcpy(deg.data(), p.deg_in, nh * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (int32_t x : deg) p.max_deg_in = std::max(p.max_deg_in, x);
        p.n_h_true = 0;
        for (int32_t x : deg) p.n_h_true += x > 0;
    }
    CK(dalloc(&p.train, d->n_train));
    if (d->n_train) CK(cudaMemcpy(p.train, d->train_ids, d->n_train * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(dalloc(&p.table, std::max<int64_t>(nl, 1) * ctx->pitch));
    launch_features(p.table, lo, nl, ctx->D, ctx->pitch, ctx->feat_seed, s);
    CKL();
    CK(cudaDeviceSynchronize());
    dfree(cols_g);
    dfree(bm);
    dfree(gmap);
    dfree(status);
    dfree(d_n);
    const int32_t lp = (int32_t)ctx->parts.size();
    ctx->tables[p.part_id] = p.table;
    ctx->lp_of[p.part_id] = lp;
    ctx->parts.push_back(p);
    mgnn_status st = upload_tables(ctx);
    if (st) return st;
    st = upload_parts(ctx);
    if (st) return st;
    if (local_index) *local_index = lp;
    return MGNN_OK;
}

mgnn_status mgnn_table_export(mgnn_ctx ctx, int32_t part_id, void* handle_out) {
    GUARD();
    if (part_id < 0 || part_id >= ctx->P || ctx->lp_of[part_id] < 0 || !handle_out)
        return fail(ctx, MGNN_EINVAL, "export: partition not hosted here");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void*)ctx->parts[ctx->lp_of[part_id]].table));
    static_assert(sizeof(h) == MGNN_IPC_HANDLE_BYTES, "ipc handle size");
    memcpy(handle_out, &h, sizeof(h));
    return MGNN_OK;
}

mgnn_status mgnn_table_import(mgnn_ctx ctx, int32_t part_id, const void* handle) {
    GUARD();
    if (part_id < 0 || part_id >= ctx->P || ctx->lp_of[part_id] >= 0 || !handle)
        return fail(ctx, MGNN_EINVAL, "import: bad partition");
    if (ctx->tables[part_id]) return fail(ctx, MGNN_EINVAL, "import: already imported");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->ipc_opened.push_back(ptr);
    ctx->tables[part_id] = (const float*)ptr;
    return upload_tables(ctx);
}

mgnn_status mgnn_part_info(mgnn_ctx ctx, int32_t lp, int64_t* info) {
    if (!ctx || !info || lp < 0 || lp >= (int32_t)ctx->parts.size()) return MGNN_EINVAL;
    const Part& p = ctx->parts[lp];
    info[0] = p.part_id;
    info[1] = p.n_local;
    info[2] = p.n_h;
    info[3] = p.cap;
    info[4] = p.n_train;
    return MGNN_OK;
}

mgnn_status mgnn_halo_get(mgnn_ctx ctx, int32_t lp, int32_t* halo_ids, int32_t* deg_in) {
    GUARD();
    if (lp < 0 || lp >= (int32_t)ctx->parts.size()) return fail(ctx, MGNN_EINVAL, "bad lp");
    const Part& p = ctx->parts[lp];
    if (halo_ids && p.n_h) CK(cudaMemcpy(halo_ids, p.halo, p.n_h * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (deg_in && p.n_h) CK(cudaMemcpy(deg_in, p.deg_in, p.n_h * sizeof(int32_t), cudaMemcpyDeviceToHost));
    return MGNN_OK;
}

mgnn_status mgnn_table_row(mgnn_ctx ctx, int64_t node, float* out) {
    GUARD();
    if (node < 0 || node >= ctx->n_global || !out) return fail(ctx, MGNN_EINVAL, "bad node");
    int q = 0;
    while (!(ctx->bounds[q] <= node && node < ctx->bounds[q + 1])) ++q;
    if (ctx->lp_of[q] < 0) return fail(ctx, MGNN_EINVAL, "node not hosted here");
    const Part& p = ctx->parts[ctx->lp_of[q]];
    if (ctx->D)
        CK(cudaMemcpy(out, p.table + (node - p.lo) * ctx->pitch, ctx->D * sizeof(float), cudaMemcpyDeviceToHost));
    return MGNN_OK;
}

// ------------------------------------------------------------------ INITIALIZE_PREFETCHER (A2)
mgnn_status mgnn_buffer_init(mgnn_ctx ctx, const mgnn_policy* pol, mgnn_stream stream) {
    GUARD();
    if (!pol || !(pol->gamma > 0.0f && pol->gamma <= 1.0f) || !(pol->alpha >= 0.0f) || pol->alpha != pol->alpha ||
        pol->alpha > 3.4e38f || pol->theta_r != pol->theta_r || pol->delta < 0 || pol->f_bp > 10000u)
        return fail(ctx, MGNN_EINVAL, "invalid policy");
    if (ctx->parts.empty()) return fail(ctx, MGNN_ESTATE, "no partition loaded");
    for (int q = 0; q < ctx->P; ++q)
        if (!ctx->tables[q]) return fail(ctx, MGNN_ESTATE, "feature table of partition " + std::to_string(q) + " missing");
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaStreamSynchronize(s));
    int64_t cap_max = 0, nh_max = 0;
    for (auto& p : ctx->parts) {
        free_buffer(p);
        p.cap = ((int64_t)pol->f_bp * p.n_h_true + 9999) / 10000;   // ceil(f |V_p^h|) (R#11)
        CK(dalloc(&p.rows, p.cap * ctx->pitch));
        CK(dalloc(&p.se, p.cap));
        CK(dalloc(&p.sa, p.n_h));
        CK(dalloc(&p.slot_of, p.n_h));
        CK(dalloc(&p.slot_h, p.cap));
        CK(dalloc(&p.hitmask, p.cap));
        CK(dalloc(&p.rank_deg, p.n_h));
        CK(dalloc(&p.deg_order, p.n_h));
        CK(dalloc(&p.ek, p.cap)); CK(dalloc(&p.ekt, p.cap)); CK(dalloc(&p.ev, p.cap)); CK(dalloc(&p.evt, p.cap));
        CK(dalloc(&p.rk, p.n_h)); CK(dalloc(&p.rkt, p.n_h)); CK(dalloc(&p.rv, p.n_h)); CK(dalloc(&p.rvt, p.n_h));
        cap_max = std::max(cap_max, p.cap);
        nh_max = std::max(nh_max, p.n_h);
    }
    mgnn_status st = upload_parts(ctx);
    if (st) return st;
    const int n_lp = (int)ctx->parts.size();
    // eviction / init sort segments: 2*lp = E (slots), 2*lp+1 = R (halo)
    std::vector<SortSeg> segs(2 * n_lp), initsegs(n_lp);
    ctx->ev_passes = 2;
    dfree(ctx->d_sel_n);
    CK(dalloc(&ctx->d_sel_n, 2 * n_lp));
    CK(cudaMemset(ctx->d_sel_n, 0, 2 * n_lp * sizeof(long long)));
    for (int lp = 0; lp < n_lp; ++lp) {
        Part& p = ctx->parts[lp];
        // E: key = S_E bits << 32, items in id order -> digits of the high word only
        segs[2 * lp] = make_seg(p.ek, p.ev, p.ekt, p.evt, ctx->d_sel_n + 2 * lp, {32, 40, 48, 56});
        // R: key = ~S_A bits << 32 | rank_deg (unique): the low word needs only the bytes n_h occupies
        // (low word = rank_deg < n_h: bytes above it are zero; an even digit count is kept so the
        // result lands in the primary buffers)
        segs[2 * lp + 1] = p.n_h <= (1 << 16)
                               ? make_seg(p.rk, p.rv, p.rkt, p.rvt, ctx->d_sel_n + 2 * lp + 1, {0, 8, 32, 40, 48, 56})
                               : make_seg(p.rk, p.rv, p.rkt, p.rvt, ctx->d_sel_n + 2 * lp + 1,
                                          {0, 8, 16, 24, 32, 40, 48, 56});
        ctx->ev_passes = std::max(ctx->ev_passes, std::max(segs[2 * lp].npass, segs[2 * lp + 1].npass));
        initsegs[lp] = make_seg(p.rk, p.rv, p.rkt, p.rvt, ctx->d_sel_n + 2 * lp + 1, {0, 8, 16, 24});
    }
    dfree(ctx->d_evsegs);
    CK(dalloc(&ctx->d_evsegs, segs.size()));
    CK(cudaMemcpy(ctx->d_evsegs, segs.data(), segs.size() * sizeof(SortSeg), cudaMemcpyHostToDevice));
    dfree(ctx->d_initsegs);
    CK(dalloc(&ctx->d_initsegs, initsegs.size()));
    CK(cudaMemcpy(ctx->d_initsegs, initsegs.data(), initsegs.size() * sizeof(SortSeg), cudaMemcpyHostToDevice));
    const int64_t n_sort_max = std::max<int64_t>(std::max(cap_max, nh_max), 1);
    ctx->ev_tiles = (n_sort_max + 2047) / 2048;
    dfree(ctx->ev_zero);
    {   // eviction-round scratch, zeroed per round: [tile ctrs | look-back words | hist | ticket | thr | n_cand]
        auto up = [](size_t x) { return (x + 255) / 256 * 256; };
        const size_t nseg = 2 * (size_t)n_lp;
        const size_t o_st = up(nseg * 4);
        const size_t o_hist = o_st + up(nseg * ctx->ev_tiles * 8);
        const size_t o_hist2 = o_hist + up(nseg * 4096 * 4);
        const size_t o_tk = o_hist2 + up(nseg * 4096 * 4);
        const size_t o_thr = o_tk + 256;
        const size_t o_nc = o_thr + up(nseg * 16);
        const size_t o_kth = o_nc + up(nseg * 8);
        const size_t o_tc2 = o_kth + up(nseg * 16);
        const size_t o_st2 = o_tc2 + up(nseg * 4);
        ctx->ev_zero_bytes = o_st2 + up(nseg * ctx->ev_tiles * 8);
        CK(dalloc((char**)&ctx->ev_zero, ctx->ev_zero_bytes));
        ctx->ev_sc.tilectr = (int32_t*)ctx->ev_zero;
        ctx->ev_sc.status = (unsigned long long*)(ctx->ev_zero + o_st);
        ctx->ev_ev.hist = (uint32_t*)(ctx->ev_zero + o_hist);
        ctx->ev_ev.hist2 = (uint32_t*)(ctx->ev_zero + o_hist2);
        ctx->ev_ev.ticket = (unsigned*)(ctx->ev_zero + o_tk);
        ctx->ev_ev.thr = (long long*)(ctx->ev_zero + o_thr);
        ctx->ev_ev.n_cand = (unsigned long long*)(ctx->ev_zero + o_nc);
        ctx->ev_ev.kth = (unsigned long long*)(ctx->ev_zero + o_kth);
        ctx->ev_sc2.tilectr = (int32_t*)(ctx->ev_zero + o_tc2);
        ctx->ev_sc2.status = (unsigned long long*)(ctx->ev_zero + o_st2);
    }
    {   // large buffers: the K winners are sorted out of the compacted candidates (k_cand appends them
        // unordered, so E sorts all 8 key bytes; R's schedule already covers every byte that differs)
        std::vector<SortSeg> cs(2 * n_lp);
        const long long* nc = reinterpret_cast<const long long*>(ctx->ev_ev.n_cand);
        for (int lp = 0; lp < n_lp; ++lp) {
            Part& p = ctx->parts[lp];
            cs[2 * lp] = make_seg(p.ekt, p.evt, p.ek, p.ev, nc + 2 * lp, {0, 8, 16, 24, 32, 40, 48, 56});
            SortSeg r = segs[2 * lp + 1];
            r.keys = p.rkt; r.vals = p.rvt; r.keys_tmp = p.rk; r.vals_tmp = p.rv; r.n = nc + 2 * lp + 1;
            cs[2 * lp + 1] = r;
        }
        dfree(ctx->d_candsegs);
        CK(dalloc(&ctx->d_candsegs, cs.size()));
        CK(cudaMemcpy(ctx->d_candsegs, cs.data(), cs.size() * sizeof(SortSeg), cudaMemcpyHostToDevice));
        // candidates from the ordered lists (k_cand_ord keeps E in id order, R in rank_deg order): the
        // stable sort needs the high word (the score) only
        for (int lp = 0; lp < n_lp; ++lp) {
            Part& p = ctx->parts[lp];
            cs[2 * lp] = make_seg(p.ekt, p.evt, p.ek, p.ev, nc + 2 * lp, {32, 40, 48, 56});
            cs[2 * lp + 1] = make_seg(p.rkt, p.rvt, p.rk, p.rv, nc + 2 * lp + 1, {32, 40, 48, 56});
        }
        dfree(ctx->d_candsegs_hi);
        CK(dalloc(&ctx->d_candsegs_hi, cs.size()));
        CK(cudaMemcpy(ctx->d_candsegs_hi, cs.data(), cs.size() * sizeof(SortSeg), cudaMemcpyHostToDevice));
    }
    {
        mgnn_status st2 = ensure_scratch(ctx, &ctx->sort_scr, &ctx->sort_scr_bytes,
                                         std::max(radix_scratch_bytes(2 * n_lp, n_sort_max, 8),
                                                             radix_scratch_bytes(1, std::max<int64_t>(nh_max, 1), 4)));
        if (st2) return st2;
    }
    WorldDev G = world_of(ctx);
    for (int lp = 0; lp < n_lp; ++lp) {
        Part& p = ctx->parts[lp];
        // order V_p^h by (deg_in desc, id asc) (R#10) and take the first cap
        launch_init_keys(ctx->d_parts + lp, p.n_h, ctx->d_initsegs + lp, ctx->d_sel_n + 2 * lp + 1, s);
        radix_sort_pairs(ctx->d_initsegs + lp, 1, std::max<int64_t>(p.n_h, 1), 4, ctx->sort_scr, s);
        launch_init_fill(ctx->d_parts + lp, p.n_h, p.cap, p.rv, s);
        launch_rows_from_owners(ctx->d_parts + lp, p.cap, G, s);
        CKL();
    }
    CK(cudaStreamSynchronize(s));
    {   // TMA row-gather descriptors of every source on this GPU (k_gather_g4)
        ctx->g4_ok = n_lp <= kMaxGatherMaps / 2 && ctx->D == ctx->pitch;
        memset(&ctx->gmaps, 0, sizeof(ctx->gmaps));
        ctx->gmaps.n_lp = n_lp;
        for (int lp = 0; lp < n_lp && ctx->g4_ok; ++lp) {
            const Part& p = ctx->parts[lp];
            ctx->g4_ok = encode_row_map(ctx->gmaps.maps[lp], p.table, std::max<int64_t>(p.n_local, 1), ctx->D,
                                        ctx->pitch) &&
                         encode_row_map(ctx->gmaps.maps[n_lp + lp], p.rows, std::max<int64_t>(p.cap, 1), ctx->D,
                                        ctx->pitch);
        }
    }
    ctx->pol = *pol;
    ctx->buffer_ready = true;
    ctx->seq_started = false;
    for (auto& w : ctx->win) w.sampled = w.gathered = w.scored = false;
    return MGNN_OK;
}

// ------------------------------------------------------------------ sampler configuration
// ------------------------------------------------------------------ NEXT-1: remote expansion
mgnn_status mgnn_ctx_set_dense_scores(mgnn_ctx ctx, int32_t enable) {
    GUARD();
    if (!ctx->parts.empty()) return fail(ctx, MGNN_ESTATE, "dense scores must be chosen before partition_load");
    ctx->dense = enable != 0;
    return MGNN_OK;
}

mgnn_status mgnn_graph_csr_load(mgnn_ctx ctx, const int64_t* indptr, const int32_t* cols) {
    GUARD();
    if (!indptr || (!cols && indptr[ctx->n_global] > 0) || indptr[0] != 0)
        return fail(ctx, MGNN_EINVAL, "global CSR");
    const int64_t nnz = indptr[ctx->n_global];
    for (int64_t v = 0; v < ctx->n_global; ++v)
        if (indptr[v + 1] < indptr[v]) return fail(ctx, MGNN_EINVAL, "global CSR indptr not monotone");
    CK(cudaDeviceSynchronize());
    dfree(ctx->g_indptr);
    dfree(ctx->g_cols);
    CK(dalloc(&ctx->g_indptr, ctx->n_global + 1));
    CK(dalloc(&ctx->g_cols, nnz));
    ctx->g_nnz = nnz;
    CK(cudaMemcpy(ctx->g_indptr, indptr, (ctx->n_global + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (nnz) CK(cudaMemcpy(ctx->g_cols, cols, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    return MGNN_OK;
}

mgnn_status mgnn_sampler_expand_remote(mgnn_ctx ctx, int32_t enable) {
    GUARD();
    if (ctx->configured) return fail(ctx, MGNN_ESTATE, "expand_remote must precede sampler_config");
    if (!enable) {
        ctx->remote = false;
        return MGNN_OK;
    }
    if (!ctx->g_indptr && (int32_t)ctx->parts.size() != ctx->P)
        return fail(ctx, MGNN_ESTATE, "remote expansion: load the global CSR (mgnn_graph_csr_load) or host every partition");
    CK(cudaDeviceSynchronize());
    for (auto& p : ctx->parts)
        if (!p.halo_map) {
            CK(dalloc(&p.halo_map, ctx->n_global));
            CK(cudaMemset(p.halo_map, 0xFF, ctx->n_global * sizeof(int32_t)));
            launch_halo_index(p.halo, p.n_h, p.halo_map, 0);
        }
    if (!ctx->g_indptr) {
        int64_t nnz = 0;
        for (auto& p : ctx->parts) nnz += p.nnz;
        CK(dalloc(&ctx->g_indptr, ctx->n_global + 1));
        CK(dalloc(&ctx->g_cols, nnz));
        ctx->g_nnz = nnz;
        mgnn_status st = upload_parts(ctx);
        if (st) return st;
        int64_t base = 0;
        for (int32_t q = 0; q < ctx->P; ++q) {          // partitions in id order = global row order
            const int lp = ctx->lp_of[q];
            Part& p = ctx->parts[lp];
            launch_global_csr(ctx->d_parts + lp, p.indptr, p.n_local, p.lo, p.nnz, base, ctx->g_indptr, ctx->g_cols, 0);
            base += p.nnz;
        }
    }
    CKL();
    CK(cudaDeviceSynchronize());
    ctx->remote = true;
    return upload_parts(ctx);
}

mgnn_status mgnn_sampler_config(mgnn_ctx ctx, const int32_t* fanouts, int32_t n_layers, int32_t batch,
                                uint64_t run_seed, int32_t max_window) {
    return mgnn_sampler_config_bounded(ctx, fanouts, n_layers, batch, run_seed, max_window, 0);
}

mgnn_status mgnn_sampler_config_bounded(mgnn_ctx ctx, const int32_t* fanouts, int32_t n_layers, int32_t batch,
                                        uint64_t run_seed, int32_t max_window, int64_t rows_bound) {
    GUARD();
    if (!fanouts || n_layers < 1 || n_layers > kMaxLayers || batch < 1 || max_window < 1 || max_window > 64 ||
        rows_bound < 0 || (rows_bound > 0 && rows_bound < batch))
        return fail(ctx, MGNN_EINVAL, "bad sampler config");
    for (int i = 0; i < n_layers; ++i)
        if (fanouts[i] < 1 || fanouts[i] > MGNN_MAX_FANOUT) return fail(ctx, MGNN_EINVAL, "fanout must be 1..32");
    if (ctx->parts.empty()) return fail(ctx, MGNN_ESTATE, "no partition loaded");
    CK(cudaDeviceSynchronize());
    {   // resuming after an arena overflow: every window from the overflowed one on was skipped on the
        // device (no buffer state changed), so the step order resumes there
        unsigned long long ovf = ~0ull;
        CK(cudaMemcpy(&ovf, ctx->d_ovf, sizeof(ovf), cudaMemcpyDeviceToHost));
        if (ovf != ~0ull) {
            ctx->next_step = ovf;
            CK(cudaMemset(ctx->d_ovf, 0xFF, sizeof(unsigned long long)));
        }
    }
    for (auto& w : ctx->win) free_win(w);
    free_sage(ctx);
    for (auto& p : ctx->parts) free_perm(p);
    ctx->configured = false;
    ctx->rows_bound = rows_bound;
    ctx->L = n_layers;
    ctx->batch = batch;
    ctx->run_seed = run_seed;
    ctx->max_window = max_window;
    for (int i = 0; i < n_layers; ++i) {
        ctx->fan[i] = fanouts[i];
        ctx->k_hop[i] = fanouts[n_layers - 1 - i];   // hop 0 (seeds) draws the last layer's fanout (R#2)
    }
    ctx->vp_max = 1;
    for (auto& p : ctx->parts) ctx->vp_max = std::max(ctx->vp_max, p.n_local + p.n_h);
    if (ctx->remote) ctx->vp_max = std::max<int64_t>(1, ctx->n_global);   // ranks are global ids (NEXT-1)
    ctx->bm_words = ((ctx->vp_max + 31) / 32 + 15) / 16 * 16;   // multiple of 16: k_compact's vector loads
    const int64_t big = (int64_t)1 << 40;
    ctx->fcap[0] = std::min<int64_t>(batch, ctx->vp_max);
    for (int i = 0; i < n_layers; ++i) {
        ctx->ecap[i] = std::max<int64_t>(sat_mul(ctx->fcap[i], ctx->k_hop[i], big), 1);
        ctx->fcap[i + 1] = std::min<int64_t>(sat_mul(ctx->fcap[i], 1 + ctx->k_hop[i], big), ctx->vp_max);
        if (rows_bound > 0) ctx->fcap[i + 1] = std::min(ctx->fcap[i + 1], rows_bound);   // realistic bound
    }
    ctx->ucap = ctx->fcap[n_layers];
    ctx->seed_h = 1;
    while (ctx->seed_h < 2 * ctx->fcap[0]) ctx->seed_h <<= 1;
    const int n_lp = (int)ctx->parts.size();
    const int64_t M = (int64_t)n_lp * max_window;
    for (auto& w : ctx->win) {
        CK(dalloc(&w.fr_rank, M * ctx->ucap));
        CK(dalloc(&w.fr_gid, M * ctx->ucap));
        CK(dalloc(&w.hop_size, M * (kMaxLayers + 1)));
        CK(cudaMemset(w.hop_size, 0, M * (kMaxLayers + 1) * sizeof(int64_t)));
        for (int i = 0; i < n_layers; ++i) {
            CK(dalloc(&w.off[i], M * (ctx->fcap[i] + 1)));
            CK(dalloc(&w.cols[i], M * ctx->ecap[i]));
        }
        CK(dalloc(&w.X, (size_t)M * ctx->ucap * ctx->pitch));
        CK(dalloc(&w.ext_seeds, M * batch));
        CK(dalloc(&w.ext_counts, M));
        // zero region: [tile counters | status words | counts | fb | fbp | seed hash], then the per-hop pairs
        size_t ctr_words = (size_t)(2 * n_layers + 1) * M;              // int32 (+ gather chunk counters)
        size_t st_words = 0;
        for (int i = 0; i < n_layers; ++i)
            st_words += (size_t)M * (scan_tiles_count(ctx->fcap[i]) + 1) + (size_t)M * (scan_tiles_words(ctx->bm_words) + 1);
        size_t off_ctr = 0;
        size_t off_st = ((ctr_words * 4 + 255) / 256) * 256;
        size_t off_cnt = off_st + ((st_words * 8 + 255) / 256) * 256;
        size_t off_fb = off_cnt + (((size_t)M * 8 * 8 + 255) / 256) * 256;
        size_t off_fbp = off_fb + (((size_t)M * ctx->bm_words * 4 + 255) / 256) * 256;
        size_t off_sp = off_fbp + (((size_t)M * ctx->bm_words * 4 + 255) / 256) * 256;
        size_t off_nb = off_sp + (((size_t)M * ctx->seed_h * 8 + 255) / 256) * 256;
        // the (bits, position) pairs follow the zeroed prefix: k_compact writes every word of them
        size_t total = off_nb + (size_t)M * n_layers * ctx->bm_words * 8;
        CK(dalloc(&w.zero, total));
        CK(cudaMemset(w.zero, 0, total));
        w.zero_bytes = off_nb;
        w.tilectr = (int32_t*)(w.zero + off_ctr);
        w.gctr = w.tilectr + (size_t)(2 * n_layers) * M;
        w.status = (unsigned long long*)(w.zero + off_st);
        w.counts = (long long*)(w.zero + off_cnt);
        w.fb = (uint32_t*)(w.zero + off_fb);
        w.fbp = (uint32_t*)(w.zero + off_fbp);
        w.seedpos = (int2*)(w.zero + off_sp);
        w.nb = (uint32_t*)(w.zero + off_nb);
        size_t so = 0;
        for (int i = 0; i < n_layers; ++i) {
            int64_t tc = scan_tiles_count(ctx->fcap[i]);
            w.sc_count[i] = Scratch{w.status + so, w.tilectr + (size_t)(2 * i) * M};
            so += (size_t)M * (tc < 1 ? 1 : tc);
            int64_t tw = scan_tiles_words(ctx->bm_words);
            w.sc_compact[i] = Scratch{w.status + so, w.tilectr + (size_t)(2 * i + 1) * M};
            so += (size_t)M * (tw < 1 ? 1 : tw);
        }
        w.alloc = true;
    }
    // epoch orders (R#8): a ring of 2G orders per partition, generated G epochs per sort call
    // (G >= the epochs one window can span, so a window's epochs live in at most two ring halves).
    ctx->perm_slots_max = 1;
    size_t scr = 0;
    for (auto& p : ctx->parts) {
        p.nbatch = p.n_train > 0 ? (p.n_train + batch - 1) / batch : 1;
        p.perm_chunk = (int32_t)std::max<int64_t>(8, (max_window + p.nbatch - 1) / p.nbatch + 1);
        p.perm_slots = 2 * p.perm_chunk;
        ctx->perm_slots_max = std::max(ctx->perm_slots_max, p.perm_slots);
        p.chunk_loaded[0] = p.chunk_loaded[1] = -1;
        const int64_t nt = std::max<int64_t>(p.n_train, 1);
        CK(dalloc(&p.perm, (int64_t)p.perm_slots * nt));
        CK(dalloc(&p.pk, p.perm_chunk * nt)); CK(dalloc(&p.pkt, p.perm_chunk * nt)); CK(dalloc(&p.pvt, p.perm_chunk * nt));
        scr = std::max(scr, (size_t)p.perm_chunk * 256 * 2 * sizeof(uint32_t));
    }
    {
        mgnn_status st2 = ensure_scratch(ctx, &ctx->perm_scr, &ctx->perm_scr_bytes, scr);
        if (st2) return st2;
    }
    std::vector<SortSeg> ps((size_t)n_lp * ctx->perm_slots_max);
    dfree(ctx->d_perm_n);
    CK(dalloc(&ctx->d_perm_n, n_lp));
    std::vector<long long> pn(n_lp);
    for (int lp = 0; lp < n_lp; ++lp) {
        Part& p = ctx->parts[lp];
        pn[lp] = p.n_train;
        for (int k = 0; k < p.perm_slots; ++k) {   // slot k = half k / G, epoch-in-chunk j = k % G
            const int64_t j = k % p.perm_chunk;
            ps[(size_t)lp * ctx->perm_slots_max + k] =
                make_seg(p.pk + j * p.n_train, (uint32_t*)(p.perm + (int64_t)k * p.n_train), p.pkt + j * p.n_train,
                         p.pvt + j * p.n_train, ctx->d_perm_n + lp, {0, 8, 16, 24, 32, 40, 48, 56});
        }
    }
    CK(cudaMemcpy(ctx->d_perm_n, pn.data(), n_lp * sizeof(long long), cudaMemcpyHostToDevice));
    dfree(ctx->d_permsegs);
    CK(dalloc(&ctx->d_permsegs, ps.size()));
    CK(cudaMemcpy(ctx->d_permsegs, ps.data(), ps.size() * sizeof(SortSeg), cudaMemcpyHostToDevice));
    mgnn_status st = upload_parts(ctx);
    if (st) return st;
    ctx->configured = true;
    return MGNN_OK;
}

// ------------------------------------------------------------------ mgnn_sample (A3-A5)
mgnn_status mgnn_sample(mgnn_ctx ctx, int32_t slot, uint64_t t0, int32_t n_steps, const int32_t* seeds,
                        const int32_t* seed_counts, int32_t seeds_on_host, mgnn_stream stream) {
    GUARD();
    if (!ctx->configured || !ctx->buffer_ready) return fail(ctx, MGNN_ESTATE, "sample before buffer_init/sampler_config");
    if (slot < 0 || slot > 1 || t0 < 1 || n_steps < 1 || n_steps > ctx->max_window)
        return fail(ctx, MGNN_EINVAL, "bad window");
    const int32_t delta = ctx->pol.delta;
    if (delta > 0) {
        for (uint64_t t = t0; t + 1 < t0 + (uint64_t)n_steps; ++t)
            if (t % (uint64_t)delta == 0) return fail(ctx, MGNN_EINVAL, "eviction step inside window (only last allowed)");
    }
    Win& w = ctx->win[slot];
    if (w.sampled && !w.scored && w.gathered) return fail(ctx, MGNN_ESTATE, "slot gathered but not scored");
    const int n_lp = (int)ctx->parts.size();
    const int64_t M = (int64_t)n_lp * n_steps;
    if (seeds && seeds_on_host) {
        if (!seed_counts) return fail(ctx, MGNN_EINVAL, "seed_counts missing");
        for (int64_t m = 0; m < M; ++m)
            if (seed_counts[m] < 1 || seed_counts[m] > ctx->batch) return fail(ctx, MGNN_EINVAL, "seed count");
    }
    if (!seeds)
        for (auto& p : ctx->parts)
            if (p.n_train < 1) return fail(ctx, MGNN_EINVAL, "partition without train ids needs external seeds");
    PartScope ps(ctx, 0, (cudaStream_t)stream);
    if (ps.err) return fail(ctx, MGNN_ECUDA, "sm partition: stream hand-off failed");
    cudaStream_t s = ps.s;
    // epoch orders needed by this window (R#8)
    if (!seeds) {
        for (int lp = 0; lp < n_lp; ++lp) {
            Part& p = ctx->parts[lp];
            const int64_t e0 = (int64_t)((t0 - 1) / (uint64_t)p.nbatch);
            const int64_t e1 = (int64_t)((t0 + n_steps - 2) / (uint64_t)p.nbatch);
            const int64_t G = p.perm_chunk;
            for (int64_t c = e0 / G; c <= e1 / G; ++c) {     // epoch e lives in ring slot e % 2G
                if (p.chunk_loaded[c % 2] == c) continue;
                const SortSeg* segs = ctx->d_permsegs + (size_t)lp * ctx->perm_slots_max + (c % 2) * G;
                launch_perm_build(ctx->d_parts + lp, p.n_train, (uint64_t)(c * G), (int)G, (uint32_t)ctx->run_seed,
                                  (uint32_t)(ctx->run_seed >> 32), segs, ctx->perm_scr, s);
                p.chunk_loaded[c % 2] = c;
            }
        }
    } else {
        const cudaMemcpyKind kind = seeds_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        CK(cudaMemcpyAsync(w.ext_seeds, seeds, M * ctx->batch * sizeof(int32_t), kind, s));
        CK(cudaMemcpyAsync(w.ext_counts, seed_counts, M * sizeof(int32_t), kind, s));
    }
    CK(cudaMemsetAsync(w.zero, 0, w.zero_bytes, s));
    w.n_steps = n_steps;
    w.step0 = t0;
    WinDev wd = win_dev(ctx, w);
    wd.n_inst = (int32_t)M;
    if (seeds) {
        wd.ext_seeds = w.ext_seeds;
        wd.ext_counts = w.ext_counts;
    }
    launch_seeds(wd, s);
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (ctx->prof == 1) {
        CK(cudaEventCreate(&pe0));
        CK(cudaEventCreate(&pe1));
        CK(cudaEventRecord(pe0, s));
    }
    for (int i = 0; i < ctx->L; ++i) {
        // per-hop scratch strides follow the max window; scans index by instance < M
        Scratch scc = w.sc_count[i], scp = w.sc_compact[i];
        launch_hop(wd, i, ctx->fcap[i], scc, s);
        launch_compact(wd, i, scp, s);
    }
    if (!ctx->defer_relabel) launch_relabel(wd, s);
    CKL();
    if (ctx->prof == 1) {
        CK(cudaEventRecord(pe1, s));
        ctx->prof_ev[0].emplace_back(pe0, pe1);
    }
    w.sampled = true;
    w.relabel_pending = ctx->defer_relabel;
    w.gathered = w.scored = false;
    return MGNN_OK;
}

mgnn_status mgnn_sampler_defer_relabel(mgnn_ctx ctx, int32_t enable) {
    GUARD();
    ctx->defer_relabel = enable != 0;
    return MGNN_OK;
}

mgnn_status mgnn_relabel(mgnn_ctx ctx, int32_t slot, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.sampled || !w.relabel_pending) return fail(ctx, MGNN_ESTATE, "relabel needs a window sampled with the relabel deferred");
    PartScope ps(ctx, 1, (cudaStream_t)stream);
    if (ps.err) return fail(ctx, MGNN_ECUDA, "sm partition: stream hand-off failed");
    cudaStream_t s = ps.s;
    WinDev wd = win_dev(ctx, w);
    wd.n_inst = (int32_t)((int64_t)ctx->parts.size() * w.n_steps);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof == 1) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
    }
    launch_relabel(wd, s);
    CKL();
    if (ctx->prof == 1) {
        CK(cudaEventRecord(e1, s));
        ctx->prof_ev[3].emplace_back(e0, e1);
    }
    w.relabel_pending = false;
    return MGNN_OK;
}

// ------------------------------------------------------------------ mgnn_lookup_gather (A6-A8, A10)
mgnn_status mgnn_lookup_gather(mgnn_ctx ctx, int32_t slot, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.sampled || w.gathered) return fail(ctx, MGNN_ESTATE, "gather needs a freshly sampled window");
    Win& other = ctx->win[slot ^ 1];
    if (other.gathered && !other.scored) return fail(ctx, MGNN_ESTATE, "previous window not scored");
    if (ctx->seq_started && w.step0 != ctx->next_step)
        return fail(ctx, MGNN_ESTATE, "windows must be gathered in step order");
    PartScope ps(ctx, 2, (cudaStream_t)stream);
    if (ps.err) return fail(ctx, MGNN_ECUDA, "sm partition: stream hand-off failed");
    cudaStream_t s = ps.s;
    WinDev wd = win_dev(ctx, w);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
    }
    // the tables this GPU's gathers read (hosted partitions; peers' misses are few) fit in L2?
    int64_t table_bytes = 0;
    for (auto& p : ctx->parts) table_bytes += p.n_local * (int64_t)ctx->pitch * 4;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device);
    launch_gather(wd, world_of(ctx), table_bytes <= (int64_t)l2 * 3 / 4, ctx->g4_ok ? &ctx->gmaps : nullptr, s);
    CKL();
    if (ctx->prof) {
        CK(cudaEventRecord(e1, s));
        ctx->prof_ev[1].emplace_back(e0, e1);
    }
    w.gathered = true;
    ctx->seq_started = true;
    ctx->next_step = w.step0 + (uint64_t)w.n_steps;
    return MGNN_OK;
}

// ------------------------------------------------------------------ mgnn_score_evict_refill (A9, A11, A12)
mgnn_status mgnn_score_evict_refill(mgnn_ctx ctx, int32_t slot, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.gathered || w.scored) return fail(ctx, MGNN_ESTATE, "score needs a gathered window");
    PartScope ps(ctx, 2, (cudaStream_t)stream);
    if (ps.err) return fail(ctx, MGNN_ECUDA, "sm partition: stream hand-off failed");
    cudaStream_t s = ps.s;
    const int n_lp = (int)ctx->parts.size();
    int64_t cap_max = 0, nmax = 1;
    for (auto& p : ctx->parts) {
        cap_max = std::max(cap_max, p.cap);
        nmax = std::max(nmax, std::max(p.cap, p.n_h));
    }
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (ctx->prof == 1) {
        CK(cudaEventCreate(&pe0));
        CK(cudaEventCreate(&pe1));
        CK(cudaEventRecord(pe0, s));
    }
    const uint64_t t_last = w.step0 + (uint64_t)w.n_steps - 1;
    const bool round = ctx->pol.delta > 0 && t_last % (uint64_t)ctx->pol.delta == 0;
    // ordered E / R lists (k_select, default) or counts and histograms straight from the scoreboards
    // with the candidates re-derived from them (MGNN_EV_SELECT=0; measured slower on products:
    // count + candidate scans 97 us per round against 70 us for select + candidates on the lists)
    const bool compact = ctx->sort_full_lists || !ctx->ev_scan;
    // on an eviction window with ordered lists the decay runs inside k_select (one launch less)
    const bool fused_decay = round && compact && !ctx->no_fused_decay;
    if (!fused_decay) launch_decay(ctx->d_parts, n_lp, cap_max, w.n_steps, ctx->pol.gamma, ctx->d_ovf, t_last, s);
    if (round) {
        CK(cudaMemsetAsync(ctx->ev_zero, 0, ctx->ev_zero_bytes, s));
        const PartDev* scan = compact ? nullptr : ctx->d_parts;
        if (compact) {
            launch_select(ctx->d_parts, n_lp, nmax, ctx->pol.alpha, ctx->pol.theta_r, ctx->d_evsegs, ctx->d_sel_n,
                          ctx->ev_sc, ctx->ev_ev, s, fused_decay ? w.n_steps : 0, ctx->pol.gamma, ctx->d_ovf, t_last);
        } else {
            CK(cudaMemsetAsync(ctx->d_sel_n, 0, 2 * n_lp * sizeof(long long), s));
            launch_ev_count(ctx->d_parts, n_lp, nmax, ctx->pol.alpha, ctx->pol.theta_r, ctx->d_sel_n, ctx->ev_ev, s);
        }
        const SortSeg* pairs = ctx->d_evsegs;     // where the K winners of E and R end, in order
        const long long* k_of = nullptr;           // K per segment (null: min(|E|, |R|) of the lists)
        if (cap_max <= kEvMax && !ctx->force_sort_path) {                   // K winners in order, no sort
            launch_cand_rank(ctx->d_evsegs, n_lp, nmax, ctx->ev_ev, scan, ctx->pol.alpha, ctx->pol.theta_r, s);
        } else if (ctx->sort_full_lists) {
            radix_sort_pairs(ctx->d_evsegs, 2 * n_lp, nmax, ctx->ev_passes, ctx->sort_scr, s);
        } else if (compact) {                      // threshold candidates in list order, sort their scores
            launch_cand_ord(ctx->d_evsegs, n_lp, nmax, ctx->ev_ev, ctx->ev_sc2, ctx->ev_tiles, s);
            radix_sort_pairs(ctx->d_candsegs_hi, 2 * n_lp, nmax, 4, ctx->sort_scr, s);
            pairs = ctx->d_candsegs_hi;
            k_of = ctx->ev_ev.thr;
        } else {                                   // threshold candidates (unordered), sort all key bytes
            launch_cand(ctx->d_evsegs, n_lp, nmax, ctx->ev_ev, scan, ctx->pol.alpha, ctx->pol.theta_r, s);
            radix_sort_pairs(ctx->d_candsegs, 2 * n_lp, nmax, 8, ctx->sort_scr, s);
            pairs = ctx->d_candsegs;
            k_of = ctx->ev_ev.thr;
        }
        launch_swap_refill(ctx->d_parts, n_lp, cap_max, pairs, k_of, world_of(ctx), w.counts, 8, w.n_steps,
                           ctx->d_ovf, t_last, s);
    }
    CKL();
    if (ctx->prof == 1) {
        CK(cudaEventRecord(pe1, s));
        ctx->prof_ev[2].emplace_back(pe0, pe1);
    }
    w.scored = true;
    return MGNN_OK;
}

// ------------------------------------------------------------------ views / readback
mgnn_status mgnn_window_get(mgnn_ctx ctx, int32_t slot, mgnn_window* out) {
    GUARD();
    if (slot < 0 || slot > 1 || !out) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.sampled) return fail(ctx, MGNN_ESTATE, "slot not sampled");
    memset(out, 0, sizeof(*out));
    out->n_steps = w.n_steps;
    out->n_parts_local = (int32_t)ctx->parts.size();
    out->n_inst = out->n_steps * out->n_parts_local;
    out->n_layers = ctx->L;
    out->step0 = w.step0;
    out->rows_stride = ctx->ucap;
    out->pitch = ctx->pitch;
    out->X = w.X;
    out->frontier = w.fr_gid;
    out->hop_size = w.hop_size;
    for (int i = 0; i < ctx->L; ++i) {
        out->offsets[i] = w.off[i];
        out->cols[i] = w.cols[i];
        out->off_stride[i] = ctx->fcap[i] + 1;
        out->col_stride[i] = ctx->ecap[i];
    }
    out->counts = (const int64_t*)w.counts;
    return MGNN_OK;
}

mgnn_status mgnn_window_shape(mgnn_ctx ctx, int64_t* rows_stride, int64_t* pitch, int64_t* max_inst) {
    GUARD();
    if (!ctx->configured) return fail(ctx, MGNN_ESTATE, "window_shape before sampler_config");
    if (rows_stride) *rows_stride = ctx->ucap;
    if (pitch) *pitch = ctx->pitch;
    if (max_inst) *max_inst = (int64_t)ctx->parts.size() * ctx->max_window;
    return MGNN_OK;
}

mgnn_status mgnn_window_bind_x(mgnn_ctx ctx, int32_t slot, float* X, int64_t capacity_floats) {
    GUARD();
    if (!ctx->configured) return fail(ctx, MGNN_ESTATE, "bind_x before sampler_config");
    if (slot < 0 || slot > 1 || !X) return fail(ctx, MGNN_EINVAL, "bind_x: bad slot / null X");
    const int64_t need = (int64_t)ctx->parts.size() * ctx->max_window * ctx->ucap * ctx->pitch;
    if (capacity_floats < need)
        return fail(ctx, MGNN_EINVAL, "bind_x: X holds " + std::to_string(capacity_floats) + " floats, the window needs " +
                                          std::to_string(need));
    if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) return fail(ctx, MGNN_EINVAL, "bind_x: X must be 16-byte aligned");
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, X) != cudaSuccess || pa.type != cudaMemoryTypeDevice || pa.device != ctx->device) {
        cudaGetLastError();
        return fail(ctx, MGNN_EINVAL, "bind_x: X is not device memory of this context's GPU");
    }
    CK(cudaDeviceSynchronize());                 // the slot's previous X may still be read or written
    Win& w = ctx->win[slot];
    if (!w.x_user) dfree(w.X);
    w.X = X;
    w.x_user = true;
    return rebind_sage_input(ctx, slot);         // the consumer's TMA descriptor of layer 0 reads X
}

mgnn_status mgnn_counts_read_async(mgnn_ctx ctx, int32_t slot, int64_t* host_counts, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1 || !host_counts) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.sampled) return fail(ctx, MGNN_ESTATE, "slot not sampled");
    const int64_t M = (int64_t)ctx->parts.size() * w.n_steps;
    CK(cudaMemcpyAsync(host_counts, w.counts, M * 8 * sizeof(long long), cudaMemcpyDeviceToHost,
                       (cudaStream_t)stream));
    return MGNN_OK;
}

mgnn_status mgnn_counts_read(mgnn_ctx ctx, int32_t slot, int64_t* host_counts, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1 || !host_counts) return fail(ctx, MGNN_EINVAL, "bad slot");
    Win& w = ctx->win[slot];
    if (!w.sampled) return fail(ctx, MGNN_ESTATE, "slot not sampled");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t M = (int64_t)ctx->parts.size() * w.n_steps;
    int32_t err = 0;
    unsigned long long ovf = ~0ull;
    CK(cudaMemcpyAsync(host_counts, w.counts, M * 8 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ovf, ctx->d_ovf, sizeof(ovf), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (err) {
        ctx->sticky = MGNN_EINVAL;
        return fail(ctx, MGNN_EINVAL, "invalid external seeds (not local or duplicated)");
    }
    if (ovf <= w.step0 + (uint64_t)w.n_steps - 1)
        return fail(ctx, MGNN_EOVERFLOW,
                    "a frontier exceeded the arena bound at the window starting at step " + std::to_string(ovf) +
                        ": that window and every later one were skipped (buffer state unchanged); reconfigure "
                        "with a larger bound (mgnn_sampler_config_bounded) and resume sampling at that step");
    return MGNN_OK;
}

mgnn_status mgnn_buffer_snapshot(mgnn_ctx ctx, int32_t lp, int32_t* node_ids, float* se, float* sa, int32_t* slot_of,
                                 float* rows) {
    GUARD();
    if (lp < 0 || lp >= (int32_t)ctx->parts.size()) return fail(ctx, MGNN_EINVAL, "bad lp");
    if (!ctx->buffer_ready) return fail(ctx, MGNN_ESTATE, "buffer not initialised");
    CK(cudaDeviceSynchronize());
    const Part& p = ctx->parts[lp];
    std::vector<int32_t> sh(p.cap), halo(p.n_h);
    if (p.cap) CK(cudaMemcpy(sh.data(), p.slot_h, p.cap * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (p.n_h) CK(cudaMemcpy(halo.data(), p.halo, p.n_h * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (node_ids)
        for (int64_t s = 0; s < p.cap; ++s) node_ids[s] = halo[sh[s]];
    if (se && p.cap) CK(cudaMemcpy(se, p.se, p.cap * sizeof(float), cudaMemcpyDeviceToHost));
    if (sa && p.n_h) CK(cudaMemcpy(sa, p.sa, p.n_h * sizeof(float), cudaMemcpyDeviceToHost));
    if (slot_of && p.n_h) CK(cudaMemcpy(slot_of, p.slot_of, p.n_h * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (rows && p.cap && ctx->D)
        CK(cudaMemcpy2D(rows, ctx->D * sizeof(float), p.rows, ctx->pitch * sizeof(float), ctx->D * sizeof(float), p.cap,
                        cudaMemcpyDeviceToHost));
    return MGNN_OK;
}

// ------------------------------------------------------------------ profiling
mgnn_status mgnn_profile_kernels(int32_t enable, char* report, int64_t report_len) {
    if (!enable && report && report_len > 0) {
        std::vector<std::pair<std::string, std::pair<double, long long>>> agg;
        for (auto& r : g_kprof_recs) {
            float ms = 0.0f;
            if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
            bool found = false;
            for (auto& a : agg)
                if (a.first == r.who) {
                    a.second.first += ms;
                    a.second.second += 1;
                    found = true;
                }
            if (!found) agg.push_back({r.who, {ms, 1}});
        }
        std::string out;
        for (auto& a : agg) {
            char line[256];
            snprintf(line, sizeof(line), "%-28s %10.3f ms %8lld calls %9.2f us/call\n", a.first.c_str(), a.second.first,
                     a.second.second, 1e3 * a.second.first / (double)a.second.second);
            out += line;
        }
        if (getenv("MGNN_KPROF_TIMELINE") && !g_kprof_recs.empty()) {   // end time of every launch (us) on
            out += "timeline (launcher stream end_us):\n";                 // one clock, base = first event
            std::vector<cudaStream_t> ss;
            for (auto& r : g_kprof_recs) {
                float ms = 0.0f;
                if (cudaEventElapsedTime(&ms, g_kprof_recs.front().a, r.b) != cudaSuccess) continue;
                int si = -1;
                for (size_t i = 0; i < ss.size(); ++i)
                    if (ss[i] == r.s) si = (int)i;
                if (si < 0) {
                    si = (int)ss.size();
                    ss.push_back(r.s);
                }
                char line[128];
                snprintf(line, sizeof(line), "%s %d %.1f\n", r.who, si, 1e3 * ms);
                out += line;
            }
        }
        snprintf(report, (size_t)report_len, "%s", out.c_str());
    }
    {   // every event exactly once: each record's start is the previous record's end (or a stream's first event)
        std::vector<cudaEvent_t> all;
        for (auto& r : g_kprof_recs) {
            all.push_back(r.a);
            all.push_back(r.b);
        }
        for (auto& l : g_kprof_last) all.push_back(l.second);
        std::sort(all.begin(), all.end());
        all.erase(std::unique(all.begin(), all.end()), all.end());
        cudaDeviceSynchronize();
        for (cudaEvent_t e : all) cudaEventDestroy(e);
        g_kprof_recs.clear();
        g_kprof_last.clear();
    }
    g_kprof = enable != 0;
    return MGNN_OK;
}

mgnn_status mgnn_profile_enable(mgnn_ctx ctx, int32_t enable) {
    if (!ctx) return MGNN_EINVAL;
    ctx->prof = enable == 2 ? 2 : (enable != 0 ? 1 : 0);
    return MGNN_OK;
}

static mgnn_status drain_events(mgnn_ctx ctx, int stage, double* ms, long long* n) {
    double tot = 0.0;
    for (auto& e : ctx->prof_ev[stage]) {
        CK(cudaEventSynchronize(e.second));
        float x = 0.0f;
        CK(cudaEventElapsedTime(&x, e.first, e.second));
        tot += x;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    *n = (long long)ctx->prof_ev[stage].size();
    ctx->prof_ev[stage].clear();
    *ms = tot;
    return MGNN_OK;
}

mgnn_status mgnn_profile_stages(mgnn_ctx ctx, double* out, int32_t n_out) {
    GUARD();
    if (!out || n_out < MGNN_PROF_N) return fail(ctx, MGNN_EINVAL, "profile_stages: need MGNN_PROF_N doubles");
    double ms[4];
    long long n[4];
    for (int st = 0; st < 4; ++st) {
        mgnn_status r = drain_events(ctx, st, &ms[st], &n[st]);
        if (r) return r;
    }
    long long su[6] = {0, 0, 0, 0, 0, 0}, rows = 0;
    CK(cudaMemcpy(su, ctx->d_sampled, sizeof(su), cudaMemcpyDeviceToHost));
    CK(cudaMemset(ctx->d_sampled, 0, sizeof(su)));
    CK(cudaMemcpy(&rows, ctx->d_gathered, sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemset(ctx->d_gathered, 0, sizeof(long long)));
    for (int i = 0; i < n_out; ++i) out[i] = 0.0;
    out[MGNN_PROF_SAMPLE_MS] = ms[0];
    out[MGNN_PROF_SAMPLE_CALLS] = (double)n[0];
    out[MGNN_PROF_EDGES] = (double)su[0];
    out[MGNN_PROF_FRONTIER] = (double)su[1];
    out[MGNN_PROF_UNIQUE] = (double)su[2];
    out[MGNN_PROF_GATHER_MS] = ms[1];
    out[MGNN_PROF_GATHER_CALLS] = (double)n[1];
    out[MGNN_PROF_GATHER_ROWS] = (double)rows;
    out[MGNN_PROF_SCORE_MS] = ms[2];
    out[MGNN_PROF_SCORE_CALLS] = (double)n[2];
    out[MGNN_PROF_HITS] = (double)su[3];
    out[MGNN_PROF_MISSES] = (double)su[4];
    out[MGNN_PROF_RELABEL_MS] = ms[3];
    out[MGNN_PROF_RELABEL_CALLS] = (double)n[3];
    out[MGNN_PROF_RELABEL_PROBES] = (double)su[5];
    return MGNN_OK;
}

mgnn_status mgnn_profile_read(mgnn_ctx ctx, double* ms, int64_t* launches, int64_t* bytes) {
    GUARD();
    double tot = 0.0;
    long long n = 0;
    mgnn_status r = drain_events(ctx, 1, &tot, &n);
    if (r) return r;
    long long rows = 0;
    CK(cudaMemcpy(&rows, ctx->d_gathered, sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemset(ctx->d_gathered, 0, sizeof(long long)));
    if (ms) *ms = tot;
    if (launches) *launches = n;
    if (bytes) *bytes = 2ll * rows * ctx->D * (long long)sizeof(float);
    return MGNN_OK;
}

}  // extern "C"
