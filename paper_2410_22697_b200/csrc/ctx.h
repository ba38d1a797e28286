// ctx.h -- internal: the context behind mgnn_ctx (include/mgnn.h) and the host helpers shared by
// api.cu (pipeline calls) and api_sage.cu (consumer / training calls).  Not part of the ABI.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mgnn.h"
#include "launch.h"

namespace mgnn {
namespace host {

struct Part {
    int32_t part_id = -1;
    int64_t lo = 0, n_local = 0, n_h = 0, h_below = 0, nnz = 0, n_train = 0, cap = 0, nbatch = 1;
    int32_t max_deg_in = 0;
    int32_t perm_slots = 0;
    int64_t* indptr = nullptr;
    int32_t* cols_rank = nullptr;
    int32_t* halo_map = nullptr;         // NEXT-1: [n_global] halo index or -1
    int64_t n_h_true = 0;                // |V_p^h| (deg_in > 0): the basis of |BUF| also with dense scores
    int32_t* halo = nullptr;
    int32_t* deg_in = nullptr;
    int32_t* train = nullptr;
    float* table = nullptr;
    float* rows = nullptr;
    float* se = nullptr;
    float* sa = nullptr;
    int32_t* slot_of = nullptr;
    int32_t* slot_h = nullptr;
    unsigned long long* hitmask = nullptr;
    int32_t* rank_deg = nullptr;
    int32_t* deg_order = nullptr;        // inverse of rank_deg (R lists are compacted in this order)
    int32_t* perm = nullptr;
    int32_t perm_chunk = 1;              // G: epoch orders generated per sort call
    int64_t chunk_loaded[2] = {-1, -1};  // chunk id c (epochs [cG, cG+G)) held by ring half c % 2
    // sort buffers: E (cap) / R (n_h) for eviction; R also serves buffer init; P (n_train) for epoch orders
    unsigned long long *ek = nullptr, *ekt = nullptr, *rk = nullptr, *rkt = nullptr, *pk = nullptr, *pkt = nullptr;
    uint32_t *ev = nullptr, *evt = nullptr, *rv = nullptr, *rvt = nullptr, *pvt = nullptr;
};

struct Win {
    bool alloc = false, sampled = false, gathered = false, scored = false;
    bool x_user = false;            // X is a caller-owned buffer (mgnn_window_bind_x)
    bool relabel_pending = false;   // sampled with the relabel deferred (mgnn_relabel not yet called)
    int32_t n_steps = 0;
    uint64_t step0 = 0;
    int32_t* fr_rank = nullptr;
    int32_t* fr_gid = nullptr;
    int64_t* hop_size = nullptr;
    int64_t* off[kMaxLayers] = {};
    int32_t* cols[kMaxLayers] = {};
    float* X = nullptr;
    int2* seedpos = nullptr;        // [M][H] seed positions (inside the zeroed region)
    uint32_t* nb = nullptr;         // [M][L][bm_words][2] new-node bits + word positions (zero region)
    char* zero = nullptr;           // [scan scratch | counts | fb], zeroed per window
    size_t zero_bytes = 0;
    unsigned long long* status = nullptr;
    int32_t* tilectr = nullptr;
    int32_t* gctr = nullptr;        // [M] gather chunk counters (dynamic claiming)
    long long* counts = nullptr;
    uint32_t* fb = nullptr;
    uint32_t* fbp = nullptr;        // [M][bm_words] frontier membership before the current hop
    int32_t* ext_seeds = nullptr;
    int32_t* ext_counts = nullptr;
    // scratch sub-regions
    Scratch sc_count[kMaxLayers], sc_compact[kMaxLayers];
};

}  // namespace host
}  // namespace mgnn

using namespace mgnn;          // internal header: the context below is written in the library's types

namespace mgnn {
namespace host {
// SM partition (partition.cu): green contexts [0] gather + scoring, [1] sampling + relabel, and one
// stream per call kind: 0 = mgnn_sample, 1 = mgnn_relabel (both on [1]), 2 = gather / score (on [0])
constexpr int kPartStreams = 3;
inline int part_of_stream(int i) { return i == 2 ? 0 : 1; }
struct SmPartition {
    bool on = false;
    void* gc[2] = {nullptr, nullptr};    // CUgreenCtx
    int sms[2] = {0, 0};
    cudaStream_t s[kPartStreams] = {};
    cudaEvent_t ev_in[kPartStreams] = {}, ev_out[kPartStreams] = {};
};
}  // namespace host
}  // namespace mgnn

struct mgnn_ctx_s {
    int device = 0;
    int32_t P = 0;
    int64_t n_global = 0;
    std::vector<int64_t> bounds;
    int32_t D = 0, pitch = 0;
    uint64_t feat_seed = 0;
    std::vector<mgnn::host::Part> parts;
    std::vector<int32_t> lp_of;          // part id -> local index or -1
    std::vector<const float*> tables;    // device-accessible table per partition
    std::vector<void*> ipc_opened;
    int64_t* d_bounds = nullptr;
    const float** d_tables = nullptr;
    uint8_t* d_on_peer = nullptr;        // [P]: table imported from another process (NVLink)
    int8_t* d_lp_of = nullptr;           // [P]: local index of each partition hosted here, else -1
    // TMA row-gather descriptors (k_gather_g4): [0, n_lp) tables, [n_lp, 2 n_lp) BUF rows; built by
    // mgnn_buffer_init (the BUF rows live there); g4_ok = every descriptor encoded
    GatherMaps gmaps{};
    bool g4_ok = false;
    PartDev* d_parts = nullptr;
    int32_t* d_err = nullptr;
    unsigned long long* d_ovf = nullptr; // first step of the first window that overflowed its arena (~0: none)
    long long* d_gathered = nullptr;
    // policy
    bool buffer_ready = false;
    mgnn_policy pol{};
    // eviction scratch
    SortSeg* d_evsegs = nullptr;
    SortSeg* d_candsegs = nullptr;       // the compacted candidates (E: all 8 key bytes; R: as d_evsegs)
    SortSeg* d_candsegs_hi = nullptr;    // candidates in list order (k_cand_ord): the score digits only
    SortSeg* d_initsegs = nullptr;
    bool force_sort_path = false;        // MGNN_EVICT_SORT=1: always use the radix-sort eviction path
    bool ev_scan = false;
    bool no_fused_decay = false;         // MGNN_FUSED_DECAY=0: k_decay stays a launch of its own on eviction windows                // MGNN_EV_SELECT=0: no ordered lists, scoreboard scans
    bool sort_full_lists = false;        // MGNN_EVICT_SORT=2: sort the whole E / R lists, not the candidates
    int32_t ev_passes = 8;
    long long* d_sel_n = nullptr;
    char* ev_zero = nullptr;
    size_t ev_zero_bytes = 0;
    Scratch ev_sc{};
    Scratch ev_sc2{};                  // k_cand_ord's look-back (same round as k_select's)
    EvScratch ev_ev{};
    int64_t ev_tiles = 1;
    void* sort_scr = nullptr;            // radix sort scratch of init / eviction (buffer stream)
    size_t sort_scr_bytes = 0;
    void* perm_scr = nullptr;            // radix sort scratch of epoch orders (sampling stream), so
    size_t perm_scr_bytes = 0;           // mgnn_sample may run concurrently with gather/score
    // NEXT-1 remote expansion: global CSR over every partition (all hosted by this context)
    bool remote = false;
    bool dense = false;                  // NEXT-1 dense S_A: every non-local node scorable
    int64_t* g_indptr = nullptr;
    int32_t* g_cols = nullptr;
    int64_t g_nnz = 0;
    // sampler
    bool configured = false;
    int32_t L = 0, batch = 0, max_window = 0;
    int32_t fan[kMaxLayers] = {}, k_hop[kMaxLayers] = {};
    uint64_t run_seed = 0;
    int64_t ucap = 0, vp_max = 0, bm_words = 0;
    int64_t rows_bound = 0;              // arena bound on |F_i| per instance (0 = the static worst case)
    int32_t seed_h = 1;                  // seed-position hash slots per instance
    int64_t fcap[kMaxLayers + 1] = {}, ecap[kMaxLayers] = {};
    mgnn::host::Win win[2];
    SortSeg* d_permsegs = nullptr;       // [n_lp][max perm slots]
    int32_t perm_slots_max = 0;
    long long* d_perm_n = nullptr;       // [n_lp]
    // A14 consumer (GraphSAGE-mean): padded weights [npad][2*kp] = [W_self | W_neigh], bias [npad],
    // ping-pong hidden buffers, and the TMA tensor maps of every operand (128 B each)
    struct Sage {
        bool ready = false;
        int32_t L = 0;
        int32_t dims[kMaxLayers + 1] = {};
        int32_t npad[kMaxLayers] = {}, kp[kMaxLayers] = {};
        // parameters: one buffer, layer l = Wcat [npad][2 kp] at w_off[l], bias [npad] at b_off[l]
        float* params = nullptr;
        int64_t n_params = 0, w_off[kMaxLayers] = {}, b_off[kMaxLayers] = {};
        float* w[kMaxLayers] = {};
        float* b[kMaxLayers] = {};
        float* h[kMaxLayers] = {};                // hidden outputs H^{l+1}, l < L-1: [M][out_rows][npad]
        int64_t out_rows[kMaxLayers] = {};        // rows per instance of layer l's output buffer (= fcap[h])
        alignas(64) unsigned char map_w[kMaxLayers][128];
        // 3xTF32 forward GEMM (default; MGNN_SAGE_TF32=1: one TF32 pass): Wcat = W_hi + W_lo, refreshed
        // with every weight update (mgnn_sage_config, k_sgd_layers)
        bool split3 = true;
        float* w3 = nullptr;                      // [W_hi of every layer | W_lo of every layer]
        float* whi[kMaxLayers] = {};
        float* wlo[kMaxLayers] = {};
        alignas(64) unsigned char map_whi[kMaxLayers][128], map_wlo[kMaxLayers][128];
        alignas(64) unsigned char map_in[2][kMaxLayers][128];   // [window slot][layer]
        // training (NEXT-3)
        bool train = false;
        int32_t* labels = nullptr;                // [n_global]
        float* grads = nullptr;                   // same layout as params
        float* wt[kMaxLayers] = {};               // transposed Wcat: [2 kp][npad] (dgrad operand)
        float* mean[kMaxLayers] = {};             // [M][out_rows][kp] neighbour means
        float* logits = nullptr;                  // [M][rows64][npad_L]
        float* dlogits = nullptr;
        float* dh[kMaxLayers] = {};               // gradient of h[l]: [M][dh_rows[l]][npad[l]]
        float* dmean = nullptr;                   // dZ W_neigh / deg of the current layer (dgrad -> scatter)
        float* loss = nullptr;                    // device scalar
        cudaStream_t side = nullptr;              // weight gradients run beside the input-gradient chain
        cudaEvent_t ev_fork[kMaxLayers] = {}, ev_join = nullptr, ev_start = nullptr, ev_zero = nullptr;
        int64_t rows64 = 0, dh_rows[kMaxLayers] = {};
        alignas(64) unsigned char map_dz128[kMaxLayers][128], map_wt[kMaxLayers][128], map_mean128[kMaxLayers][128];
    } sage;
    bool defer_relabel = false;          // mgnn_sample leaves the columns in rank space (mgnn_relabel)
    // ordering of windows through the buffer
    bool seq_started = false;
    uint64_t next_step = 0;
    // status
    int sticky = MGNN_OK;
    std::string err;
    // profiling
    int prof = 0;                        // 1: every stage timed by events, 2: only the gather launch
    // event pairs per stage: 0 = sampler kernels (k_hop, k_compact, k_relabel) of mgnn_sample,
    // 1 = the gather launch of mgnn_lookup_gather, 2 = all of mgnn_score_evict_refill
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[4];   // [3] = deferred k_relabel
    long long* d_sampled = nullptr;      // [6] sampled edges E, expanded frontier F, |F_L| U, hits, misses,
                                         //     k_relabel's (bits, position) / seed-hash probes
    mgnn::host::SmPartition smp;         // mgnn_sm_partition
};

namespace mgnn {
namespace host {

mgnn_status fail(mgnn_ctx c, mgnn_status st, const std::string& msg);

// Runs one API call's kernels on its SM-partition stream when a partition is set (else on the
// caller's stream): `s` is the stream to launch on; the destructor hands ordering back to the caller.
struct PartScope {
    mgnn_ctx ctx;
    int idx;
    cudaStream_t caller_s, s;
    bool active = false, err = false;
    PartScope(mgnn_ctx c, int which, cudaStream_t caller);
    ~PartScope();
    PartScope(const PartScope&) = delete;
    PartScope& operator=(const PartScope&) = delete;
};
void partition_free(mgnn_ctx ctx);

#define CK(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? MGNN_ENOMEM : MGNN_ECUDA,            \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                        \
    } while (0)

#define CKL()                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = cudaGetLastError();                                                         \
        if (e_ != cudaSuccess) return fail(ctx, MGNN_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

#define GUARD()                                                                                      \
    do {                                                                                             \
        if (!ctx) return MGNN_EINVAL;                                                                \
        if (ctx->sticky) return (mgnn_status)ctx->sticky;                                            \
        if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MGNN_ECUDA, "cudaSetDevice"); \
    } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t n) {
    if (n == 0) n = 1;
    return cudaMalloc((void**)p, n * sizeof(T));
}

template <class T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

inline int64_t sat_mul(int64_t a, int64_t b, int64_t cap) {
    if (a == 0 || b == 0) return 0;
    if (a > cap / b) return cap;
    int64_t r = a * b;
    return r > cap ? cap : r;
}

void fill_partdev(const mgnn_ctx_s* c, const Part& p, PartDev* d);
mgnn_status upload_parts(mgnn_ctx ctx);
mgnn_status upload_tables(mgnn_ctx ctx);
WorldDev world_of(mgnn_ctx ctx);
void free_win(Win& w);
void free_sage(mgnn_ctx_s* ctx);           // api_sage.cu
mgnn_status rebind_sage_input(mgnn_ctx ctx, int slot);   // api_sage.cu: re-encode layer 0's X descriptor
void free_buffer(Part& p);
void free_perm(Part& p);
mgnn_status ensure_scratch(mgnn_ctx ctx, void** p, size_t* have, size_t bytes);
WinDev win_dev(mgnn_ctx ctx, Win& w);

}  // namespace host
}  // namespace mgnn
