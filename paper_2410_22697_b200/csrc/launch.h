// launch.h -- host-side launch wrappers shared by the .cu units of libmgnn.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>

#include "common.cuh"

namespace mgnn {

constexpr int kMaxLayers = MGNN_MAX_LAYERS;

// Kernel launches issued by the library (process-wide; bench evidence).
// With MGNN_DEBUG_SYNC=1 in the environment every launcher synchronises and
// reports the first failing kernel by name (debug aid, never on by default).
// With per-kernel profiling on (mgnn_profile_kernels), an event is recorded after every launcher
// and the time since the previous event on the same stream is attributed to that launcher.
void count_launches(long long n, const char* who, cudaStream_t s);
long long launches_total();

// SM count of the current device (cudaDevAttrMultiProcessorCount, cached per device): every grid is
// sized from it instead of assuming B200's 148.
int num_sms();
// Opt-in dynamic shared memory for `func` on the CURRENT device: raised to `bytes` once per
// (device, kernel) -- the attribute is per device, so a second context on another GPU sets it again.
// Thread-safe.  Returns the CUDA error of the attribute call (cudaSuccess if already set).
cudaError_t ensure_smem(const void* func, int bytes);
template <typename F>
inline cudaError_t ensure_smem_k(F* func, int bytes) {
    return ensure_smem(reinterpret_cast<const void*>(func), bytes);
}

// ------------------------------------------------------------------ window (device view)
struct WinDev {
    int32_t n_inst, n_steps, L, batch, pitch, feat_dim;
    uint64_t step0;
    uint32_t seed_lo, seed_hi;           // run seed (Philox key, R#4)
    int32_t k_hop[kMaxLayers];           // fanout drawn at hop i (R#2)
    int64_t ucap;                        // rows per instance (X, frontier)
    int64_t off_stride[kMaxLayers];      // offsets row stride per hop (>= fcap_i + 1)
    int64_t col_stride[kMaxLayers];      // cols stride per hop (= ecap_i)
    int32_t seed_hmask;                  // seed-position hash: slots per instance - 1 (power of two >= 2 B)
    int64_t bm_words;                    // bitmap words per instance
    int32_t* fr_rank;                    // [M][ucap]
    int32_t* fr_gid;                     // [M][ucap]
    int64_t* hop_size;                   // [M][kMaxLayers+1]
    int64_t* off[kMaxLayers];
    int32_t* cols[kMaxLayers];
    float* X;                            // [M][ucap][pitch]
    long long* counts;                   // [M][8]
    int32_t* gctr;                       // [M] gather chunk counters (zeroed per window)
    int2* seedpos;                       // [M][seed_hmask+1] (rank + 1, position in F_0): open addressing,
                                         // zeroed per window -- the seeds' positions for k_relabel
    unsigned long long* ovf;             // smallest first step of a window whose frontier exceeded its
                                         // arena bound (~0 = none); that window and later ones are skipped
                                         // by every kernel that changes buffer state
    uint32_t* fb;                        // [M][bm_words] frontier membership (cumulative: F_i, then F_{i+1})
    uint32_t* fbp;                       // [M][bm_words] membership of F_i while hop i runs (new_i = fb & ~fbp)
    uint32_t* nb;                        // [M][L][bm_words][2]: new_i bits of hop i (R#7) and the position
                                         // in F_{i+1} of the word's first new node (one 8-byte pair);
                                         // written in full by k_compact (never zeroed)
    const int32_t* ext_seeds;            // [M][batch] or nullptr
    const int32_t* ext_counts;           // [M]
    const PartDev* parts;                // [n_parts_local]
    int32_t* err;                        // device error word
    long long* gathered_rows;            // profiling counter
    long long* sampled_units;            // profiling: [3] += E, F, U of every instance (k_relabel)
    long long* prof_hm;                  // profiling: [2] += hits, misses of every gathered instance
    // NEXT-1 remote expansion: ranks are global ids; every frontier node is sampled from the
    // global CSR (all partitions hosted by this context)
    int32_t remote;
    int64_t n_global;
    const int64_t* g_indptr;             // [n_global+1]
    const int32_t* g_cols;               // [nnz] global ids
    int32_t idx32;                       // every CSR index the sampler reads fits in 32 bits
};

// Segment of a radix sort (device array of these).
struct SortSeg {
    unsigned long long* keys;    // primary (result ends here after an even number of passes)
    uint32_t* vals;
    unsigned long long* keys_tmp;
    uint32_t* vals_tmp;
    const long long* n;          // device element count
    int32_t npass;               // even number of 8-bit digit passes for this segment
    uint8_t shift[8];            // bit offset of each pass's digit, least significant first
};

// Digit schedule: the key bytes that can differ, least significant first.  The caller
// guarantees every other byte is constant and passes an EVEN number of shifts (so the
// sorted data ends in the primary buffers).
inline SortSeg make_seg(unsigned long long* k, uint32_t* v, unsigned long long* kt, uint32_t* vt, const long long* n,
                        std::initializer_list<int> shifts) {
    SortSeg s{k, v, kt, vt, n, 0, {0, 0, 0, 0, 0, 0, 0, 0}};
    for (int sh : shifts) s.shift[s.npass++] = (uint8_t)sh;
    return s;
}

struct Scratch {          // zeroed look-back status words + tile counters
    unsigned long long* status;
    int32_t* tilectr;
};

struct EvScratch {        // eviction-round scratch, zeroed per round
    uint32_t* hist;                 // [2*n_lp][4096] histogram of key >> 52
    uint32_t* hist2;                // [2*n_lp][4096] bits [40,52) inside the threshold bucket
    unsigned* ticket;               // last-block detection of k_select
    long long* thr;                 // [2*n_lp][2] = {K, threshold digit T (-1: none)}
    unsigned long long* n_cand;     // [2*n_lp] candidates appended by k_cand
    unsigned long long* kth;        // [2*n_lp][2] {1, exact K-th smallest key} when k_tie resolved ties, else 0
};

// Launch with programmatic stream serialization (PDL) unless MGNN_PDL=0; the kernel must call
// pdl_enter() before its first global-memory access.
bool pdl_enabled();
template <typename... P, typename... A>
inline void launch_k(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// sample.cu
void launch_seeds(const WinDev& w, cudaStream_t s);
void launch_hop(const WinDev& w, int hop, int64_t fcap, Scratch sc, cudaStream_t s);
void launch_compact(const WinDev& w, int hop, Scratch sc, cudaStream_t s);
void launch_relabel(const WinDev& w, cudaStream_t s);
int64_t scan_tiles_count(int64_t fcap);   // tiles used by count_scan for fcap items
int64_t scan_tiles_words(int64_t words);  // tiles used by compact for `words`

// gather.cu
// TMA row-gather descriptors of the sources on this GPU: maps[lp] = table of local partition lp,
// maps[n_lp + lp] = its BUF rows (2-D fp32 [rows][D], box {D, 1}, for cp.async.bulk.tensor gather4).
constexpr int kMaxGatherMaps = 16;
struct alignas(64) GatherMaps {
    unsigned char maps[kMaxGatherMaps][128];
    int32_t n_lp;
};
void launch_gather(const WinDev& w, const WorldDev& world, bool l2_resident, const GatherMaps* g4, cudaStream_t s);
// sage.cu: 2-D fp32 row map for the gather4 path (box = one whole row of `cols` floats)
bool encode_row_map(void* map_out, const float* base, int64_t rows, int64_t cols, int64_t pitch);

// score.cu
// ovf / t_last: the window is skipped when *ovf <= t_last (arena overflow, mgnn_sampler_config_bounded)
void launch_decay(const PartDev* parts, int n_lp, int64_t cap_max, int n_steps, float gamma,
                  const unsigned long long* ovf, uint64_t t_last, cudaStream_t s);
void launch_select(const PartDev* parts, int n_lp, int64_t n_max, float alpha, float theta_r, const SortSeg* segs,
                   long long* n_out, Scratch sc, EvScratch ev, cudaStream_t s, int decay_steps = 0, float gamma = 1.0f,
                   const unsigned long long* ovf = nullptr, uint64_t t_last = 0);
// |E|, |R| and the top-digit histograms straight from the scoreboards (no ordered lists)
void launch_ev_count(const PartDev* parts, int n_lp, int64_t n_max, float alpha, float theta_r, long long* n_out,
                     EvScratch ev, cudaStream_t s);
// small-buffer path: candidates below the threshold digit, ranked by counting into sorted order.
// scan_parts != nullptr: candidates are re-derived from the scoreboards (after launch_ev_count);
// nullptr: from the compacted lists of launch_select.
void launch_cand_rank(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, const PartDev* scan_parts,
                      float alpha, float theta_r, cudaStream_t s);
void launch_cand_ord(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, Scratch sc, int64_t tiles_max,
                     cudaStream_t s);
void launch_cand(const SortSeg* segs, int n_lp, int64_t n_max, EvScratch ev, const PartDev* scan_parts, float alpha,
                 float theta_r, cudaStream_t s);   // candidates only
void launch_swap_refill(const PartDev* parts, int n_lp, int64_t cap_max, const SortSeg* segs, const long long* k_of,
                        const WorldDev& world,
                        long long* counts, int64_t inst_stride_counts, int n_steps, const unsigned long long* ovf,
                        uint64_t t_last, cudaStream_t s);
// |BUF| up to which the candidate-rank path (no sort) is used for eviction rounds
constexpr int kEvMax = 65536;
void launch_init_keys(const PartDev* pd_dev, int64_t n_h, const SortSeg* seg, long long* n_dev, cudaStream_t s);
void launch_init_fill(const PartDev* pd_dev, int64_t n_h, int64_t cap, const uint32_t* order, cudaStream_t s);
void launch_rows_from_owners(const PartDev* pd_dev, int64_t cap, const WorldDev& world, cudaStream_t s);
// n_epochs consecutive epoch orders (epoch0 ...) into segs[j].vals; keys / keys_tmp / vals_tmp
// are work buffers of n_train each; scratch holds 2 * 256 * n_epochs counters (zeroed here)
void launch_perm_build(const PartDev* pd_dev, int64_t n_train, uint64_t epoch0, int n_epochs, uint32_t seed_lo,
                       uint32_t seed_hi, const SortSeg* segs, void* scratch, cudaStream_t s);

// sort.cu: stable LSD radix sort of (u64 key, u32 value) pairs, each segment with its own digit
// schedule (SortSeg::shift, at most max_passes); n_max bounds every segment's length.
void radix_sort_pairs(const SortSeg* segs_dev, int n_seg, int64_t n_max, int max_passes, void* scratch, cudaStream_t s);
size_t radix_scratch_bytes(int n_seg, int64_t n_max, int max_passes);

// sage.cu: GraphSAGE-mean consumer (A14), one launch per layer over every instance of a window
struct SageLayerArgs {
    int32_t n_inst;
    int32_t hop;               // block of hop h: dst F_h, src positions in F_{h+1}
    int32_t k_in;              // input features (columns of H_in that carry data)
    int32_t n_panels;          // ceil(k_in / panel width), set by the launcher
    int32_t kp;                // K offset of W_neigh inside Wcat (k_in rounded up to 128)
    int32_t npad;              // UMMA N (multiple of 16, <= 256)
    int32_t n_out;             // columns written per output row (npad for hidden, C for logits)
    int32_t relu;
    int32_t k_hop;             // fanout of the hop (max neighbours per dst row)
    int32_t stages;            // weight-chunk ring depth
    uint32_t idesc;
    uint32_t tmem_cols;
    const int64_t* hop_size;   // [M][kMaxLayers+1]
    const int64_t* off;        // [M][off_stride]
    int64_t off_stride;
    const int32_t* cols;       // [M][col_stride]
    int64_t col_stride;
    const float* h_in;         // [M][in_rows][in_pitch]
    int64_t in_rows, in_pitch;
    float* h_out;              // [M][out_rows][out_pitch]
    int64_t out_rows, out_pitch;
    const float* bias;         // [npad], zero padded
    int32_t inst0, inst_step;  // kernel instance k is window instance inst0 + k * inst_step
    float* mean_out;           // optional [M][mean_rows][mean_pitch]: neighbour means (training)
    int64_t mean_rows, mean_pitch;
    int32_t b_resident;        // k_sage_gemm: all weight chunks stay in shared memory (set by the launcher)
    int32_t split3;            // k_sage_gemm: 3xTF32 (A_hi W_hi + A_hi W_lo + A_lo W_hi), fp32-grade products
};
bool sage_encode_map(void* map_out, const float* base, int64_t rows, int64_t cols, int64_t pitch, int box_rows);
bool launch_sage_layer(const void* map_in, const void* map_w, const SageLayerArgs& a, cudaStream_t s);
// out = act([H_in | mean] Wcat^T + b) with the means precomputed (warp-specialised, TMA + tcgen05)
// map_w is W_hi (low 13 mantissa bits zero) and map_wlo W - W_hi when a.split3, else map_w = W, map_wlo unused
bool launch_sage_gemm(const void* map_in, const void* map_w, const void* map_wlo, const void* map_mean,
                      const SageLayerArgs& a, cudaStream_t s);
// hi = w with the low 13 mantissa bits cleared (exactly a TF32 value), lo = w - hi (exact), n floats
void launch_split_tf32(const float* w, float* hi, float* lo, int64_t n, cudaStream_t s);
// neighbour means of a layer's dst rows into mean_out (warp per row, all SMs): the training step's
// forward, whose per-step instance count is too small for the fused aggregation to fill the GPU
void launch_mean(const SageLayerArgs& a, cudaStream_t s);

// train.cu: backward of the GraphSAGE-mean consumer (NEXT-3: loss, weight and input gradients)
struct XentArgs {
    int32_t n_inst, inst0, inst_step, n_classes;
    const int64_t* hop_size;   // [M][kMaxLayers+1] (|F_0| = hop_size[m][0])
    const int32_t* frontier;   // [M][ucap] global ids (F_0 prefix)
    int64_t ucap;
    const int32_t* labels;     // [n_global]
    const float* logits;       // [M][rows][pitch]
    float* dlogits;            // [M][rows][pitch]
    int64_t rows, pitch;
    float scale;               // 1 / (trainers in the DDP step)
    float* db;                 // [pitch] bias gradient of the last layer (accumulated)
    float* loss;               // device scalar (accumulated: sum over trainers of mean loss, times scale)
};
void launch_xent(const XentArgs& a, cudaStream_t s);

struct MaskArgs {              // dZ = dH * [H > 0] over rows < hop_size[m][hop], column sums -> db
    int32_t n_inst, inst0, inst_step, hop;
    const int64_t* hop_size;
    float* dz;                 // [M][rows][pitch] in place (holds dH on entry)
    int64_t rows, pitch;
    const float* h;            // [M][h_rows][h_pitch] layer output H
    int64_t h_rows, h_pitch;
    int32_t ncols;             // columns carrying data (npad)
    float* db;                 // [pitch]
};
void launch_relu_mask(const MaskArgs& a, cudaStream_t s);

struct ZeroRowsArgs {          // buf[m][r][*] = 0 for r < hop_size[m][hop]
    int32_t n_inst, inst0, inst_step, hop;
    const int64_t* hop_size;
    float* buf;
    int64_t rows, pitch;
};
void launch_zero_rows(const ZeroRowsArgs& a, cudaStream_t s);

struct WgradArgs {             // dW[npad][2 kp] += dZ^T [H | mean] over the step's rows
    int32_t n_inst, inst0, inst_step, hop;
    const int64_t* hop_size;
    const float* dz;           // [M][dz_rows][dz_pitch]
    int64_t dz_rows, dz_pitch;
    const float* h_in;         // [M][in_rows][in_pitch], in_cols columns carry data
    int64_t in_rows, in_pitch;
    int32_t in_cols;
    const float* mean;         // [M][mean_rows][mean_pitch]
    int64_t mean_rows, mean_pitch;
    int32_t mean_cols;
    int32_t kp, npad;
    float* dw;                 // [npad][2 kp]
    int64_t max_chunks;        // upper bound of the step's 64-row chunks (host hint for the K split)
    int32_t ksplit;            // CTAs per (M-tile, N-tile), set by the launcher
    int32_t split3;            // 3xTF32 (fp32-grade products), else one TF32 pass
};
bool launch_wgrad(const WgradArgs& a, cudaStream_t s);

struct DgradArgs {             // dH[i] += dZ_i W_self; dH[j] += dZ_i W_neigh / deg(i) for j in N(i)
    int32_t n_inst, inst0, inst_step, hop;
    const int64_t* hop_size;
    const int64_t* off;
    int64_t off_stride;
    const int32_t* cols;
    int64_t col_stride;
    int64_t dz_rows;           // rows per instance of dZ
    int32_t npad_out;          // K of the GEMM (dZ columns)
    int32_t kp;                // N of each half (input features, padded)
    int32_t k_in;              // input features with data
    float* dh;                 // [M][dh_rows][dh_pitch] (zeroed rows < |F_{h+1}|)
    int64_t dh_rows, dh_pitch;
    float* dmean;              // [M][dmean_rows][kp]: dZ_i W_neigh / deg(i), scattered by k_scatter
    int64_t dmean_rows;
    int32_t split3;            // 3xTF32: dZ and Wt tiles split into hi / lo in shared memory
};
bool launch_dgrad(const void* map_dz, const void* map_wt, const DgradArgs& a, cudaStream_t s);
// dH[j] += dmean[i] for every sampled neighbour j of dst row i (warp per row, vector atomics)
void launch_scatter(const DgradArgs& a, cudaStream_t s);

// W <- W - lr * g, g <- 0, and the transposed copy Wt[c][o] = W[o][c] (dgrad operand)
struct SgdLayers {             // per layer: Wcat [rows][cols] followed by the bias [rows]; Wt [cols][rows]
    int32_t n_layers;
    float* w[kMaxLayers];
    float* g[kMaxLayers];
    float* wt[kMaxLayers];
    float* whi[kMaxLayers];    // optional 3xTF32 split of the updated Wcat (k_sage_gemm operands)
    float* wlo[kMaxLayers];
    int64_t rows[kMaxLayers], cols[kMaxLayers];
};
void launch_sgd_layers(const SgdLayers& d, float lr, cudaStream_t s);
void launch_transpose(const float* w, float* wt, int32_t rows, int32_t cols, cudaStream_t s);

// load.cu
void launch_mark_halo(const int32_t* cols, int64_t nnz, int64_t lo, int64_t hi, uint32_t* bm, cudaStream_t s);
void launch_bitmap_to_ids(const uint32_t* bm, int64_t nwords, int32_t* out, long long* out_n, Scratch sc,
                          cudaStream_t s);
void launch_lower_bound(const int32_t* arr, int64_t n, int64_t v, long long* out, cudaStream_t s);
void launch_halo_index(const int32_t* halo, int64_t n_h, int32_t* gmap, cudaStream_t s);
void launch_deg_rank(const int32_t* cols, int64_t nnz, int64_t lo, int64_t n_local, int64_t h_below,
                     const int32_t* gmap, int32_t* deg_in, int32_t* cols_rank, cudaStream_t s);
void launch_features(float* table, int64_t lo, int64_t n_rows, int32_t dim, int32_t pitch, uint64_t feat_seed,
                     cudaStream_t s);
void launch_global_csr(const PartDev* pd_dev, const int64_t* indptr, int64_t n_local, int64_t lo, int64_t nnz,
                       int64_t base, int64_t* g_indptr, int32_t* g_cols, cudaStream_t s);

}  // namespace mgnn
