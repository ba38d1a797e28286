/* mgnn.h -- C ABI of the B200 halo feature pipeline of arXiv 2410.22697
 * ("MassiveGNN": continuous prefetch + eviction for distributed GNN minibatch
 * training).  PAPER.md line refs are "P:n"; readings "R#n" are listed in
 * DESIGN.md §Readings.
 *
 * One mgnn_ctx lives in one process and drives one GPU.  It hosts one or more
 * partitions p ("trainers"), each with its own CSR, feature table
 * (the KVStore), prefetch buffer BUF_p and scoreboards S_E, S_A
 * (P:111).  The unit of work is a WINDOW: `n_steps` consecutive global steps
 * t0..t0+n_steps-1 for every hosted partition ("instances" m = lp*n_steps+w).
 * A window may contain an eviction step (t % Delta == 0, R#14) only as its
 * last step, so buffer membership is constant inside it and the result is
 * bit-identical to running PREFETCH_WITH_EVICTION (Alg.2) step by step.
 *
 * Every call returns mgnn_status and never aborts.  EINVAL leaves the state
 * unchanged.  CUDA errors are sticky: the ctx is poisoned and every later call
 * returns MGNN_ECUDA (mgnn_last_error explains).  A ctx belongs to one host
 * thread; its device work is ordered on the stream the caller passes, so pass
 * the same stream to every call (or order streams with events).
 * All device memory is owned by the library; window outputs are exposed as
 * device pointers valid until the same window slot is sampled again.
 *
 * Typical sequence (one process per GPU; examples/train_ddp.py):
 *   mgnn_ctx_create -> mgnn_partition_load (each hosted partition)
 *   [multi-GPU: mgnn_table_export / mgnn_table_import of every other partition]
 *   mgnn_buffer_init -> mgnn_sampler_config
 *   per window w (two slots, so sampling runs ahead):
 *     mgnn_sample(slot w%2)               -- stream A, may run one window ahead
 *     mgnn_lookup_gather(slot)            -- stream B: X feature-ready (the measured path)
 *     [mgnn_sage_forward or, per step, mgnn_sage_train_step + all-reduce + mgnn_sage_sgd]
 *     mgnn_score_evict_refill(slot)       -- stream B: decay, eviction round at t % Delta == 0
 *     mgnn_counts_read[_async](slot)      -- hits / misses / rows fetched per minibatch
 */
#ifndef MGNN_H
#define MGNN_H
#include <stdint.h>

#if defined(__GNUC__)
#define MGNN_API __attribute__((visibility("default")))
#else
#define MGNN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mgnn_ctx_s* mgnn_ctx;
typedef void* mgnn_stream;  /* a cudaStream_t (0 = legacy default stream) */

typedef enum {
    MGNN_OK = 0,
    MGNN_EINVAL = 1,    /* bad argument; no state change */
    MGNN_ENOMEM = 2,    /* device allocation failed */
    MGNN_ECUDA = 3,     /* CUDA error (sticky) */
    MGNN_ESTATE = 5,    /* call-order violation (e.g. gather before sample) */
    MGNN_EOVERFLOW = 6  /* a frontier exceeded the arena bound of mgnn_sampler_config_bounded (not sticky:
                           the window and later ones were skipped; reconfigure and resume) */
} mgnn_status;

#define MGNN_MAX_LAYERS 8
#define MGNN_MAX_FANOUT 32
#define MGNN_IPC_HANDLE_BYTES 64

/* One partition p of G(V, E) (first-level partitioning).  Host memory,
 * read during mgnn_partition_load only; the caller keeps ownership.
 * V_p^l = [part_bounds[p], part_bounds[p+1]) (R#9). */
typedef struct {
    int32_t part_id;            /* p, 0 <= p < n_parts of the ctx */
    const int64_t* indptr;      /* [n_local+1], indptr[0] == 0: local rows of the symmetric CSR */
    const int32_t* cols;        /* [indptr[n_local]] global neighbour ids; each row strictly
                                   ascending, no self loops (simple graph) */
    const int32_t* train_ids;   /* [n_train] sorted, distinct, local training seeds */
    int64_t n_train;
} mgnn_partition_desc;

/* Prefetcher policy (Table 1; Eq.1). */
typedef struct {
    float gamma;     /* decay rate gamma, 0 < gamma <= 1 */
    float alpha;     /* eviction threshold alpha >= 0 (use mgnn_alpha_default for Eq.1, R#13) */
    float theta_r;   /* replacement eligibility S_A >= theta_r (R#17) */
    int32_t delta;   /* eviction interval Delta in steps; 0 = prefetch without eviction */
    uint32_t f_bp;   /* f_p^h in basis points, 0..10000; |BUF| = ceil(f*|V_p^h|) (R#11) */
} mgnn_policy;

/* Per-instance counters (int64), layout of mgnn_counts_read rows. */
enum {
    MGNN_C_NODES = 0,      /* |F_L| (unique sampled nodes incl. seeds, R#23) */
    MGNN_C_LOCAL = 1,      /* |F_L ∩ V_p^l|  (Alg.2 l.2) */
    MGNN_C_HIT = 2,        /* |Hits|         (Alg.2 l.4) */
    MGNN_C_MISS = 3,       /* |Misses|       (Alg.2 l.5) */
    MGNN_C_EVICTED = 4,    /* k of the eviction round ending at this step (Alg.2 l.14) */
    MGNN_C_REFILLED = 5,   /* = k (constant |BUF|) */
    MGNN_C_ROWS_FETCHED = 6, /* remote rows this step = misses + refills */
    MGNN_C_PEER_ROWS = 7,    /* of those, rows read from another GPU's table over NVLink */
    MGNN_C_N = 8
};

/* Device view of one window slot.  Instance m = lp*n_steps + w holds global
 * step t0+w of local partition lp.  All pointers are DEVICE pointers. */
typedef struct {
    int32_t n_inst, n_steps, n_parts_local, n_layers;
    uint64_t step0;
    int64_t rows_stride;        /* rows between consecutive instances in X / frontier */
    int64_t pitch;              /* floats per X row (feat_dim rounded up to 4) */
    const float* X;             /* [n_inst][rows_stride][pitch]: X[m][i] = feature row of F_L[i] (R#24) */
    const int32_t* frontier;    /* [n_inst][rows_stride]: F_L as global ids (F_0 = seeds) */
    const int64_t* hop_size;    /* [n_inst][MGNN_MAX_LAYERS+1]: |F_i|, i = 0..L */
    const int64_t* offsets[MGNN_MAX_LAYERS];  /* hop i: [n_inst][off_stride[i]]: CSR offsets over F_i */
    const int32_t* cols[MGNN_MAX_LAYERS];     /* hop i: [n_inst][col_stride[i]]: sampled neighbour as
                                                 its POSITION in F_{i+1} (DGL block layout) */
    int64_t off_stride[MGNN_MAX_LAYERS];
    int64_t col_stride[MGNN_MAX_LAYERS];
    const int64_t* counts;      /* [n_inst][MGNN_C_N] */
} mgnn_window;

/* Eq.1 with initial S_E = 1: alpha = gamma^Delta as the iterated fp32
 * product (R#13).  Pure host function. */
MGNN_API float mgnn_alpha_default(float gamma, int32_t delta);

/* Create a context on CUDA device `device` for a graph of n_global nodes cut
 * into n_parts contiguous ranges part_bounds[0..n_parts] (host array), with
 * feat_dim-wide fp32 features synthesised from feat_seed (R#4; the synthetic
 * stand-in for the dataset's node features). */
MGNN_API mgnn_status mgnn_ctx_create(int32_t device, int32_t n_parts, int64_t n_global, const int64_t* part_bounds,
                            int32_t feat_dim, uint64_t feat_seed, mgnn_ctx* out);
MGNN_API void mgnn_destroy(mgnn_ctx ctx);
MGNN_API const char* mgnn_last_error(mgnn_ctx ctx);

/* Load partition p onto the device (synchronous, one-time):
 * validates the CSR, builds V_p^h (sorted halo ids), deg_in (R#10), the
 * local-rank relabelling of the CSR, the train seeds and the feature table.
 * *local_index receives the partition's index lp among this ctx's partitions. */
MGNN_API mgnn_status mgnn_partition_load(mgnn_ctx ctx, const mgnn_partition_desc* desc, int32_t* local_index);

/* Feature tables of partitions hosted by OTHER processes (multi-GPU): export
 * writes a CUDA IPC handle (MGNN_IPC_HANDLE_BYTES) of local partition p's
 * table; import maps partition p's table from another process's handle so
 * that miss / refill rows are read directly over NVLink (peer loads inside
 * the gather kernels).  Tables of partitions in the same ctx need nothing. */
MGNN_API mgnn_status mgnn_table_export(mgnn_ctx ctx, int32_t part_id, void* handle_out);
MGNN_API mgnn_status mgnn_table_import(mgnn_ctx ctx, int32_t part_id, const void* handle);

/* INITIALIZE_PREFETCHER (Alg.1) for every hosted partition:
 * BUF = top ceil(f*|V_p^h|) halo nodes by (deg_in desc, id asc), rows fetched
 * from their owners, S_E = 1, S_A = -1 (buffered) / 0 (other halo).  Needs
 * every partition's table (local or imported), else ESTATE. */
MGNN_API mgnn_status mgnn_buffer_init(mgnn_ctx ctx, const mgnn_policy* policy, mgnn_stream stream);

/* Sampler configuration and window arenas: fanouts in GNN-layer order, input
 * layer first (R#2; hop i draws fanouts[n_layers-1-i]), batch size B, run seed
 * of the counter-based Philox streams (R#4), and the largest window. */
MGNN_API mgnn_status mgnn_sampler_config(mgnn_ctx ctx, const int32_t* fanouts, int32_t n_layers, int32_t batch,
                                uint64_t run_seed, int32_t max_window);

/* The same with REALISTIC window arenas: every frontier F_i (i >= 1) of an instance is given room
 * for at most rows_bound nodes (0 = the static worst case min(B * prod(1 + k_i), |V_p|), which
 * for ogbn-products-shaped graphs is ~12x the frontiers that occur and for papers100M does not fit
 * a window of 16 steps x 8 trainers).  X, the frontier and the per-hop blocks are sized from it.
 * A window whose frontier does not fit is detected on the device: its frontiers are truncated,
 * and it and every later window are SKIPPED by every kernel that changes buffer state (gather /
 * tally, decay, eviction swap), so the prefetcher state stays that of the last good window.  The
 * next mgnn_counts_read of such a window returns MGNN_EOVERFLOW (not sticky; mgnn_last_error
 * names the step).  Recovery: call this again with a larger bound -- it resumes the step order at
 * the overflowed window -- and sample from that step on.  rows_bound must be 0 or >= batch. */
MGNN_API mgnn_status mgnn_sampler_config_bounded(mgnn_ctx ctx, const int32_t* fanouts, int32_t n_layers,
                                                 int32_t batch, uint64_t run_seed, int32_t max_window,
                                                 int64_t rows_bound);

/* SURVEY §8(f) NEXT-1, the alternative to reading R#1 (call before mgnn_sampler_config): with
 * enable != 0 every non-local frontier node is sampled too, from its owner's CSR row, with the
 * same Philox counter -- DistDGL's sampling through the owning server.  Sampled nodes
 * outside V_p^l and V_p^h are misses: fetched from the owner's table, never buffered, never
 * scored (S_A covers V_p^h; the dense S_A of P:228 is not modelled).  Ranks become global ids
 * (window arenas sized by |V|).  Needs the global CSR: loaded (mgnn_graph_csr_load) or assembled
 * from every partition hosted by this context (ESTATE otherwise). */
MGNN_API mgnn_status mgnn_sampler_expand_remote(mgnn_ctx ctx, int32_t enable);
/* The replicated global CSR for remote expansion across GPUs (host arrays, copied; SURVEY §8(f)
 * NEXT-1's "replicated CSR"): indptr [n_global+1], cols [indptr[n_global]] global ids, rows as in
 * mgnn_partition_desc.  Without it, mgnn_sampler_expand_remote needs every partition hosted here. */
MGNN_API mgnn_status mgnn_graph_csr_load(mgnn_ctx ctx, const int64_t* indptr, const int32_t* cols);
/* NEXT-1's dense S_A ("O(|V|)"), before any mgnn_partition_load: every non-local node is
 * scorable (halo arrays over V \ V_p^l, deg_in = 0 for nodes without a local neighbour), so the
 * remote nodes remote expansion reaches are tallied and may enter the buffer by replacement.
 * |BUF| stays ceil(f * |true halo|); the initial buffer is unchanged. */
MGNN_API mgnn_status mgnn_ctx_set_dense_scores(mgnn_ctx ctx, int32_t enable);

/* NeighborSampler (Alg.2 l.1) for steps t0..t0+n_steps-1 of every hosted
 * partition into window slot `slot` (0 or 1).  Seeds are the step's slice of
 * the partition's epoch order (R#8) when seeds == NULL; otherwise seeds holds
 * [n_parts_local][n_steps][batch] ids (the first seed_counts[lp*n_steps+w] of
 * each row used), in host memory if seeds_on_host (copied inside the call,
 * use pinned memory to keep it async) else device memory.  Uses no buffer
 * state, so it may run ahead of the scoring of earlier windows. */
MGNN_API mgnn_status mgnn_sample(mgnn_ctx ctx, int32_t slot, uint64_t t0, int32_t n_steps, const int32_t* seeds,
                        const int32_t* seed_counts, int32_t seeds_on_host, mgnn_stream stream);

/* Alg.2 l.2-5, l.10-11, l.21-22 for the window in `slot`: classify every node
 * of F_L (local / hit / miss), gather its feature row into X (local table,
 * BUF row, or the owner's table over NVLink for misses), record hits, tally
 * S_A += 1 per miss, relabel the block columns to frontier positions. */
MGNN_API mgnn_status mgnn_lookup_gather(mgnn_ctx ctx, int32_t slot, mgnn_stream stream);

/* Alg.2 l.6-9 (decay of unused BUF entries, once per step of the window) and,
 * if the window's last step is a multiple of Delta, EVICT_AND_REPLACE
 * (l.12-19, l.25-34) with the swap of P:224 and the refill of the k new rows. */
MGNN_API mgnn_status mgnn_score_evict_refill(mgnn_ctx ctx, int32_t slot, mgnn_stream stream);

/* ------------------------------------------------------------------ A14: the consumer
 * GraphSAGE-mean forward pass over a prepared window (Alg.1 l.6-7: the trainer
 * consumes the minibatch "by computing the forward pass" over the sampled blocks; SAGEConv
 * 'mean' of DGL).  Layer l = 0..L-1 uses the block of hop h = L-1-l (dst = F_h, the
 * first |F_h| rows of F_{h+1}; neighbours = that hop's cols, positions in F_{h+1}):
 *     H^{l+1}[i] = act( W_self^l H^l[i] + W_neigh^l mean_{j in N_h(i)} H^l[j] + b^l ),
 * H^0 = X, act = ReLU for l < L-1 and identity for the last layer, mean over an empty
 * neighbourhood = 0.  The tensor cores multiply in TF32 with fp32 accumulation.
 * The weights are copied to the device by mgnn_sage_config (host arrays, caller keeps them). */
typedef struct {
    int32_t n_layers;               /* must equal the sampler's n_layers */
    const int32_t* dims;            /* [n_layers+1]: dims[0] = feat_dim, 1 <= dims[l] <= 256 for l >= 1 */
    const float* const* w_self;     /* [n_layers] host: [dims[l+1]][dims[l]] row-major (nn.Linear.weight) */
    const float* const* w_neigh;    /* [n_layers] host: same shapes */
    const float* const* bias;       /* [n_layers] host: [dims[l+1]] */
} mgnn_sage_desc;

/* Upload the weights and size the hidden-activation buffers for the current sampler
 * configuration (call again after mgnn_sampler_config).  EINVAL on bad shapes, ESTATE
 * before mgnn_sampler_config. */
MGNN_API mgnn_status mgnn_sage_config(mgnn_ctx ctx, const mgnn_sage_desc* desc);
/* Forward pass of every instance of the window in `slot` (after mgnn_lookup_gather of that
 * slot, ordered on `stream`).  logits: DEVICE [n_inst][batch][logits_pitch] fp32, caller-
 * owned; row i < |F_0| of instance m receives the dims[L] outputs of seed F_0[i]; other rows
 * and columns are not written.  logits_pitch >= dims[L].  One kernel launch per layer. */
MGNN_API mgnn_status mgnn_sage_forward(mgnn_ctx ctx, int32_t slot, float* logits, int64_t logits_pitch,
                                       mgnn_stream stream);

/* ------------------------------------------------------------------ NEXT-3: a DDP training step
 * (Alg.1 l.6-8: every trainer runs forward and backward on its
 * minibatch, gradients are all-reduced across trainers, the replicated model is updated).
 * One step of the DDP job = window step `step_in_window` of every partition (trainer) hosted
 * here.  Loss = mean softmax cross-entropy over each trainer's seeds F_0, averaged over the
 * n_trainers of the whole job (all ranks); gradients accumulate into the ctx's gradient buffer
 * (mgnn_sage_grads), which the caller all-reduces (sum) across ranks -- e.g. NCCL through
 * torch.distributed -- before mgnn_sage_sgd.  fp32 weights, TF32 tensor-core GEMMs, fp32
 * atomics for the gradient reductions (so gradients are reproducible only up to rounding). */
/* Labels (host int32 [n_global], 0 <= label < dims[L]) and training buffers; after
 * mgnn_sage_config.  Weights stay those of mgnn_sage_config until mgnn_sage_sgd. */
MGNN_API mgnn_status mgnn_sage_train_config(mgnn_ctx ctx, const int32_t* labels);
/* Forward + loss + backward of the instances lp * n_steps + step_in_window of the window in
 * `slot` (after mgnn_lookup_gather of that slot); gradients ADD to the gradient buffer. */
MGNN_API mgnn_status mgnn_sage_train_step(mgnn_ctx ctx, int32_t slot, int32_t step_in_window, int32_t n_trainers,
                                          mgnn_stream stream);
/* Device pointer and length (floats) of the gradient buffer (the all-reduce operand); its
 * layout mirrors the padded parameters (per layer [W_self | W_neigh] rows, then the bias). */
MGNN_API mgnn_status mgnn_sage_grads(mgnn_ctx ctx, float** grads, int64_t* n_floats);
/* W <- W - lr * g for every parameter, then g <- 0 (plain SGD, ordered on `stream`). */
MGNN_API mgnn_status mgnn_sage_sgd(mgnn_ctx ctx, float lr, mgnn_stream stream);
/* Loss accumulated since the last call (sum over steps), copied to the host and reset
 * (synchronises `stream`). */
MGNN_API mgnn_status mgnn_sage_loss(mgnn_ctx ctx, float* host_loss, mgnn_stream stream);
/* Host copies of layer l's current parameters (unpadded, nn.Linear layout; any may be NULL). */
MGNN_API mgnn_status mgnn_sage_params(mgnn_ctx ctx, int32_t l, float* w_self, float* w_neigh, float* bias);

/* Device view of a window slot (valid after mgnn_sample of that slot). */
MGNN_API mgnn_status mgnn_window_get(mgnn_ctx ctx, int32_t slot, mgnn_window* out);

/* SM partition of the prepare-ahead pipeline (Alg.1 l.5-9; the overlap of Eq.4-5,
 * P:245-251).  gather_sms > 0 splits the device's SMs into two green contexts: gather_sms SMs
 * (rounded by the driver's split granularity) run mgnn_lookup_gather and mgnn_score_evict_refill,
 * the remaining SMs run mgnn_sample and mgnn_relabel; gather_sms = 0 removes the partition (every
 * call runs on the whole GPU, the default).  Each call still takes the caller's stream: its kernels
 * start after the work queued there and the stream continues after them (an event hand-off to and
 * from an internal stream of the partition), so results and ordering are unchanged -- only where
 * the kernels run.  The consumer and training calls always use the whole GPU.  sms_out (may be
 * NULL) receives the SM counts of [gather side, prepare side] (0, 0 when off).  Synchronises the
 * device.  EINVAL: gather_sms < 0 or not below the SM count; ECUDA: green contexts unavailable. */
MGNN_API mgnn_status mgnn_sm_partition(mgnn_ctx ctx, int32_t gather_sms, int32_t* sms_out);

/* Deferred relabelling: with enable != 0, mgnn_sample stops after the last compaction and leaves
 * every hop's columns as LOCAL RANKS; mgnn_relabel(slot) then rewrites them as positions in
 * F_{i+1} (the DGL block layout of mgnn_window) on the given stream.  The gather does not read the
 * columns, so the relabel of window w can run on a third stream beside its gather (it is L2-bound,
 * the gather HBM-bound); the consumer and the training step refuse (ESTATE) a window whose relabel
 * is still pending.  mgnn_relabel: ESTATE unless the slot was sampled with the relabel deferred. */
MGNN_API mgnn_status mgnn_sampler_defer_relabel(mgnn_ctx ctx, int32_t enable);
MGNN_API mgnn_status mgnn_relabel(mgnn_ctx ctx, int32_t slot, mgnn_stream stream);

/* Caller-owned X (SURVEY §8(b) allocates X on the caller's side, e.g. a torch tensor): the arena
 * shape is n_inst_max x rows_stride rows of `pitch` floats (mgnn_window_shape, after
 * mgnn_sampler_config[_bounded]); mgnn_window_bind_x makes window slot `slot` gather into the
 * caller's DEVICE buffer X (16-byte aligned, >= n_inst_max * rows_stride * pitch floats, on this
 * context's GPU) and frees the library's arena of that slot.  The binding lasts until the next
 * sampler configuration (which allocates library arenas again); the caller keeps ownership and
 * must keep X alive while the slot is in use.  Synchronises the device.  EINVAL: too small,
 * misaligned, not device memory of this GPU; ESTATE: before the sampler configuration. */
MGNN_API mgnn_status mgnn_window_shape(mgnn_ctx ctx, int64_t* rows_stride, int64_t* pitch, int64_t* n_inst_max);
MGNN_API mgnn_status mgnn_window_bind_x(mgnn_ctx ctx, int32_t slot, float* X, int64_t capacity_floats);

/* Copy the window's counters ([n_inst][MGNN_C_N] int64) to host memory and
 * synchronise `stream`. */
MGNN_API mgnn_status mgnn_counts_read(mgnn_ctx ctx, int32_t slot, int64_t* host_counts, mgnn_stream stream);
/* Asynchronous variant: enqueues the copy of the window's counters into host_counts (pinned
 * memory) on `stream` and returns; the caller synchronises (stream or event) before reading
 * them.  Device-side seed errors are reported by the next mgnn_counts_read. */
MGNN_API mgnn_status mgnn_counts_read_async(mgnn_ctx ctx, int32_t slot, int64_t* host_counts, mgnn_stream stream);

/* Host copies of local partition lp's prefetcher state (synchronous):
 * node_ids[cap] (BUF in slot order), se[cap], sa[n_halo] and slot_of[n_halo]
 * in halo-index (ascending id) order, rows[cap][feat_dim] (may be NULL). */
MGNN_API mgnn_status mgnn_buffer_snapshot(mgnn_ctx ctx, int32_t lp, int32_t* node_ids, float* se, float* sa,
                                 int32_t* slot_of, float* rows);
/* Sizes of local partition lp: [0]=part_id [1]=n_local [2]=n_halo [3]=cap [4]=n_train. */
MGNN_API mgnn_status mgnn_part_info(mgnn_ctx ctx, int32_t lp, int64_t* info5);
/* Halo ids (sorted) and deg_in of local partition lp (synchronous). */
MGNN_API mgnn_status mgnn_halo_get(mgnn_ctx ctx, int32_t lp, int32_t* halo_ids, int32_t* deg_in);
/* Feature table row of a node hosted here (synchronous; tests). */
MGNN_API mgnn_status mgnn_table_row(mgnn_ctx ctx, int64_t node, float* out);

/* The first step of the next window mgnn_lookup_gather accepts (windows are gathered in step
 * order); after mgnn_sampler_config_bounded resumed from an arena overflow, the overflowed step. */
MGNN_API mgnn_status mgnn_next_step(mgnn_ctx ctx, uint64_t* next_step);

/* Kernel launches issued by this ctx since creation (bench evidence). */
MGNN_API int64_t mgnn_launch_count(mgnn_ctx ctx);

/* Optional CUDA-event timing of the gather kernel (the dominant HBM kernel):
 * when enabled, each mgnn_lookup_gather brackets its gather launch with events
 * on the stream it runs on; enable = 1 also brackets mgnn_sample, mgnn_relabel and
 * mgnn_score_evict_refill (mgnn_profile_stages), enable = 2 times the gather only
 * (an event between two launches ends their programmatic overlap, so the other
 * stages stay untouched); both levels count the sampled units and hits / misses; read returns the summed milliseconds, the number of
 * launches timed and the algorithmic bytes they moved (2 * rows * feat_dim * 4),
 * and resets them (synchronises the events). */
MGNN_API mgnn_status mgnn_profile_enable(mgnn_ctx ctx, int32_t enable);
MGNN_API mgnn_status mgnn_profile_read(mgnn_ctx ctx, double* ms, int64_t* launches, int64_t* bytes);

/* Per-stage CUDA-event timing of the three calls of the path (with mgnn_profile_enable on; each
 * call brackets its launches with events on the caller's stream, so under a two-stream schedule
 * the spans are the stages' durations while they overlap).  Fills out[0..MGNN_PROF_N-1] (doubles)
 * with the indices below, summed since the last read, then resets (synchronises the events):
 *   sampler kernels of mgnn_sample (k_hop, k_compact x L, k_relabel; not the seeds / epoch orders)
 *   and the sampled units the sampling roofline counts (8 E + 24 F + 8 U bytes),
 *   the gather launch and the rows it copied (2 * rows * D * 4 algorithmic bytes), and
 *   mgnn_score_evict_refill (decay + eviction round).  EINVAL if n_out < MGNN_PROF_N. */
enum {
    MGNN_PROF_SAMPLE_MS = 0, MGNN_PROF_SAMPLE_CALLS = 1,
    MGNN_PROF_EDGES = 2,      /* E: sampled edges, all hops and instances */
    MGNN_PROF_FRONTIER = 3,   /* F: expanded frontier nodes, sum over hops 0..L-1 of |F_i| */
    MGNN_PROF_UNIQUE = 4,     /* U: |F_L| summed over instances */
    MGNN_PROF_GATHER_MS = 5, MGNN_PROF_GATHER_CALLS = 6, MGNN_PROF_GATHER_ROWS = 7,
    MGNN_PROF_SCORE_MS = 8, MGNN_PROF_SCORE_CALLS = 9,
    MGNN_PROF_HITS = 10, MGNN_PROF_MISSES = 11,   /* buffer hits / misses of every gathered minibatch */
    MGNN_PROF_RELABEL_MS = 12, MGNN_PROF_RELABEL_CALLS = 13,   /* deferred k_relabel (mgnn_relabel) */
    MGNN_PROF_RELABEL_PROBES = 14,   /* k_relabel's dependent probes (hop pairs + seed hash), all columns */
    MGNN_PROF_N = 16
};
MGNN_API mgnn_status mgnn_profile_stages(mgnn_ctx ctx, double* out, int32_t n_out);

/* Process-wide per-launcher timing (diagnostics): enable = 1 clears and starts recording an
 * event after every kernel launcher (time since the previous event on the same stream is
 * attributed to it); enable = 0 stops, synchronises and writes a text table into report. */
MGNN_API mgnn_status mgnn_profile_kernels(int32_t enable, char* report, int64_t report_len);

#ifdef __cplusplus
}
#endif
#endif
