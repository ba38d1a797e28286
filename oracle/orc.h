/* orc.h -- CPU ORACLE for the halo feature pipeline of arXiv 2410.22697
 * (continuous prefetch + eviction, §3.1 Alg.1/Alg.2, §3.2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * library under paper_2410_22697_b200/csrc (and neither includes the other).
 *
 * Plain, slow, obviously-correct C: fp32 scores (reading R12:
 * IEEE binary32, round-to-nearest-even, denormals kept, no contraction),
 * qsort for every ordering, binary search for halo lookups (the paper's
 * "memory-efficient S_A").  Line refs "P:n" are PAPER.md lines,
 * "R#n" are the readings listed in DESIGN.md §Readings (= SURVEY §8(c)).
 */
#ifndef MGNN_ORACLE_ORC_H
#define MGNN_ORACLE_ORC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_world orc_world;   /* all P partitions' KVStores */
typedef struct orc_part  orc_part;    /* one trainer's partition + prefetcher state */

/* Philox4x32-10 (Salmon et al., SC'11 "Random123"), used for every random
 * draw (R#4): out = philox(ctr[4], key[2]). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Synthetic feature row of global node `node` (R#4 feature stream). */
void orc_feature_row(int64_t node, int32_t dim, uint64_t feat_seed, float* out);

/* Floyd's k-of-d resolution (R#6) on pre-drawn r[j] in [0, d-k+j]. */
void orc_floyd(int64_t d, int32_t k, const uint32_t* r, int64_t* pos_out);

/* Uniform draw r_j = floor(u*(t+1)/2^32) (R#5). */
uint32_t orc_range(uint32_t u, uint32_t t_plus_1);

/* alpha = gamma^Delta as the iterated fp32 product (Eq.1; R#13). */
float orc_alpha_default(float gamma, int32_t delta);

orc_world* orc_world_new(int32_t n_parts, int64_t n_global, const int64_t* bounds,
                         int32_t feat_dim, uint64_t feat_seed);
void orc_world_free(orc_world* w);

/* Build partition p: copies the host arrays, builds V_p^h,
 * deg_in, and materialises the local feature table ("KVStore").  Returns
 * NULL on invalid input. */
orc_part* orc_part_new(orc_world* w, int32_t part_id, const int64_t* indptr, const int32_t* cols,
                       const int32_t* train_ids, int64_t n_train);
void orc_part_free(orc_part* p);

int64_t orc_n_local(const orc_part* p);
int64_t orc_n_halo(const orc_part* p);
void    orc_halo(const orc_part* p, int32_t* halo_ids, int32_t* deg_in);   /* either may be NULL */

/* INITIALIZE_PREFETCHER (Alg.1).  f_bp = f_p^h in basis points.
 * Returns 0 or -1 (invalid params). */
int orc_buffer_init(orc_part* p, float gamma, float alpha, float theta_r, int32_t delta, uint32_t f_bp);
int64_t orc_capacity(const orc_part* p);

/* Epoch permutation of the partition's training ids (R#8). out[n_train]. */
void orc_epoch_perm(const orc_part* p, uint64_t run_seed, uint64_t epoch, int32_t* out);

/* PREFETCH_WITH_EVICTION for global 1-based step `step` (Alg.2).
 * fanouts: GNN-layer order, input layer first (R#2).  If seeds != NULL the
 * given n_seeds seed ids are used instead of the epoch order.  Returns 0,
 * or -1 on invalid input / missing init. */
int orc_step(orc_part* p, uint64_t run_seed, uint64_t step, const int32_t* fanouts, int32_t n_layers,
             int32_t batch, const int32_t* seeds, int32_t n_seeds);

/* EVICT_AND_REPLACE on explicit state arrays (Alg.2 l.25-34 + the swap of
 * P:224); orc_step calls exactly this.  Arrays are modified in place;
 * returns k.  The pair lists (node ids, slots) are written when non-NULL. */
int64_t orc_evict_and_replace(int64_t cap, int64_t n_h, int32_t* node_of_slot, float* se, float* sa,
                              int32_t* slot_of, const int32_t* halo, const int32_t* deg_in, float alpha,
                              float theta_r, int32_t* evicted_out, int32_t* replaced_out, int32_t* slots_out);

/* SURVEY §8(f) NEXT-1 (the alternative to reading R#1): with on != 0, every non-local frontier
 * node is sampled too, from its owner's CSR row, with the same Philox counter (sampling trainer
 * p, node, hop, slot, step) -- DistDGL's sampling through the owning server.  Sampled
 * nodes outside V_p^l and V_p^h are misses (class 3): fetched from the owner, never buffered and
 * never scored (S_A covers V_p^h only; the dense S_A of P:228 is not modelled). */
void orc_set_expand_remote(orc_part* p, int32_t on);
/* NEXT-1's dense S_A ("a compact S_A over V_p^h ... or O(|V|)"): with on != 0 (before any
 * orc_part_new) every non-local node is scorable -- in the halo arrays with deg_in = 0 when it has
 * no local neighbour -- so remote nodes reached by remote expansion are tallied and can enter
 * the buffer by replacement.  |BUF| stays ceil(f * |true halo|), and the initial buffer is the
 * same (true halo nodes rank first by deg_in). */
void orc_world_set_dense(orc_world* w, int32_t on);

/* Results of the last orc_step (valid until the next one). */
enum { ORC_C_NODES = 0, ORC_C_LOCAL, ORC_C_HIT, ORC_C_MISS, ORC_C_EVICTED, ORC_C_REFILLED,
       ORC_C_ROWS_FETCHED, ORC_C_N };
void    orc_counts(const orc_part* p, int64_t* out /* ORC_C_N */);
int64_t orc_hop_size(const orc_part* p, int32_t hop);      /* |F_hop|, hop = 0..L */
int64_t orc_hop_edges(const orc_part* p, int32_t hop);     /* |cols_hop|, hop = 0..L-1 */
void    orc_frontier(const orc_part* p, int32_t* out);     /* F_L, |F_L| global ids */
void    orc_hop_block(const orc_part* p, int32_t hop, int64_t* offsets /* |F_hop|+1 */,
                      int32_t* cols /* global ids */);
void    orc_features_out(const orc_part* p, float* out /* |F_L| x D */);
void    orc_classes(const orc_part* p, int8_t* out /* |F_L|: 0 local, 1 hit, 2 miss */);

/* Prefetcher state (host copies). node_of_slot/se: [cap]; sa/slot_of: [n_halo]
 * in halo-index order; rows [cap x D] may be NULL. */
void orc_buffer_state(const orc_part* p, int32_t* node_of_slot, float* se, float* sa,
                      int32_t* slot_of, float* rows);
/* Cumulative counters since init: [0]=sum hits, [1]=sum misses, [2]=sum refills, [3]=init fetches */
void orc_totals(const orc_part* p, int64_t* out4);

#ifdef __cplusplus
}
#endif
#endif
