/*
 * ef200.h — C ABI of the B200 frontier-expansion-and-pricing library
 * (libef200.so, built from paper_2005_05837_b200/csrc).
 *
 * This is the drop-in boundary for the reference's search hot path
 * (arxiv/paper_2005_05837, package `enerflow`).  The reference is pure
 * Python, so it has no FFI of its own; each entry point below names the
 * reference function whose work it replaces, and INTEGRATION.md shows the
 * ctypes binding a maintainer would add to the reference.  Plain pointers
 * and sizes only; no torch types.  Every call returns EF_OK (0) or a negative
 * error code; ef_error() returns the message of the last failure.
 *
 * Device data model (all in HBM):
 *   - signature table: one ef_sig_desc + signature text + cost rows
 *     (alg, time_ms, energy) per interned signature text;
 *   - weight-set table: per node weight dict, its 16-byte BLAKE2b digest
 *     (reference graph.py:510-517) and its float64 tensors in a weight pool;
 *   - graph records: fixed-geometry slots holding one graph in CSR form
 *     (see EF_REC_* layout below), nodes ordered by reference node id;
 *   - the visited set: open-addressing table of 64-bit canonical hashes.
 */
#ifndef EF200_H
#define EF200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EF_OK 0
#define EF_ERR_ARG (-1)
#define EF_ERR_CUDA (-2)
#define EF_ERR_CAPACITY (-3)
#define EF_ERR_INTERNAL (-4) /* a device-side invariant failed (a bug: reported, never silent) */
#define EF_NEED_RESOLVE 1 /* ef_expand found signatures/weight sets not yet interned */

/* operator kinds (order of reference graph.py:25-36 OpKind) */
enum {
  EF_K_INPUT = 0, EF_K_CONV2D, EF_K_MATMUL, EF_K_RELU, EF_K_ADD, EF_K_CONCAT,
  EF_K_SPLIT, EF_K_MAXPOOL, EF_K_AVGPOOL, EF_K_BATCHNORM, EF_K_IDENTITY
};

/* rewrite rules (order of reference rules.py:338-353 default_rules) */
enum {
  EF_R_FUSE_CONV_RELU = 0, EF_R_SPLIT_CONV_ACT = 1, EF_R_MERGE_CONVS = 2,
  EF_R_SPLIT_MERGED = 3, EF_R_FOLD_IDENTITY = 4, EF_R_FUSE_CONV_BN = 5
};

/* cost-function kinds (reference cost.py:172) */
enum { EF_C_TIME = 0, EF_C_ENERGY, EF_C_POWER, EF_C_LINEAR, EF_C_PRODUCT, EF_C_MIX };

/* weight-set derivations created by rewrites */
enum {
  EF_D_MERGE = 1,    /* rules.py:231-232 concat(left, right), bias default zeros */
  EF_D_SLICE_LO = 2, /* rules.py:272-273 weight[:s0], bias[:s0]                 */
  EF_D_SLICE_HI = 3, /* rules.py:275-276 weight[s0:], bias[s0:]                 */
  EF_D_FOLD = 4      /* rules.py:326-327 w*scale, bias*scale+shift              */
};

/* Structural signature of a node.  For conv2d / relu / 2-way split it is an
 * exact key (the device builds these for rewritten nodes and looks them up);
 * for other kinds only kind/rank/in/out are filled. */
typedef struct {
  int32_t kind, rank;
  int32_t in[4];  /* input-0 dims, zero padded */
  int32_t out[4]; /* output-0 dims, zero padded */
  int32_t oc, kh, kw, sh, sw, ph, pw, act;
  int32_t axis, nsizes, s0, s1;
} ef_sig_desc;

/* Record geometry: every graph slot of a context has the same capacity. */
typedef struct {
  uint32_t cap_nodes, cap_refs, cap_outs;
  uint32_t record_bytes;                        /* total slot size            */
  uint32_t off_nid, off_sig, off_aux, off_nin;  /* byte offsets of the arrays  */
  uint32_t off_inoff, off_topo, off_refs, off_outs, off_keys, off_alg, off_sperm, off_skeys, off_srank;
} ef_geometry;

/* Record header (first 64 bytes of a slot). */
typedef struct {
  int32_t n, n_refs, n_out, n_compute;
  int32_t pad[12];
} ef_rec_header;
/* Arrays after the header (indexed by node position, positions sorted by id):
 *   int32  nid[cap_nodes]      reference node id
 *   uint32 sig[cap_nodes]      signature id
 *   uint32 aux[cap_nodes]      weight-set id (input nodes: input-name id)
 *   uint32 nin[cap_nodes]      number of input refs
 *   uint32 inoff[cap_nodes+1]  CSR offsets into refs
 *   uint32 topo[cap_nodes]     a topological order of positions
 *   uint32 refs[cap_refs]      (producer position << 8) | port
 *   uint32 outs[cap_outs]      graph outputs, same packing
 *   uint8  keys[cap_nodes][16] Merkle node keys (graph.py:528-540)
 *   uint8  alg[cap_nodes]      algorithm per node after pricing
 *   uint32 sperm[cap_nodes]    positions in ascending key order (sorted(keys) of graph.py:547)
 *   uint8  skeys[cap_nodes][16] the node keys in that order (streamed by the step's graph digest)
 *   uint32 srank[cap_nodes]    rank of each position in that order (inverse of sperm)
 */

/* Pricing parameters: cost function (cost.py:234-254) + inner search (search.py:106-153). */
typedef struct {
  int32_t kind;       /* EF_C_* */
  int32_t d;          /* inner neighbourhood radius (>= 1) */
  int32_t use_inner;  /* 0: default assignment only (search.py:196-202) */
  int32_t node_cap;   /* compute-node cap (search.py:205-208) */
  double w, ct, ce, cp, t_ref, e_ref, p_ref;
  /* alpha-prune of the step (search.py:258-267): over the priced candidates in (parent, rule,
   * site) order, prev = min(best, costs of the priced candidates before it); EF_F_BEST marks
   * cost < prev, EF_F_ENQUEUE cost < alpha * prev.  alpha = 0: no prune flags. */
  double best, alpha;
  /* start totals: 0 = CPython >= 3.12 sum() (Neumaier-compensated), 1 = plain left-to-right sum
   * (CPython <= 3.11), so the sweep starts from the totals the caller's interpreter computes */
  int32_t naive_sum;
  /* 0: price the first occurrence of each hash in the step (the reference's order when the
   * parents are expanded in step order); 1: the first occurrence within each parent (EF_F_PFIRST),
   * so every parent's own rewrite of a graph is priced with its own node ids even when the caller
   * consumes the parents out of step order (the batched, speculative outer search) */
  int32_t per_parent;
} ef_price_params;

/* Per-candidate result of one expansion step, in (parent, rule, site) order. */
enum {
  EF_F_FIRST = 1,     /* first occurrence of this hash within the step  (rules.py:79-88) */
  EF_F_VISITED = 2,   /* hash was in the visited set before the step    (search.py:248)  */
  EF_F_CAPPED = 4,    /* compute-node count above the cap               (search.py:252)  */
  EF_F_PRICED = 8,    /* inner search ran                                                */
  EF_F_MISSING = 16,  /* some node has no cost rows (MissingEntry)                        */
  EF_F_INCOMPLETE = 32,
  EF_F_BEST = 64,     /* priced, cost < the best before it              (search.py:259-261)  */
  EF_F_ENQUEUE = 128, /* priced, cost < alpha * the best before it     (search.py:262-267)  */
  EF_F_PFIRST = 256   /* first occurrence of this hash within its parent (per_parent pricing) */
};
typedef struct {
  uint64_t hash;
  double cost, time_ms, energy;
  int64_t evals;
  int32_t sweeps, n_compute;
  uint32_t flags, parent;
  uint32_t rule, site_a, site_b; /* positions in the parent */
  uint32_t touched_sig[2];       /* signatures of rewritten nodes (UINT32_MAX: none) */
  uint32_t n_nodes;              /* nodes of the candidate graph */
} ef_cand_result;

typedef struct ef_ctx ef_ctx;

/* ---- context ---------------------------------------------------------- */
ef_ctx* ef_create(int device);
void ef_destroy(ef_ctx* ctx);
const char* ef_error(ef_ctx* ctx);
int ef_device_count(void);

/* ---- tables ----------------------------------------------------------- */
/* signature text + structure; replaces graph.py:441-448/480-498 on the path */
int ef_sig_put(ef_ctx* ctx, uint32_t id, const ef_sig_desc* desc, const char* text, uint32_t text_len, int exact);
/* cost rows of one signature, ascending alg; replaces cost.py:120-134 node_cost_table rows */
int ef_sig_costs(ef_ctx* ctx, uint32_t id, uint32_t n, const int32_t* alg, const double* time_ms, const double* energy);
/* input-node names (hashed into input-node keys, graph.py:534-535) */
int ef_name_put(ef_ctx* ctx, uint32_t id, const char* name, uint32_t len);
/* an original weight set.  kind is EF_K_CONV2D (w = weight, b = optional
 * bias), EF_K_BATCHNORM (w = scale, b = shift), EF_K_MATMUL (w = weight) or
 * anything else (no tensors).  hdr_w / hdr_b are the digest headers
 * key + str(shape) (graph.py:514-515); the device digests the set in sorted
 * key order ("bias" < "weight", "scale" < "shift") in ef_tables_commit. */
int ef_wset_put(ef_ctx* ctx, uint32_t id, int32_t kind, int32_t oc,
                const double* w, uint64_t w_n, const double* b, uint64_t b_n,
                const char* hdr_w, uint32_t hlen_w, const char* hdr_b, uint32_t hlen_b);
/* a derived weight set (EF_D_*) computed on the device from set a (and b:
 * the right conv for MERGE, the batchnorm for FOLD); s0 = split point for
 * SLICE_*.  The result is a conv set with weight and bias. */
int ef_wset_derive(ef_ctx* ctx, uint32_t id, int32_t op, uint32_t a, uint32_t b, int32_t s0,
                   const char* hdr_w, uint32_t hlen_w, const char* hdr_b, uint32_t hlen_b);
/* copy a weight set's tensors back; returns counts through w_n / b_n when the pointers are NULL */
int ef_wset_read(ef_ctx* ctx, uint32_t id, double* w, uint64_t* w_n, double* b, uint64_t* b_n);
int ef_wset_digest(ef_ctx* ctx, uint32_t id, uint8_t out[16]);
/* upload lookup tables, compute pending digests; call after puts/derives */
int ef_tables_commit(ef_ctx* ctx);
/* host->device bytes the last ef_tables_commit sent: a commit sends only the signatures, rows,
 * names and weight sets added (or changed) since the previous one and the lookup-table slots
 * they occupy, so its cost does not grow with the tables (profiling.py:211-252: the reference
 * memoises once per new signature) */
int ef_commit_bytes(ef_ctx* ctx, uint64_t* bytes);

/* ---- graph records ------------------------------------------------------ */
int ef_set_geometry(ef_ctx* ctx, uint32_t cap_nodes, uint32_t cap_refs, uint32_t cap_outs,
                    const char* input_text, uint32_t input_text_len, ef_geometry* out);
int ef_record_alloc(ef_ctx* ctx, uint32_t* slot);
int ef_record_free(ef_ctx* ctx, uint32_t slot);
/* n slots at once (the search materialises and releases candidates in batches) */
int ef_records_alloc(ef_ctx* ctx, uint32_t n, uint32_t* slots);
int ef_records_free(ef_ctx* ctx, const uint32_t* slots, uint32_t n);
int ef_record_write(ef_ctx* ctx, uint32_t slot, const void* host, uint64_t bytes);
int ef_record_read(ef_ctx* ctx, uint32_t slot, void* host, uint64_t bytes);
/* batched upload: record i comes from host + i * stride (one stream sync for all) */
int ef_records_write(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host, uint64_t stride,
                     uint64_t bytes);
/* page-locked host staging memory for ef_records_write / ef_results */
void* ef_host_alloc(uint64_t bytes);
void ef_host_free(void* p);
/* canonical hash of records (graph.py:520-549): recomputes all keys */
int ef_hash_records(ef_ctx* ctx, const uint32_t* slots, uint32_t n, uint64_t* hashes);
/* inner search on records (search.py:106-153); writes alg[] into the records */
int ef_price_records(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const ef_price_params* pp,
                     ef_cand_result* out);

/* ---- visited set ---------------------------------------------------------- */
/* The reference's `visited` Python set (search.py:241-251).  An open-addressing table of 64-bit
 * hashes that the library keeps at most half full: every insertion path (ef_visited_insert,
 * ef_expand with insert_visited, ef_owner_mark) first grows it by rehashing on the device, so
 * `capacity` is only the initial size.  Probe loops are bounded; a full table is reported as an
 * error, never a hang. */
int ef_visited_reset(ef_ctx* ctx, uint64_t capacity);
int ef_visited_insert(ef_ctx* ctx, const uint64_t* hashes, uint32_t n);
int ef_visited_count(ef_ctx* ctx, uint64_t* count);
int ef_visited_capacity(ef_ctx* ctx, uint64_t* capacity);

/* ---- the hot path ---------------------------------------------------------- */
/* One frontier step: match every rule at every site of every parent
 * (rules.py:61-71), materialise each rewrite (rules.py:96-331), hash it
 * (graph.py:520-549), dedup within the step and against the visited set
 * (rules.py:79-88, search.py:247-251), price survivors (search.py:189-202).
 * Returns EF_OK with the number of candidates in *n_candidates,
 * EF_NEED_RESOLVE when new signatures / weight sets must be interned first
 * (see ef_pending; nothing was inserted into the visited set), or < 0. */
int ef_expand(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents,
              const int32_t* rules, uint32_t n_rules, const ef_price_params* pp, int insert_visited,
              uint32_t* n_candidates);
/* requests behind EF_NEED_RESOLVE: new signature descriptors and weight derivations
 * (op, a, b, s0) quadruples */
int ef_pending(ef_ctx* ctx, ef_sig_desc* sigs, uint32_t sig_cap, uint32_t* n_sigs,
               int32_t* derives, uint32_t derive_cap, uint32_t* n_derives);
int ef_results(ef_ctx* ctx, ef_cand_result* out, uint32_t n);
/* the same copy, asynchronous: the last step's results are snapshotted on the device (so the
 * next step may start at once) and copied to `out` (page-locked host memory) on a copy
 * stream, overlapping whatever the caller queues next; ef_results_wait blocks until `out`
 * holds them.  One copy in flight at a time. */
int ef_results_async(ef_ctx* ctx, ef_cand_result* out, uint32_t n);
int ef_results_wait(ef_ctx* ctx);
/* copy step candidates into record slots (the ones the search keeps) */
int ef_keep(ef_ctx* ctx, const uint32_t* cand_idx, uint32_t n, const uint32_t* slots);
/* Materialise rewrites of parent records without a step: candidate i is the cand_local[i]-th
 * rewrite, in (rule, site) order (rules.py:61-71), of parent_slots[cand_parent[i]] under the
 * given rules, written into slots[i] with its node keys and sorted order.  The search keeps
 * enqueued graphs as (parent, rewrite index) and materialises them only when it expands them
 * (search.py:239-243 keeps candidates in `pending`).  Replaces the last step's state (ef_keep
 * is invalid afterwards); alg[] of the new records is not set (ef_price_records sets it). */
int ef_materialise(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                   uint32_t n_rules, const uint32_t* cand_parent, const uint32_t* cand_local, uint32_t n,
                   const uint32_t* slots);
/* ---- hash-owner sharding (one process per GPU) ------------------------------------------ */
/* The frontier is split across ranks by parent; deduplication is owned by hash:
 * rank h % world decides, for every candidate hash, its first occurrence in the
 * global (rank-major) candidate order and its membership in that rank's shard of
 * the visited set (search.py:245-251 across ranks).  A sharded step is
 *   ef_expand_hashes -> ef_route_owners -> all-to-all (caller, NCCL) ->
 *   ef_owner_mark -> all-to-all back -> ef_expand_finish.
 * Pointers named d_* are device pointers on the context's GPU. */
/* match, plan and hash the candidates of the given parents (no dedup, no pricing) */
int ef_expand_hashes(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                     uint32_t n_rules, uint32_t* n_candidates);
/* the same, pricing every complete candidate speculatively beside the hashing (large graphs,
 * the policy of ef_expand); ef_expand_finish / ef_expand_finish_padded then take the prices of
 * the survivors instead of pricing them */
int ef_expand_hashes_spec(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                          uint32_t n_rules, const ef_price_params* pp, uint32_t* n_candidates);
/* (hash, order_base + candidate index) pairs grouped by owner rank into d_send
 * (room for 2 * n_candidates uint64); counts[world] = pairs per owner (host) */
int ef_route_owners(ef_ctx* ctx, uint32_t world, uint64_t order_base, uint64_t* d_send, uint32_t* counts);
/* owner side: verdict (EF_F_FIRST | EF_F_VISITED) for each received pair;
 * inserts first occurrences into this rank's visited shard when insert_visited */
int ef_owner_mark(ef_ctx* ctx, const uint64_t* d_recv, uint32_t n_recv, uint32_t* d_verdict, int insert_visited);
/* verdicts back in send order -> candidate flags, node cap, pricing of the survivors */
int ef_expand_finish(ef_ctx* ctx, const uint32_t* d_verdict_back, const ef_price_params* pp);
/* The same exchange with fixed-capacity buckets, so no count ever travels through the host:
 * d_send is [world][cap] pairs (cap >= this rank's candidates: the caller all-reduces MAX of
 * the candidate counts), d_counts[world] the pairs per owner (device).  The collectives run on
 * the context's stream (ef_stream), so the whole sharded step is stream-ordered. */
int ef_route_owners_padded(ef_ctx* ctx, uint32_t world, uint64_t order_base, uint32_t cap, uint64_t* d_send,
                           uint32_t* d_counts);
/* owner side over [world][cap] received pairs, d_recv_counts[world] valid per source rank;
 * d_verdict is [world][cap] */
int ef_owner_mark_padded(ef_ctx* ctx, const uint64_t* d_recv, const uint32_t* d_recv_counts, uint32_t world,
                         uint32_t cap, uint32_t* d_verdict, int insert_visited);
/* verdicts back ([world][cap], this rank's send layout) -> flags, node cap, pricing */
int ef_expand_finish_padded(ef_ctx* ctx, const uint32_t* d_verdict_back, uint32_t world, uint32_t cap,
                            const ef_price_params* pp);
/* the CUDA stream (cudaStream_t) the context issues its work on */
int ef_stream(ef_ctx* ctx, void** stream);
/* recompute the last step's alpha-prune flags (EF_F_BEST / EF_F_ENQUEUE) from a new best cost
 * before its first candidate: a rank of a sharded step passes the minimum over the best and
 * the candidates of the ranks before it (search.py:258-267 across ranks) */
int ef_reprune(ef_ctx* ctx, double best, double alpha);

/* device time (ms) of the last ef_expand, measured with CUDA events on its stream, per
 * stage: match, plan, dirty walk, node keys, key sort, graph digest, dedup, price, and [8] the
 * whole step from match to price (for a sharded step: including the exchange) (n <= 9) */
int ef_last_timing(ef_ctx* ctx, float* ms, uint32_t n);
/* counters of the last step: BLAKE2b compressions in node keys, in graph digests,
 * candidates, priced survivors, kernels the library launched for it (n <= 5) */
int ef_last_stats(ef_ctx* ctx, uint64_t* out, uint32_t n);
/* batched upload of compact records (host): record i at host + offsets[i] is
 * [n, n_refs, n_out, n_compute] nid[n] sig[n] aux[n] nin[n] inoff[n+1] topo[n] refs outs
 * (uint32); the device unpacks it into slots[i] and computes keys / sorted order / ranks */
int ef_records_write_packed(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host, const uint64_t* offsets,
                            uint64_t bytes);
/* the same on the context's upload stream, returning at once, so the copy, unpacking and
 * hashing overlap a step (pipelining frontier batches).  It starts after the main-stream work
 * queued before it; a step reads the uploaded records only after ef_upload_fence.  `host`
 * must be page-locked (ef_host_alloc) and stay unchanged until the upload is fenced. */
int ef_records_write_packed_async(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host,
                                  const uint64_t* offsets, uint64_t bytes);
/* main-stream work queued after this call waits for every asynchronous upload issued before it */
int ef_upload_fence(ef_ctx* ctx);
/* measured BLAKE2b compression rate of this GPU (register-only loop): the ALU roofline */
int ef_b2b_peak(ef_ctx* ctx, double* compress_per_s);
/* self-check of the pricing's division by a normalisation reference (cost.py:284-296 t / t_ref,
 * e / e_ref, p / p_ref; reciprocal + two FMA corrections) against the IEEE division: per_divisor
 * random dividends for each divisor; *mismatches = results differing in any bit (must be 0) */
int ef_check_division(ef_ctx* ctx, const double* divisors, uint32_t n_divisors, uint64_t per_divisor, uint64_t seed,
                      uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* EF200_H */
