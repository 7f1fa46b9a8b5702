// C ABI of libef200.so (declared in include/ef200.h): context, tables, records and the
// frontier step.  All device work is issued on the context's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <thread>
#include <cstring>
#include <string>
#include <vector>

#include "ef_step.cuh"

using namespace ef;

namespace {

constexpr int kMatchThreads = 256;
constexpr int kMatThreads = 256;
constexpr int kHashThreads = 128;
constexpr int kPriceThreads = EF_PRICE_THREADS;
constexpr uint32_t kFastRows = 256;  // rows (max parent nodes + 2) served by the fast step kernels
constexpr uint32_t kPrefixMinOuts = 64;  // graph outputs from which k_prefix builds the digest's prefix

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  // grow (optionally preserving contents); returns cudaError
  cudaError_t reserve(size_t n, cudaStream_t st, bool keep = false) {
    if (n <= cap) return cudaSuccess;
    size_t nc = std::max(n, cap * 2 + 16);
    T* q = nullptr;
    cudaError_t e = cudaMalloc(&q, nc * sizeof(T));
    if (e != cudaSuccess) return e;
    if (keep && p && cap) {
      e = cudaMemcpyAsync(q, p, cap * sizeof(T), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return e;
      cudaStreamSynchronize(st);
    }
    if (p) cudaFree(p);
    p = q;
    cap = nc;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct WeightSet {
  int32_t kind = 0, oc = 0;
  uint64_t w_off = 0, w_n = 0, b_off = 0, b_n = 0;
  bool has_b = false;
  int32_t dv[4] = {0, 0, 0, 0};
  std::string hdr_w, hdr_b;
  bool ready = false;  // tensors present + digest computed
  std::vector<uint64_t> hw, hb;  // host copies (raw float64 bits) until the digest is taken
};

// one lookup-table slot written by an incremental commit (k_ht_scatter)
struct HtUpd {
  uint32_t slot, val;
  unsigned long long key;
};

__global__ void k_ht_scatter(unsigned long long* keys, uint32_t* vals, const HtUpd* u, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    keys[u[i].slot] = u[i].key;
    vals[u[i].slot] = u[i].val;
  }
}

// per-chunk hashing scratch (ef_step.cuh): one set for steps / keeps on the main stream, one
// for asynchronous uploads on the upload stream
struct Scratch {
  DevBuf<uint32_t> didx, jv, refsrc, dcount, dorder, sval2, rmask, outsrc, cbins;
  DevBuf<Job> jobs;
  DevBuf<uint16_t> jlvl;
  DevBuf<uint64_t> fresh, fresh2, skey, skey2, merged, pfx;
  DevBuf<int32_t> seg_b, seg_e;
  DevBuf<uint32_t> recmax, pdir, pfx_first;
  DevBuf<uint64_t> pfx_state;
  void release() {
    pdir.release();
    pfx_first.release();
    pfx_state.release();
    jlvl.release();
    merged.release();
    didx.release(); jv.release(); refsrc.release(); dcount.release(); dorder.release(); cbins.release();
    sval2.release(); rmask.release(); outsrc.release(); jobs.release(); pfx.release();
    fresh.release(); fresh2.release(); skey.release(); skey2.release(); seg_b.release(); seg_e.release();
    recmax.release();
  }
};

}  // namespace

struct ef_ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  std::string err;
  int n_sm = 148;
  bool big_merge = true;  // rows > 256: merge-path key stream + streaming digest (EF_BIG_MERGE=0: in-thread merge)
  uint32_t wide_min = 512;  // jobs per candidate from which k_keys_wide takes it (EF_WIDE_MIN; 0: off)
  bool dirty_big = true;  // rows > kFastRows: k_dirty_big (warp window walk); EF_DIRTY_BIG=0: k_dirty
  uint32_t wide_lpc = 8;  // lanes per candidate in k_keys_wide: 32, 16, 8 or 4 (EF_WIDE_LPC; DAG-20k keys 70.8 -> 63.9 ms from 16 to 8, 85.3 at 4)
  bool fuse_merge = false;  // rows > kFastRows: k_digest_mg merges on the fly (EF_FUSE_MERGE=1; measured slower: 52.9 vs 12.0 + 38.5 ms on DAG-20k)
  bool merge_scatter = true;  // rows > kFastRows: k_merge_scatter (EF_MERGE_SCATTER=0: k_merge_big)
  // ... on rows above EF_MS_MIN_ROWS (k_merge_big below), sorting the fresh keys itself on rows
  // above EF_MS_SORT_MIN (k_sortkeys below).  Both 0: every row > kFastRows.  Measured per step
  // against k_sortkeys + k_merge_big: Inception-v3 8.61 -> 8.17 ms, NasNet-A 9.39 -> 6.73 ms,
  // DAG-1k 11.8 -> 10.0 ms (k_sortkeys + k_merge_scatter: 9.37 / 9.44 / 11.8)
  uint32_t ms_min_rows = 0;
  uint32_t ms_sort_min_rows = 0;
  bool sparse_sweep = true;  // rows > kFastRows: d = 1 sweeps visit only movable nodes (EF_SPARSE_SWEEP=0: all)
  DevBuf<uint32_t> d_nsk;
  bool pfx_share = true;  // k_prefix / the digest start at the parent's prefix state (EF_PFX_SHARE=0: from block 0)
  bool digest_pf = true;  // rows > kFastRows: k_digest_pm loads the next block's key words ahead (EF_DIGEST_PF)
  uint32_t quad_max = 20000;  // chunks below this many candidates hash with k_keys_quad (EF_QUAD_MAX)
  uint64_t chunk_mib = 0;  // per-chunk hashing scratch budget, MiB (0: 80% of the HBM free at the first sizing, <= 144 GiB)

  // host mirrors of the tables
  std::vector<ef_sig_desc> sig_desc;
  std::vector<uint8_t> sig_exact;
  std::vector<std::string> sig_text;
  std::vector<std::vector<int32_t>> row_alg;
  std::vector<std::vector<double>> row_t, row_e;
  std::vector<std::string> names;
  std::vector<WeightSet> ws;
  bool dirty = true;

  // device tables
  DevBuf<ef_sig_desc> d_sig_desc;
  DevBuf<uint32_t> d_text_off, d_text_len, d_row_off, d_row_n, d_sig_ht_val, d_dv_ht_val, d_name_off, d_name_len;
  DevBuf<uint8_t> d_text, d_names, d_input_text;
  DevBuf<int32_t> d_row_alg, d_dv_tuple;
  DevBuf<double> d_row_t, d_row_e;
  DevBuf<unsigned long long> d_sig_ht_key, d_dv_ht_key;
  DevBuf<uint64_t> d_ws_digest;
  std::vector<uint64_t> h_ws_digest;  // host mirror (the digests are taken on host cores)
  DevBuf<double> d_pool;
  uint64_t pool_used = 0;
  uint32_t sig_ht_mask = 0, dv_ht_mask = 0;
  std::string input_text;
  // incremental commit (ef_tables_commit uploads what changed since the last commit): the
  // device tables mirror ids < c_ns / c_nw / c_names; older ids changed since are listed
  bool c_valid = false;
  size_t c_ns = 0, c_nw = 0, c_names = 0;
  std::vector<uint32_t> sig_touched;  // ids < c_ns whose text or cost rows changed
  bool sig_key_changed = false;       // an old id's desc / exactness changed: rebuild its lookup
  bool names_changed = false, input_changed = true, dv_changed = false;
  std::vector<uint32_t> h_toff, h_tlen, h_roff, h_rn, h_info;  // per-id arrays as on the device
  uint64_t text_used = 0, rows_used = 0, name_used = 0;
  std::vector<unsigned long long> h_sig_ht_key, h_dv_ht_key;  // lookup tables as on the device
  std::vector<uint32_t> h_sig_ht_val, h_dv_ht_val;
  uint32_t sig_ht_n = 0;
  DevBuf<HtUpd> d_upd_sig, d_upd_dv;
  uint64_t commit_bytes = 0;  // host->device bytes of the last commit (tests: independent of table size)

  // records
  Geo geo{};
  bool have_geo = false;
  std::vector<char*> chunks;
  uint32_t slots_per_chunk = 0;
  std::vector<uint32_t> free_slots;
  uint32_t n_slots = 0;

  // step buffers
  DevBuf<unsigned long long> d_parent_addr, d_sites, d_step_key, d_addr_a, d_addr_b;
  DevBuf<uint32_t> d_pscratch, d_site_count, d_cand_off, d_step_seq, d_scalars;
  DevBuf<char> d_stage;
  DevBuf<int32_t> d_req_dv;
  DevBuf<ef_cand_result> d_res, d_res_aux, d_res_snap;
  cudaStream_t st_copy = nullptr;  // results copies (ef_results_async)
  cudaEvent_t ev_snap = nullptr, ev_copy = nullptr;
  DevBuf<ef_sig_desc> d_req_sig;
  DevBuf<uint64_t> d_hash_out;
  DevBuf<uint32_t> d_sperm;
  uint32_t cand_cap = 0, site_cap = 0;
  uint32_t req_cap = 4096;
  uint32_t last_total = 0;
  uint32_t last_req_sig = 0, last_req_dv = 0;
  uint32_t* h_scalars = nullptr;  // pinned: total, err, n_req_sig, n_req_dv, vis_count lo/hi

  // virtual-candidate step (ef_step.cuh)
  DevBuf<VPlan> d_plan;
  DevBuf<uint32_t> d_route, d_perm;
  DevBuf<unsigned long long> d_stats;
  DevBuf<unsigned long long> d_step_ord;
  uint32_t n_send = 0;
  DevBuf<uint32_t> d_plist, d_sig_info;
  DevBuf<uint8_t> d_alg8, d_algt;
  Scratch sc[2];
  cudaStream_t st_up = nullptr;  // asynchronous uploads
  cudaStream_t st_wide = nullptr;  // k_keys_wide beside k_keys
  // speculative pricing (rows > kFastRows): every complete candidate priced on st_price while
  // the chunks hash, the survivors' prices committed after the dedup (EF_SPEC_PRICE: 0 off,
  // 1 from the first digest on, 2 from the plans on; the side stream has the lowest priority, so
  // its CTAs fill what the hashing kernels leave free.  Measured per step: DAG-20k 211.9 -> 206.7
  // ms from the plans, 219.7 from the digest; DAG-5k 41.4 -> 39.3 from the plans; DAG-1k 14.9 ->
  // 13.8 and NasNet-A 10.9 -> 10.5 from the digest (15.9 / 13.1 from the plans); Inception-v3
  // (187k candidates) 9.11 -> 9.55 from the digest: enough short candidates keep every SM busy,
  // and pricing there only competes)
  // lanes per candidate of the d=1 sweep after the dedup (k_price_lanes; EF_PRICE_LANES, 0 / 1 =
  // k_price_v), rows up to 2048.  Measured: Inception-v3 price 2.00 -> 1.79 ms with 2 lanes,
  // 2.60 with 4, 4.47 with 8; ResNet-50 0.384 -> 0.372 / 0.514 / 0.902 ms: the first sweep
  // takes at most nodes, so its windows commit one node each and the converged sweeps' L-fold
  // parallelism only pays at 2 lanes.  DAG-20k (global rows): 28.8 -> 53.5 ms at 2 lanes.
  // Since the sparse sweeps (k_price_nsk), one thread per candidate visiting only the movable
  // nodes wins everywhere, so lanes are off by default: ResNet-50 0.367 -> 0.328 ms, Inception-v3
  // 1.80 -> 1.39 ms (dense k_price_v: 0.370 / 2.33).  Small steps (the batched outer_search's,
  // a few thousand candidates) are latency-bound and keep 2 lanes: ResNet-50 3000-expansion
  // search 0.85 s warm with 2 lanes, 1.67 s with one thread.
  uint32_t price_lanes = 0;
  int price_lanes_env = 0;          // EF_PRICE_LANES given: that, whatever the step size
  uint32_t lanes_max_cands = 32768;  // steps below this many candidates: 2 lanes (EF_LANES_MAX_CANDS)
  int spec_price = -1;             // -1: by row size and candidate count (below), 0 off, 1 .. 4 forced
  int spec_mode = 0;               // this step's launch point (1 digest, 2 plans, 3 node keys, 4 key sort; 0: none)
  uint32_t spec_min_rows = 2048;   // rows (S) from which the auto policy prices from the plans on
  uint32_t spec_max_cands = 131072;  // rows of 257..2048: from the first digest on, up to this many candidates
  uint32_t spec_min_cands = 32768;   // and never below this many: a search's small steps price mostly
                                     // visited duplicates speculatively (NasNet-A search 5.5 -> 6.4 s)
  const ef_price_params* spec_pp = nullptr;  // set by ef_expand for step_hash
  bool spec_sharded = false;                 // the step's survivors come from owner verdicts (FIRST)
  bool spec_live = false;                    // this step's speculative pricing was launched
  cudaStream_t st_price = nullptr;
  cudaEvent_t ev_sp0 = nullptr, ev_sp1 = nullptr;
  cudaEvent_t ev_pf0 = nullptr, ev_pf1 = nullptr;  // k_pfx_chain on st_wide, beside the dirty walk
  DevBuf<ef_cand_result> d_spec;
  DevBuf<uint32_t> d_spec_list;
  cudaEvent_t ev_w0 = nullptr, ev_w1 = nullptr;
  cudaEvent_t ev_up = nullptr;    // end of the last asynchronous upload (upload stream)
  cudaEvent_t ev_main = nullptr;  // main-stream work an upload must not overtake
  DevBuf<char> d_up_stage;
  DevBuf<unsigned long long> d_up_off, d_up_dst;
  std::vector<unsigned long long> h_up_off, h_up_dst;
  uint32_t step_S = 0, step_Rs = 0, step_n_parents = 0;
  StepArgs last_step{};
  DevBuf<uint32_t> d_sel;
  DevBuf<unsigned long long> d_dst;
  DevBuf<double> d_tile;  // alpha-prune tile minima

  // visited set (kept at most half full: vis_reserve grows it by rehashing)
  DevBuf<unsigned long long> d_vis, d_vis_count;
  DevBuf<uint32_t> d_vis_err;
  uint32_t vis_mask = 0;
  uint64_t vis_bound = 0;        // upper bound of the stored hashes (exact after every synchronised insert)
  unsigned long long* h_vis = nullptr;  // pinned: count, err

  cudaEvent_t ev[6] = {};
  std::vector<cudaEvent_t> ev_chunk;  // 5 per hashing chunk: dirty | keys | sort | digest
  uint32_t n_chunks = 0;
  float last_ms[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t last_stats[5] = {0, 0, 0, 0, 0};
  uint32_t* pad_counts = nullptr;  // the send counts of the last ef_route_owners_padded (device)
  bool alg_rows = false;  // the last step's alg8 rows hold row indices (price_d1), not algorithm ids
  uint64_t kcount = 0;  // kernels launched by the library (every launch site counts)
  uint64_t kcount_step0 = 0;  // kcount when the last step began
};

#define EF_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(_e);                     \
      return EF_ERR_CUDA;                                                                \
    }                                                                                    \
  } while (0)

#define EF_REQUIRE(cond, msg)  \
  do {                         \
    if (!(cond)) {             \
      ctx->err = (msg);        \
      return EF_ERR_ARG;       \
    }                          \
  } while (0)

static Tables make_tables(ef_ctx* ctx) {
  Tables T{};
  T.sig_desc = ctx->d_sig_desc.p;
  T.sig_info = reinterpret_cast<const uint2*>(ctx->d_sig_info.p);
  T.sig_text_off = ctx->d_text_off.p;
  T.sig_text_len = ctx->d_text_len.p;
  T.sig_text = ctx->d_text.p;
  T.row_off = ctx->d_row_off.p;
  T.row_n = ctx->d_row_n.p;
  T.row_alg = ctx->d_row_alg.p;
  T.row_t = ctx->d_row_t.p;
  T.row_e = ctx->d_row_e.p;
  T.sig_ht_key = ctx->d_sig_ht_key.p;
  T.sig_ht_val = ctx->d_sig_ht_val.p;
  T.sig_ht_mask = ctx->sig_ht_mask;
  T.ws_digest = ctx->d_ws_digest.p;
  T.dv_tuple = ctx->d_dv_tuple.p;
  T.dv_ht_key = ctx->d_dv_ht_key.p;
  T.dv_ht_val = ctx->d_dv_ht_val.p;
  T.dv_ht_mask = ctx->dv_ht_mask;
  T.name_off = ctx->d_name_off.p;
  T.name_len = ctx->d_name_len.p;
  T.names = ctx->d_names.p;
  T.input_text = ctx->d_input_text.p;
  T.input_text_len = (uint32_t)ctx->input_text.size();
  return T;
}

static char* slot_addr(ef_ctx* ctx, uint32_t slot) {
  return ctx->chunks[slot / ctx->slots_per_chunk] + (uint64_t)(slot % ctx->slots_per_chunk) * ctx->geo.bytes;
}

int ef_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

ef_ctx* ef_create(int device) {
  ef_ctx* ctx = new ef_ctx();
  ctx->dev = device;
  // stream priorities: the step's main stream (and its wide-key side stream) above the
  // speculative pricing, so price CTAs only fill what the hashing kernels leave free
  int prio_lo = 0, prio_hi = 0;
  if (cudaSetDevice(device) == cudaSuccess) cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithPriority(&ctx->st, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    delete ctx;
    return nullptr;
  }
  cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (const char* e = getenv("EF_BIG_MERGE")) ctx->big_merge = atoi(e) != 0;
  if (const char* e = getenv("EF_WIDE_MIN")) ctx->wide_min = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_DIRTY_BIG")) ctx->dirty_big = atoi(e) != 0;
  if (const char* e = getenv("EF_WIDE_LPC")) {
    const uint32_t v = (uint32_t)strtoul(e, nullptr, 10);
    ctx->wide_lpc = v >= 32 ? 32u : v >= 16 ? 16u : v >= 8 ? 8u : 4u;
  }
  if (const char* e = getenv("EF_FUSE_MERGE")) ctx->fuse_merge = atoi(e) != 0;
  if (const char* e = getenv("EF_SPEC_PRICE")) ctx->spec_price = atoi(e);
  if (const char* e = getenv("EF_PRICE_LANES")) {
    const uint32_t v = (uint32_t)strtoul(e, nullptr, 10);
    ctx->price_lanes = v >= 8 ? 8u : v >= 4 ? 4u : v >= 2 ? 2u : 0u;
    ctx->price_lanes_env = 1;
  }
  if (const char* e = getenv("EF_SPEC_MIN_ROWS")) ctx->spec_min_rows = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_SPEC_MAX_CANDS")) ctx->spec_max_cands = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_SPEC_MIN_CANDS")) ctx->spec_min_cands = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_DIGEST_PF")) ctx->digest_pf = atoi(e) != 0;
  if (const char* e = getenv("EF_MERGE_SCATTER")) ctx->merge_scatter = atoi(e) != 0;
  if (const char* e = getenv("EF_LANES_MAX_CANDS")) ctx->lanes_max_cands = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_MS_MIN_ROWS")) ctx->ms_min_rows = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_MS_SORT_MIN")) ctx->ms_sort_min_rows = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_PFX_SHARE")) ctx->pfx_share = atoi(e) != 0;
  if (const char* e = getenv("EF_SPARSE_SWEEP")) ctx->sparse_sweep = atoi(e) != 0;
  if (const char* e = getenv("EF_QUAD_MAX")) ctx->quad_max = (uint32_t)strtoul(e, nullptr, 10);
  if (const char* e = getenv("EF_CHUNK_MIB")) ctx->chunk_mib = std::max<uint64_t>(64, strtoull(e, nullptr, 10));
  cudaMallocHost(&ctx->h_scalars, 16 * sizeof(uint32_t));
  cudaStreamCreateWithFlags(&ctx->st_up, cudaStreamNonBlocking);
  cudaStreamCreateWithPriority(&ctx->st_wide, cudaStreamNonBlocking, prio_hi);
  cudaStreamCreateWithPriority(&ctx->st_price, cudaStreamNonBlocking, prio_lo);
  cudaEventCreateWithFlags(&ctx->ev_sp0, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_sp1, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_pf0, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_pf1, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_w0, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_w1, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&ctx->st_copy, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ctx->ev_snap, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_up, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_main, cudaEventDisableTiming);
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  // weight set 0 = "no weights" (digest of the empty message)
  ctx->ws.emplace_back();
  ctx->ws[0].dv[0] = 0;
  return ctx;
}

void ef_destroy(ef_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev);
  cudaStreamSynchronize(ctx->st);
  for (char* c : ctx->chunks) cudaFree(c);
  ctx->d_sig_desc.release();
  ctx->d_text_off.release();
  ctx->d_text_len.release();
  ctx->d_row_off.release();
  ctx->d_row_n.release();
  ctx->d_sig_ht_val.release();
  ctx->d_dv_ht_val.release();
  ctx->d_name_off.release();
  ctx->d_name_len.release();
  ctx->d_text.release();
  ctx->d_names.release();
  ctx->d_input_text.release();
  ctx->d_row_alg.release();
  ctx->d_dv_tuple.release();
  ctx->d_row_t.release();
  ctx->d_row_e.release();
  ctx->d_sig_ht_key.release();
  ctx->d_dv_ht_key.release();
  ctx->d_ws_digest.release();
  ctx->d_pool.release();
  ctx->d_parent_addr.release();
  ctx->d_sites.release();
  ctx->d_step_key.release();
  ctx->d_addr_a.release();
  ctx->d_addr_b.release();
  ctx->d_pscratch.release();
  ctx->d_site_count.release();
  ctx->d_cand_off.release();
  ctx->d_step_seq.release();
  ctx->d_scalars.release();
  ctx->d_stage.release();
  ctx->d_req_dv.release();
  ctx->d_res.release();
  ctx->d_res_aux.release();
  if (ctx->st_copy) cudaStreamSynchronize(ctx->st_copy);
  ctx->d_res_snap.release();
  ctx->d_req_sig.release();
  ctx->d_hash_out.release();
  ctx->d_sperm.release();
  ctx->d_vis.release();
  ctx->d_vis_count.release();
  ctx->d_vis_err.release();
  ctx->d_tile.release();
  if (ctx->h_vis) cudaFreeHost(ctx->h_vis);
  ctx->d_plan.release();
  ctx->d_route.release();
  ctx->d_stats.release();
  ctx->d_perm.release();
  ctx->d_step_ord.release();
  ctx->d_plist.release();
  ctx->d_sig_info.release();
  ctx->d_alg8.release();
  ctx->d_algt.release();
  ctx->d_nsk.release();
  ctx->sc[0].release();
  ctx->sc[1].release();
  ctx->d_up_stage.release();
  ctx->d_up_off.release();
  ctx->d_up_dst.release();
  if (ctx->ev_up) cudaEventDestroy(ctx->ev_up);
  if (ctx->ev_main) cudaEventDestroy(ctx->ev_main);
  if (ctx->st_up) cudaStreamDestroy(ctx->st_up);
  if (ctx->st_wide) cudaStreamDestroy(ctx->st_wide);
  if (ctx->st_price) cudaStreamDestroy(ctx->st_price);
  if (ctx->ev_sp0) cudaEventDestroy(ctx->ev_sp0);
  if (ctx->ev_sp1) cudaEventDestroy(ctx->ev_sp1);
  if (ctx->ev_pf0) cudaEventDestroy(ctx->ev_pf0);
  if (ctx->ev_pf1) cudaEventDestroy(ctx->ev_pf1);
  ctx->d_spec.release();
  ctx->d_spec_list.release();
  ctx->d_upd_sig.release();
  ctx->d_upd_dv.release();
  if (ctx->ev_w0) cudaEventDestroy(ctx->ev_w0);
  if (ctx->ev_w1) cudaEventDestroy(ctx->ev_w1);
  if (ctx->st_copy) cudaStreamDestroy(ctx->st_copy);
  if (ctx->ev_snap) cudaEventDestroy(ctx->ev_snap);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  ctx->d_sel.release();
  ctx->d_dst.release();
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  for (auto& e : ctx->ev_chunk) cudaEventDestroy(e);
  if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
  cudaStreamDestroy(ctx->st);
  delete ctx;
}

const char* ef_error(ef_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// ---------------------------------------------------------------------------------------------
// tables
// ---------------------------------------------------------------------------------------------

int ef_sig_put(ef_ctx* ctx, uint32_t id, const ef_sig_desc* desc, const char* text, uint32_t text_len, int exact) {
  EF_REQUIRE(desc && text, "ef_sig_put: null argument");
  if (id >= ctx->sig_desc.size()) {
    ctx->sig_desc.resize(id + 1);
    ctx->sig_exact.resize(id + 1, 0);
    ctx->sig_text.resize(id + 1);
    ctx->row_alg.resize(id + 1);
    ctx->row_t.resize(id + 1);
    ctx->row_e.resize(id + 1);
  }
  if (id < ctx->c_ns) {  // a committed id changes: its entries are re-sent, its lookup rebuilt if keyed
    if (std::memcmp(&ctx->sig_desc[id], desc, sizeof(ef_sig_desc)) || ctx->sig_exact[id] != (exact ? 1 : 0))
      ctx->sig_key_changed = true;
    ctx->sig_touched.push_back(id);
  }
  ctx->sig_desc[id] = *desc;
  ctx->sig_exact[id] = exact ? 1 : 0;
  ctx->sig_text[id].assign(text, text_len);
  ctx->dirty = true;
  return EF_OK;
}

int ef_sig_costs(ef_ctx* ctx, uint32_t id, uint32_t n, const int32_t* alg, const double* time_ms, const double* energy) {
  EF_REQUIRE(id < ctx->sig_desc.size(), "ef_sig_costs: unknown signature id");
  EF_REQUIRE(n <= 255, "ef_sig_costs: too many algorithms");
  if (ctx->row_alg[id].size() == n && std::equal(alg, alg + n, ctx->row_alg[id].begin()) &&
      std::memcmp(ctx->row_t[id].data(), time_ms, n * 8) == 0 && std::memcmp(ctx->row_e[id].data(), energy, n * 8) == 0)
    return EF_OK;  // the same rows (a search re-binding its cost source): nothing to send
  if (id < ctx->c_ns) ctx->sig_touched.push_back(id);
  ctx->row_alg[id].assign(alg, alg + n);
  ctx->row_t[id].assign(time_ms, time_ms + n);
  ctx->row_e[id].assign(energy, energy + n);
  ctx->dirty = true;
  return EF_OK;
}

int ef_name_put(ef_ctx* ctx, uint32_t id, const char* name, uint32_t len) {
  if (id >= ctx->names.size()) ctx->names.resize(id + 1);
  if (id < ctx->c_names) ctx->names_changed = true;
  ctx->names[id].assign(name, len);
  ctx->dirty = true;
  return EF_OK;
}

static int pool_alloc(ef_ctx* ctx, uint64_t n, uint64_t* off) {
  uint64_t need = ctx->pool_used + n + 2;  // +2 keeps zero-length sets at distinct offsets
  EF_CUDA(ctx->d_pool.reserve(need, ctx->st, true));
  *off = ctx->pool_used;
  ctx->pool_used += n;
  return EF_OK;
}

int ef_wset_put(ef_ctx* ctx, uint32_t id, int32_t kind, int32_t oc, const double* w, uint64_t w_n, const double* b,
                uint64_t b_n, const char* hdr_w, uint32_t hlen_w, const char* hdr_b, uint32_t hlen_b) {
  EF_REQUIRE(id != kEmptyWset || (w_n == 0 && b_n == 0), "weight set 0 is reserved for 'no weights'");
  if (id >= ctx->ws.size()) ctx->ws.resize(id + 1);
  if (id < ctx->c_nw) ctx->dv_changed = true;
  WeightSet& S = ctx->ws[id];
  S = WeightSet();
  S.kind = kind;
  S.oc = oc;
  S.w_n = w_n;
  S.b_n = b_n;
  S.has_b = b != nullptr;
  if (hdr_w) S.hdr_w.assign(hdr_w, hlen_w);
  if (hdr_b) S.hdr_b.assign(hdr_b, hlen_b);
  int rc = pool_alloc(ctx, w_n, &S.w_off);
  if (rc) return rc;
  rc = pool_alloc(ctx, b_n, &S.b_off);
  if (rc) return rc;
  if (w_n) EF_CUDA(cudaMemcpyAsync(ctx->d_pool.p + S.w_off, w, w_n * 8, cudaMemcpyHostToDevice, ctx->st));
  if (b_n && b) EF_CUDA(cudaMemcpyAsync(ctx->d_pool.p + S.b_off, b, b_n * 8, cudaMemcpyHostToDevice, ctx->st));
  // host copies for the digest (taken on host cores at commit: one BLAKE2b stream per set)
  S.hw.resize(w_n);
  if (w_n) std::memcpy(S.hw.data(), w, w_n * 8);
  S.hb.assign(b_n, 0);
  if (b_n && b) std::memcpy(S.hb.data(), b, b_n * 8);
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  ctx->dirty = true;
  return EF_OK;
}

int ef_wset_derive(ef_ctx* ctx, uint32_t id, int32_t op, uint32_t a, uint32_t b, int32_t s0, const char* hdr_w,
                   uint32_t hlen_w, const char* hdr_b, uint32_t hlen_b) {
  EF_REQUIRE(a < ctx->ws.size() && ctx->ws[a].kind == EF_K_CONV2D, "ef_wset_derive: source must be a conv weight set");
  const WeightSet A = ctx->ws[a];
  EF_REQUIRE(A.oc > 0, "ef_wset_derive: conv without out channels");
  const uint64_t inner = A.w_n / (uint64_t)A.oc;
  WeightSet S;
  S.kind = EF_K_CONV2D;
  S.has_b = true;
  S.dv[0] = op;
  S.dv[1] = (int32_t)a;
  S.dv[2] = (int32_t)b;
  S.dv[3] = s0;
  S.hdr_w.assign(hdr_w, hlen_w);
  S.hdr_b.assign(hdr_b, hlen_b);
  if (op == EF_D_MERGE) {
    EF_REQUIRE(b < ctx->ws.size() && ctx->ws[b].kind == EF_K_CONV2D, "merge needs two conv weight sets");
    S.oc = A.oc + ctx->ws[b].oc;
  } else if (op == EF_D_SLICE_LO) {
    S.oc = s0;
  } else if (op == EF_D_SLICE_HI) {
    S.oc = A.oc - s0;
  } else if (op == EF_D_FOLD) {
    EF_REQUIRE(b < ctx->ws.size() && ctx->ws[b].kind == EF_K_BATCHNORM, "fold needs a batchnorm weight set");
    S.oc = A.oc;
  } else {
    EF_REQUIRE(false, "ef_wset_derive: unknown op");
  }
  S.w_n = (uint64_t)S.oc * inner;
  S.b_n = (uint64_t)S.oc;
  int rc = pool_alloc(ctx, S.w_n, &S.w_off);
  if (rc) return rc;
  rc = pool_alloc(ctx, S.b_n, &S.b_off);
  if (rc) return rc;
  if (id >= ctx->ws.size()) ctx->ws.resize(id + 1);
  if (id < ctx->c_nw) ctx->dv_changed = true;
  ctx->ws[id] = S;
  ctx->dirty = true;
  return EF_OK;
}

int ef_wset_read(ef_ctx* ctx, uint32_t id, double* w, uint64_t* w_n, double* b, uint64_t* b_n) {
  EF_REQUIRE(id < ctx->ws.size(), "ef_wset_read: unknown weight set");
  const WeightSet& S = ctx->ws[id];
  if (w_n) {
    if (w) EF_CUDA(cudaMemcpyAsync(w, ctx->d_pool.p + S.w_off, std::min(*w_n, S.w_n) * 8, cudaMemcpyDeviceToHost, ctx->st));
    *w_n = S.w_n;
  }
  if (b_n) {
    uint64_t have = S.has_b ? S.b_n : 0;
    if (b && have) EF_CUDA(cudaMemcpyAsync(b, ctx->d_pool.p + S.b_off, std::min(*b_n, have) * 8, cudaMemcpyDeviceToHost, ctx->st));
    *b_n = have;
  }
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_wset_digest(ef_ctx* ctx, uint32_t id, uint8_t out[16]) {
  EF_REQUIRE(id < ctx->ws.size() && ctx->ws[id].ready, "ef_wset_digest: weight set not committed");
  EF_CUDA(cudaMemcpyAsync(out, ctx->d_ws_digest.p + 2 * id, 16, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

template <typename T>
static int upload(ef_ctx* ctx, DevBuf<T>& buf, const std::vector<T>& v) {
  EF_CUDA(buf.reserve(std::max<size_t>(v.size(), 1), ctx->st));
  if (!v.empty()) EF_CUDA(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->st));
  return EF_OK;
}

static uint32_t pow2_at_least(uint64_t n) {
  uint32_t m = 16;
  while (m < n) m <<= 1;
  return m;
}

// hi - lo host elements (src) to [lo, hi) of a device array that keeps its contents as it grows
// to `total` elements
template <typename T>
static int upload_range(ef_ctx* ctx, DevBuf<T>& buf, const T* src, size_t lo, size_t hi, size_t total) {
  EF_CUDA(buf.reserve(std::max<size_t>(total, 1), ctx->st, true));
  if (hi > lo) {
    EF_CUDA(cudaMemcpyAsync(buf.p + lo, src, (hi - lo) * sizeof(T), cudaMemcpyHostToDevice, ctx->st));
    ctx->commit_bytes += (hi - lo) * sizeof(T);
  }
  return EF_OK;
}

// the sweep's exact skips of price_d1 (no row below row 0 in time / in energy) + row count
static uint32_t sig_info_word(const ef_ctx* ctx, size_t i) {
  const uint32_t rn = (uint32_t)ctx->row_alg[i].size();
  uint32_t y = rn | (ctx->sig_desc[i].kind == EF_K_INPUT ? kInfoInput : 0u);
  if (rn) {
    bool tmin = true, emin = true;
    for (uint32_t q = 1; q < rn; ++q) {
      tmin = tmin && ctx->row_t[i][q] >= ctx->row_t[i][0];
      emin = emin && ctx->row_e[i][q] >= ctx->row_e[i][0];
    }
    y |= (tmin ? kInfoTMin : 0u) | (emin ? kInfoEMin : 0u);
  }
  return y;
}

// insert id i into a host lookup table; the exact-signature table keeps the first of equal descs
static bool ht_insert(std::vector<unsigned long long>& keys, std::vector<uint32_t>& vals, uint64_t k, uint32_t i,
                      const ef_ctx* ctx, bool sig, std::vector<HtUpd>* upd) {
  const uint32_t mask = (uint32_t)keys.size() - 1;
  uint32_t s = (uint32_t)k & mask;
  while (keys[s]) {
    if (sig && keys[s] == k && desc_eq(ctx->sig_desc[vals[s]], ctx->sig_desc[i])) return false;
    s = (s + 1) & mask;
  }
  keys[s] = k;
  vals[s] = i;
  if (upd) upd->push_back(HtUpd{s, i, k});
  return true;
}

static int ht_scatter(ef_ctx* ctx, DevBuf<HtUpd>& ub, const std::vector<HtUpd>& upd, unsigned long long* keys,
                      uint32_t* vals) {
  if (upd.empty()) return EF_OK;
  int rc = upload(ctx, ub, upd);
  if (rc) return rc;
  ctx->commit_bytes += upd.size() * sizeof(HtUpd);
  const uint32_t n = (uint32_t)upd.size();
  ++ctx->kcount, k_ht_scatter<<<std::min<uint32_t>((n + 255) / 256, 64), 256, 0, ctx->st>>>(keys, vals, ub.p, n);
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

// signatures: texts, cost rows, per-id arrays and the exact-signature lookup.  Ids committed
// before and unchanged are not sent again; changed ones get fresh text / row space at the end
// (the old space is left unused) and their per-id entries re-sent.
static int commit_sigs(ef_ctx* ctx) {
  const size_t ns = ctx->sig_desc.size();
  const bool full = !ctx->c_valid;
  std::vector<uint32_t> ids;
  if (full) {
    ctx->text_used = ctx->rows_used = 0;
    for (size_t i = 0; i < ns; ++i) ids.push_back((uint32_t)i);
  } else {
    std::sort(ctx->sig_touched.begin(), ctx->sig_touched.end());
    ctx->sig_touched.erase(std::unique(ctx->sig_touched.begin(), ctx->sig_touched.end()), ctx->sig_touched.end());
    ids = ctx->sig_touched;
    for (size_t i = ctx->c_ns; i < ns; ++i) ids.push_back((uint32_t)i);
  }
  ctx->h_toff.resize(ns);
  ctx->h_tlen.resize(ns);
  ctx->h_roff.resize(ns);
  ctx->h_rn.resize(ns);
  ctx->h_info.resize(2 * std::max<size_t>(ns, 1), 0);
  // texts 8-byte aligned and zero padded (the hash kernel reads them as words), +8 zero bytes
  std::vector<uint8_t> text;
  std::vector<int32_t> ralg;
  std::vector<double> rt, re;
  for (uint32_t i : ids) {
    ctx->h_toff[i] = (uint32_t)(ctx->text_used + text.size());
    ctx->h_tlen[i] = (uint32_t)ctx->sig_text[i].size();
    text.insert(text.end(), ctx->sig_text[i].begin(), ctx->sig_text[i].end());
    while (text.size() % 8) text.push_back(0);
    ctx->h_roff[i] = (uint32_t)(ctx->rows_used + ralg.size());
    ctx->h_rn[i] = (uint32_t)ctx->row_alg[i].size();
    ralg.insert(ralg.end(), ctx->row_alg[i].begin(), ctx->row_alg[i].end());
    rt.insert(rt.end(), ctx->row_t[i].begin(), ctx->row_t[i].end());
    re.insert(re.end(), ctx->row_e[i].begin(), ctx->row_e[i].end());
    ctx->h_info[2 * i] = ctx->h_roff[i];
    ctx->h_info[2 * i + 1] = sig_info_word(ctx, i);
  }
  text.resize(text.size() + 8, 0);
  int rc;
  const uint64_t t0 = ctx->text_used, r0 = ctx->rows_used;
  if ((rc = upload_range(ctx, ctx->d_text, text.data(), t0, t0 + text.size(), t0 + text.size())) ||
      (rc = upload_range(ctx, ctx->d_row_alg, ralg.data(), r0, r0 + ralg.size(), r0 + ralg.size())) ||
      (rc = upload_range(ctx, ctx->d_row_t, rt.data(), r0, r0 + rt.size(), r0 + rt.size())) ||
      (rc = upload_range(ctx, ctx->d_row_e, re.data(), r0, r0 + re.size(), r0 + re.size())))
    return rc;
  ctx->text_used += text.size() - 8;  // the padding is overwritten by the next commit's texts
  ctx->rows_used += ralg.size();
  // per-id arrays from the first changed id on
  const size_t lo = ids.empty() ? ns : ids.front();
  if ((rc = upload_range(ctx, ctx->d_sig_desc, ctx->sig_desc.data() + lo, lo, ns, ns)) ||
      (rc = upload_range(ctx, ctx->d_text_off, ctx->h_toff.data() + lo, lo, ns, ns)) ||
      (rc = upload_range(ctx, ctx->d_text_len, ctx->h_tlen.data() + lo, lo, ns, ns)) ||
      (rc = upload_range(ctx, ctx->d_row_off, ctx->h_roff.data() + lo, lo, ns, ns)) ||
      (rc = upload_range(ctx, ctx->d_row_n, ctx->h_rn.data() + lo, lo, ns, ns)) ||
      (rc = upload_range(ctx, ctx->d_sig_info, ctx->h_info.data() + 2 * lo, 2 * lo, 2 * ns, 2 * std::max<size_t>(ns, 1))))
    return rc;
  // exact-signature lookup: new exact ids into the table, or a rebuild (first commit, a keyed
  // id changed, or the load would pass 1/2: rebuilt at load <= 1/4, so rebuilds are amortised)
  size_t n_exact_new = 0;
  for (size_t i = full ? 0 : ctx->c_ns; i < ns; ++i) n_exact_new += ctx->sig_exact[i] ? 1 : 0;
  const bool rebuild = full || ctx->sig_key_changed || 2ull * (ctx->sig_ht_n + n_exact_new) + 2 > ctx->h_sig_ht_key.size();
  if (rebuild) {
    const uint32_t cap = pow2_at_least(4 * ns + 2);
    ctx->h_sig_ht_key.assign(cap, 0);
    ctx->h_sig_ht_val.assign(cap, 0);
    ctx->sig_ht_n = 0;
    for (size_t i = 0; i < ns; ++i)
      if (ctx->sig_exact[i])
        ctx->sig_ht_n += ht_insert(ctx->h_sig_ht_key, ctx->h_sig_ht_val, desc_key(ctx->sig_desc[i]), (uint32_t)i, ctx, true, nullptr);
    ctx->sig_ht_mask = cap - 1;
    ctx->commit_bytes += (uint64_t)cap * 12;
    if ((rc = upload(ctx, ctx->d_sig_ht_key, ctx->h_sig_ht_key)) || (rc = upload(ctx, ctx->d_sig_ht_val, ctx->h_sig_ht_val)))
      return rc;
  } else {
    std::vector<HtUpd> upd;
    for (size_t i = ctx->c_ns; i < ns; ++i)
      if (ctx->sig_exact[i])
        ctx->sig_ht_n += ht_insert(ctx->h_sig_ht_key, ctx->h_sig_ht_val, desc_key(ctx->sig_desc[i]), (uint32_t)i, ctx, true, &upd);
    if ((rc = ht_scatter(ctx, ctx->d_upd_sig, upd, ctx->d_sig_ht_key.p, ctx->d_sig_ht_val.p))) return rc;
  }
  ctx->sig_touched.clear();
  ctx->sig_key_changed = false;
  ctx->c_ns = ns;
  return EF_OK;
}

// node names (appended) and the graph-input text (sent when the geometry set it)
static int commit_names(ef_ctx* ctx) {
  const size_t nn = ctx->names.size();
  const bool full = !ctx->c_valid || ctx->names_changed;
  const size_t lo = full ? 0 : ctx->c_names;
  if (full) ctx->name_used = 0;
  std::vector<uint32_t> off(nn), len(nn);
  std::vector<uint8_t> pool;
  for (size_t i = lo; i < nn; ++i) {
    off[i] = (uint32_t)(ctx->name_used + pool.size());
    len[i] = (uint32_t)ctx->names[i].size();
    pool.insert(pool.end(), ctx->names[i].begin(), ctx->names[i].end());
  }
  pool.push_back(0);
  const uint64_t p0 = ctx->name_used;
  int rc;
  if ((rc = upload_range(ctx, ctx->d_name_off, off.data() + lo, lo, nn, nn)) ||
      (rc = upload_range(ctx, ctx->d_name_len, len.data() + lo, lo, nn, nn)) ||
      (rc = upload_range(ctx, ctx->d_names, pool.data(), p0, p0 + pool.size(), p0 + pool.size())))
    return rc;
  ctx->name_used += pool.size() - 1;
  ctx->names_changed = false;
  ctx->c_names = nn;
  if (ctx->input_changed || !ctx->c_valid) {
    std::vector<uint8_t> it(ctx->input_text.begin(), ctx->input_text.end());
    it.resize(((it.size() + 7) & ~size_t(7)) + 8, 0);  // 8-byte words, zero padded (k_digest)
    if ((rc = upload(ctx, ctx->d_input_text, it))) return rc;
    ctx->commit_bytes += it.size();
    ctx->input_changed = false;
  }
  return EF_OK;
}

// derivation tuples and their lookup (weight sets are only appended during a search)
static int commit_derives(ef_ctx* ctx) {
  const size_t nw = ctx->ws.size();
  const bool full = !ctx->c_valid || ctx->dv_changed;
  const size_t lo = full ? 0 : ctx->c_nw;
  std::vector<int32_t> tup(4 * nw, 0);
  for (size_t i = lo; i < nw; ++i)
    for (int k = 0; k < 4; ++k) tup[4 * i + k] = ctx->ws[i].dv[k];
  int rc;
  if ((rc = upload_range(ctx, ctx->d_dv_tuple, tup.data() + 4 * lo, 4 * lo, 4 * nw, 4 * nw))) return rc;
  auto key_of = [&](size_t i) {
    const int32_t* d = ctx->ws[i].dv;
    return (uint64_t)derive_key(d[0], (uint32_t)d[1], (uint32_t)d[2], d[3]);
  };
  size_t n_dv = 0;
  for (size_t i = 0; i < nw; ++i) n_dv += ctx->ws[i].dv[0] != 0;
  if (full || 2ull * n_dv + 2 > ctx->h_dv_ht_key.size()) {
    const uint32_t cap = pow2_at_least(4 * nw + 2);
    ctx->h_dv_ht_key.assign(cap, 0);
    ctx->h_dv_ht_val.assign(cap, 0);
    for (size_t i = 0; i < nw; ++i)
      if (ctx->ws[i].dv[0] != 0) ht_insert(ctx->h_dv_ht_key, ctx->h_dv_ht_val, key_of(i), (uint32_t)i, ctx, false, nullptr);
    ctx->dv_ht_mask = cap - 1;
    ctx->commit_bytes += (uint64_t)cap * 12;
    if ((rc = upload(ctx, ctx->d_dv_ht_key, ctx->h_dv_ht_key)) || (rc = upload(ctx, ctx->d_dv_ht_val, ctx->h_dv_ht_val)))
      return rc;
  } else {
    std::vector<HtUpd> upd;
    for (size_t i = lo; i < nw; ++i)
      if (ctx->ws[i].dv[0] != 0) ht_insert(ctx->h_dv_ht_key, ctx->h_dv_ht_val, key_of(i), (uint32_t)i, ctx, false, &upd);
    if ((rc = ht_scatter(ctx, ctx->d_upd_dv, upd, ctx->d_dv_ht_key.p, ctx->d_dv_ht_val.p))) return rc;
  }
  ctx->dv_changed = false;
  ctx->c_nw = nw;
  return EF_OK;
}

int ef_tables_commit(ef_ctx* ctx) {
  cudaSetDevice(ctx->dev);
  ctx->commit_bytes = 0;
  int rc;
  if ((rc = commit_sigs(ctx)) || (rc = commit_names(ctx)) || (rc = commit_derives(ctx))) return rc;
  ctx->c_valid = true;
  const size_t nw = ctx->ws.size();
  // derived tensors, in id order (a derivation may use an earlier derived set)
  EF_CUDA(ctx->d_ws_digest.reserve(2 * nw + 2, ctx->st, true));
  std::vector<uint32_t> pending;
  for (size_t i = 0; i < nw; ++i)
    if (!ctx->ws[i].ready) pending.push_back((uint32_t)i);
  if (!pending.empty()) {
    std::vector<DeriveJob> djobs;
    for (uint32_t i : pending) {
      const WeightSet& S = ctx->ws[i];
      if (S.dv[0] == 0) continue;
      const WeightSet& A = ctx->ws[S.dv[1]];
      DeriveJob J{};
      J.op = S.dv[0];
      J.wa = ctx->d_pool.p + A.w_off;
      J.ba = A.has_b ? ctx->d_pool.p + A.b_off : nullptr;
      J.oc_a = (uint64_t)A.oc;
      J.inner = A.w_n / (uint64_t)A.oc;
      J.s0 = S.dv[3];
      if (J.op == EF_D_MERGE || J.op == EF_D_FOLD) {
        const WeightSet& B = ctx->ws[S.dv[2]];
        J.wb = ctx->d_pool.p + B.w_off;
        J.bb = B.has_b ? ctx->d_pool.p + B.b_off : nullptr;
        J.oc_b = (uint64_t)B.oc;
      }
      J.w_out = ctx->d_pool.p + S.w_off;
      J.b_out = ctx->d_pool.p + S.b_off;
      J.w_n = S.w_n;
      J.b_n = S.b_n;
      djobs.push_back(J);
    }
    if (!djobs.empty()) {
      // one job per launch keeps dependencies between derived sets ordered on the stream
      DevBuf<DeriveJob> dj;
      EF_CUDA(dj.reserve(djobs.size(), ctx->st));
      EF_CUDA(cudaMemcpyAsync(dj.p, djobs.data(), djobs.size() * sizeof(DeriveJob), cudaMemcpyHostToDevice, ctx->st));
      for (size_t j = 0; j < djobs.size(); ++j) ++ctx->kcount, k_derive<<<ctx->n_sm * 4, 256, 0, ctx->st>>>(dj.p + j, 1);
      EF_CUDA(cudaGetLastError());
      EF_CUDA(cudaStreamSynchronize(ctx->st));
      dj.release();
    }
    // derived tensors back to the host for their digests
    for (uint32_t i : pending) {
      WeightSet& S = ctx->ws[i];
      if (S.dv[0] == 0) continue;
      S.hw.resize(S.w_n);
      S.hb.resize(S.b_n);
      if (S.w_n) EF_CUDA(cudaMemcpy(S.hw.data(), ctx->d_pool.p + S.w_off, S.w_n * 8, cudaMemcpyDeviceToHost));
      if (S.b_n) EF_CUDA(cudaMemcpy(S.hb.data(), ctx->d_pool.p + S.b_off, S.b_n * 8, cudaMemcpyDeviceToHost));
    }
    // Digests (graph.py:510-517) on host cores, a set per thread.  A digest is one BLAKE2b
    // stream over headers and tensor bytes: inherently sequential, and a CPU core runs one
    // stream several times faster than a lone GPU thread (ResNet-50 merged convs: 19 MB).
    // Header order is the sorted key order of the reference's weight dict (bias < weight,
    // scale < shift).
    ctx->h_ws_digest.resize(2 * nw, 0);
    std::atomic<size_t> next{0};
    auto worker = [&]() {
      for (size_t j; (j = next.fetch_add(1)) < pending.size();) {
        const uint32_t i = pending[j];
        const WeightSet& S = ctx->ws[i];
        const std::string* h0 = nullptr;
        const std::string* h1 = nullptr;
        const std::vector<uint64_t>* t0 = nullptr;
        const std::vector<uint64_t>* t1 = nullptr;
        if (S.kind == EF_K_CONV2D) {
          if (S.has_b) {
            h0 = &S.hdr_b, t0 = &S.hb, h1 = &S.hdr_w, t1 = &S.hw;
          } else {
            h0 = &S.hdr_w, t0 = &S.hw;
          }
        } else if (S.kind == EF_K_BATCHNORM) {
          h0 = &S.hdr_w, t0 = &S.hw, h1 = &S.hdr_b, t1 = &S.hb;
        } else if (S.kind == EF_K_MATMUL) {
          h0 = &S.hdr_w, t0 = &S.hw;
        }
        B2b st;
        st.init(16);
        for (const auto& [h, t] : {std::make_pair(h0, t0), std::make_pair(h1, t1)}) {
          if (h) st.bytes(reinterpret_cast<const uint8_t*>(h->data()), (uint32_t)h->size());
          if (t)
            for (uint64_t x : *t) st.word_le(x);
        }
        st.final();
        ctx->h_ws_digest[2 * i] = st.h[0];
        ctx->h_ws_digest[2 * i + 1] = st.h[1];
      }
    };
    const size_t nt = std::min<size_t>(pending.size(), std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    const size_t d0 = 2ull * pending.front();  // the sets digested now (ids ascending)
    EF_CUDA(cudaMemcpyAsync(ctx->d_ws_digest.p + d0, ctx->h_ws_digest.data() + d0, (2 * nw - d0) * 8,
                            cudaMemcpyHostToDevice, ctx->st));
    ctx->commit_bytes += (2 * nw - d0) * 8;
    for (uint32_t i : pending) {
      WeightSet& S = ctx->ws[i];
      std::vector<uint64_t>().swap(S.hw);
      std::vector<uint64_t>().swap(S.hb);
    }
    for (uint32_t i : pending) ctx->ws[i].ready = true;
  }
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  ctx->dirty = false;
  return EF_OK;
}

// ---------------------------------------------------------------------------------------------
// records
// ---------------------------------------------------------------------------------------------

int ef_set_geometry(ef_ctx* ctx, uint32_t cap_nodes, uint32_t cap_refs, uint32_t cap_outs, const char* input_text,
                    uint32_t input_text_len, ef_geometry* out) {
  EF_REQUIRE(cap_nodes > 0 && cap_nodes < (1u << 24), "ef_set_geometry: cap_nodes out of range");
  EF_REQUIRE(!ctx->have_geo || ctx->n_slots == ctx->free_slots.size(), "ef_set_geometry: records still in use");
  for (char* c : ctx->chunks) cudaFree(c);
  ctx->chunks.clear();
  ctx->free_slots.clear();
  ctx->n_slots = 0;
  auto al = [](uint32_t x) { return (x + 15u) & ~15u; };
  Geo& g = ctx->geo;
  g.cap_nodes = cap_nodes;
  g.cap_refs = std::max<uint32_t>(cap_refs, 1);
  g.cap_outs = std::max<uint32_t>(cap_outs, 1);
  uint32_t o = 64;
  g.o_nid = o;
  o = al(o + 4 * cap_nodes);
  g.o_sig = o;
  o = al(o + 4 * cap_nodes);
  g.o_aux = o;
  o = al(o + 4 * cap_nodes);
  g.o_nin = o;
  o = al(o + 4 * cap_nodes);
  g.o_inoff = o;
  o = al(o + 4 * (cap_nodes + 1));
  g.o_topo = o;
  o = al(o + 4 * cap_nodes);
  g.o_refs = o;
  o = al(o + 4 * g.cap_refs);
  g.o_outs = o;
  o = al(o + 4 * g.cap_outs);
  g.o_keys = o;
  o = al(o + 16 * cap_nodes);
  g.o_alg = o;
  o = al(o + cap_nodes);
  g.o_sperm = o;
  o = al(o + 4 * cap_nodes);
  g.o_skeys = o;
  o = al(o + 16 * cap_nodes);
  g.o_srank = o;
  o = al(o + 4 * cap_nodes);
  g.bytes = o;
  ctx->slots_per_chunk = std::max<uint32_t>(1, (uint32_t)((64ull << 20) / g.bytes));
  ctx->input_text.assign(input_text ? input_text : "", input_text ? input_text_len : 0);
  ctx->input_changed = true;
  ctx->have_geo = true;
  ctx->dirty = true;
  if (out) {
    out->cap_nodes = g.cap_nodes;
    out->cap_refs = g.cap_refs;
    out->cap_outs = g.cap_outs;
    out->record_bytes = g.bytes;
    out->off_nid = g.o_nid;
    out->off_sig = g.o_sig;
    out->off_aux = g.o_aux;
    out->off_nin = g.o_nin;
    out->off_inoff = g.o_inoff;
    out->off_topo = g.o_topo;
    out->off_refs = g.o_refs;
    out->off_outs = g.o_outs;
    out->off_keys = g.o_keys;
    out->off_alg = g.o_alg;
    out->off_sperm = g.o_sperm;
    out->off_skeys = g.o_skeys;
    out->off_srank = g.o_srank;
  }
  return EF_OK;
}

int ef_record_alloc(ef_ctx* ctx, uint32_t* slot) {
  EF_REQUIRE(ctx->have_geo, "ef_record_alloc: no geometry");
  if (ctx->free_slots.empty()) {
    char* chunk = nullptr;
    EF_CUDA(cudaMalloc(&chunk, (uint64_t)ctx->slots_per_chunk * ctx->geo.bytes));
    uint32_t base = (uint32_t)ctx->chunks.size() * ctx->slots_per_chunk;
    ctx->chunks.push_back(chunk);
    for (uint32_t i = ctx->slots_per_chunk; i-- > 0;) ctx->free_slots.push_back(base + i);
    ctx->n_slots += ctx->slots_per_chunk;
  }
  *slot = ctx->free_slots.back();
  ctx->free_slots.pop_back();
  return EF_OK;
}

int ef_record_free(ef_ctx* ctx, uint32_t slot) {
  EF_REQUIRE(slot < ctx->n_slots, "ef_record_free: bad slot");
  ctx->free_slots.push_back(slot);
  return EF_OK;
}

int ef_records_alloc(ef_ctx* ctx, uint32_t n, uint32_t* slots) {
  for (uint32_t i = 0; i < n; ++i) {
    int rc = ef_record_alloc(ctx, slots + i);
    if (rc) return rc;
  }
  return EF_OK;
}

int ef_records_free(ef_ctx* ctx, const uint32_t* slots, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) EF_REQUIRE(slots[i] < ctx->n_slots, "ef_records_free: bad slot");
  ctx->free_slots.insert(ctx->free_slots.end(), slots, slots + n);
  return EF_OK;
}

int ef_record_write(ef_ctx* ctx, uint32_t slot, const void* host, uint64_t bytes) {
  EF_REQUIRE(slot < ctx->n_slots && bytes <= ctx->geo.bytes, "ef_record_write: bad slot/size");
  EF_CUDA(cudaMemcpyAsync(slot_addr(ctx, slot), host, bytes, cudaMemcpyHostToDevice, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_record_read(ef_ctx* ctx, uint32_t slot, void* host, uint64_t bytes) {
  EF_REQUIRE(slot < ctx->n_slots && bytes <= ctx->geo.bytes, "ef_record_read: bad slot/size");
  EF_CUDA(cudaMemcpyAsync(host, slot_addr(ctx, slot), bytes, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}


// Node keys, sorted order, sorted keys, ranks and graph hash of whole records (uploads and
// kept candidates): the step's job pipeline with every node a job (ef_step.cuh, full mode).
static int sort_fresh_keys(ef_ctx* ctx, Scratch& sc, cudaStream_t st, const VArgs& V);

// node keys: a thread per candidate when the chunk fills the GPU, four lanes per candidate
// (lower latency per compression) when it does not
static int launch_wide(ef_ctx* ctx, cudaStream_t st, const VArgs& V) {
  const uint32_t lpc = ctx->wide_lpc;
  const uint32_t per_block = 4u * (32u / lpc);  // candidates per 128-thread block
  const uint32_t gw = std::max<uint32_t>(1, std::min<uint32_t>((V.n + per_block - 1) / per_block, ctx->n_sm * 16));
  if (lpc == 32) ++ctx->kcount, k_keys_wide<128, 32><<<gw, 128, 0, st>>>(V);
  else if (lpc == 16) ++ctx->kcount, k_keys_wide<128, 16><<<gw, 128, 0, st>>>(V);
  else if (lpc == 8) ++ctx->kcount, k_keys_wide<128, 8><<<gw, 128, 0, st>>>(V);
  else ++ctx->kcount, k_keys_wide<128, 4><<<gw, 128, 0, st>>>(V);
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

static int launch_keys(ef_ctx* ctx, cudaStream_t st, const VArgs& V) {
  const bool wide = V.wide_min && st == ctx->st;
  int rc;
  if (wide) {  // large graphs: the longest candidates by level (lane groups), on a side
               // stream so their resident warps run beside k_keys instead of before it
    EF_CUDA(cudaEventRecord(ctx->ev_w0, st));
    EF_CUDA(cudaStreamWaitEvent(ctx->st_wide, ctx->ev_w0, 0));
    if ((rc = launch_wide(ctx, ctx->st_wide, V))) return rc;
    EF_CUDA(cudaEventRecord(ctx->ev_w1, ctx->st_wide));
  } else if (V.wide_min) {
    if ((rc = launch_wide(ctx, st, V))) return rc;
  }
  if (V.n < ctx->quad_max) {
    const uint32_t gq = std::max<uint32_t>(1, (V.n + 31) / 32);
    ++ctx->kcount, k_keys_quad<128><<<gq, 128, 0, st>>>(V);
  } else {
    const uint32_t gd = std::max<uint32_t>(1, std::min<uint32_t>((V.n + kHashThreads - 1) / kHashThreads, ctx->n_sm * 16));
    ++ctx->kcount, k_keys<kHashThreads><<<gd, kHashThreads, 0, st>>>(V);
  }
  EF_CUDA(cudaGetLastError());
  if (wide) EF_CUDA(cudaStreamWaitEvent(st, ctx->ev_w1, 0));
  return EF_OK;
}
static int ensure_chunk(ef_ctx* ctx, Scratch& sc, cudaStream_t st, uint32_t items, uint32_t S, uint32_t Rs, uint32_t* chunk,
                        bool lean = false);
// chunk candidates by job count, largest first (counting sort: k_count_*)
static int order_by_count(ef_ctx* ctx, Scratch& sc, cudaStream_t st, uint32_t n, uint32_t S) {
  if (!n) return EF_OK;
  EF_CUDA(cudaMemsetAsync(sc.cbins.p, 0, 4ull * (S + 1), st));
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, ctx->n_sm * 8));
  ++ctx->kcount, k_count_hist<<<grid, 256, 0, st>>>(sc.dcount.p, n, S, sc.cbins.p);
  ++ctx->kcount, k_count_scan<1024><<<1, 1024, 0, st>>>(sc.cbins.p, S + 1);
  ++ctx->kcount, k_count_scatter<<<grid, 256, 0, st>>>(sc.dcount.p, n, S, sc.cbins.p, sc.dorder.p);
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}
static VArgs chunk_args(ef_ctx* ctx, Scratch& sc, uint32_t S, uint32_t Rs, bool lean = false);
static int hash_records_full(ef_ctx* ctx, Scratch& sc, cudaStream_t st, const unsigned long long* d_rec, uint32_t n,
                             uint64_t* d_hash_out, uint32_t max_n = 0, uint32_t max_refs = 0) {
  if (!n) return EF_OK;
  if (!max_n) {  // sizes unknown on the host: read them from the records
    EF_CUDA(sc.recmax.reserve(2, st));
    EF_CUDA(cudaMemsetAsync(sc.recmax.p, 0, 8, st));
    ++ctx->kcount, k_rec_max<<<std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, ctx->n_sm)), 256, 0, st>>>(d_rec, n,
                                                                                                   sc.recmax.p);
    EF_CUDA(cudaGetLastError());
    uint32_t mx[2] = {0, 0};
    EF_CUDA(cudaMemcpyAsync(mx, sc.recmax.p, 8, cudaMemcpyDeviceToHost, st));
    EF_CUDA(cudaStreamSynchronize(st));
    max_n = mx[0];
    max_refs = mx[1];
  }
  const uint32_t S = (std::max<uint32_t>(max_n, 1) + 2 + 3) & ~3u;
  const uint32_t Rs = max_refs + 4;
  uint32_t chunk = 0;
  int rc = ensure_chunk(ctx, sc, st, n, S, Rs, &chunk);
  if (rc) return rc;
  VArgs V = chunk_args(ctx, sc, S, Rs);
  V.parent_addr = d_rec;
  V.full = 1;
  V.hash_out = d_hash_out;
  for (uint32_t c0 = 0; c0 < n; c0 += chunk) {
    V.c0 = c0;
    V.n = std::min(chunk, n - c0);
    const uint32_t gd = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 127) / 128, ctx->n_sm * 16));
    ++ctx->kcount, k_full_jobs<256><<<std::max<uint32_t>(1, std::min<uint32_t>(V.n, ctx->n_sm * 8)), 256, 0, st>>>(V);
    EF_CUDA(cudaGetLastError());
    if ((rc = order_by_count(ctx, sc, st, V.n, S))) return rc;
    if ((rc = launch_keys(ctx, st, V))) return rc;
    if ((rc = sort_fresh_keys(ctx, sc, st, V))) return rc;
    ++ctx->kcount, k_digest<kHashThreads><<<gd, kHashThreads, 0, st>>>(V);
    ++ctx->kcount, k_full_store<<<std::max<uint32_t>(1, std::min<uint32_t>(V.n, ctx->n_sm * 8)), 128, 0, st>>>(V);
    EF_CUDA(cudaGetLastError());
  }
  return EF_OK;
}

int ef_records_write(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host, uint64_t stride,
                     uint64_t bytes) {
  EF_REQUIRE(bytes <= ctx->geo.bytes, "ef_records_write: record too large");
  EF_REQUIRE(stride % 16 == 0 && bytes % 16 == 0, "ef_records_write: stride/bytes must be multiples of 16");
  if (!n) return EF_OK;
  // one bulk host->device copy into a staging area, then a device-side scatter into the slots
  EF_CUDA(ctx->d_stage.reserve((uint64_t)n * stride, ctx->st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_stage.p, host, (uint64_t)n * stride, cudaMemcpyHostToDevice, ctx->st));
  std::vector<unsigned long long> src(n), dst(n);
  for (uint32_t i = 0; i < n; ++i) {
    EF_REQUIRE(slots[i] < ctx->n_slots, "ef_records_write: bad slot");
    src[i] = (unsigned long long)(ctx->d_stage.p + (uint64_t)i * stride);
    dst[i] = (unsigned long long)slot_addr(ctx, slots[i]);
  }
  int rc;
  if ((rc = upload(ctx, ctx->d_addr_a, src)) || (rc = upload(ctx, ctx->d_addr_b, dst))) return rc;
  ++ctx->kcount, k_copy_records<<<std::min<uint32_t>(n, ctx->n_sm * 8), 256, 0, ctx->st>>>(ctx->d_addr_a.p, ctx->d_addr_b.p, n,
                                                                            (uint32_t)bytes);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

void* ef_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}

void ef_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

static int stage_addrs(ef_ctx* ctx, DevBuf<unsigned long long>& buf, const uint32_t* slots, uint32_t n) {
  std::vector<unsigned long long> a(n);
  for (uint32_t i = 0; i < n; ++i) {
    EF_REQUIRE(slots[i] < ctx->n_slots, "bad record slot");
    a[i] = (unsigned long long)slot_addr(ctx, slots[i]);
  }
  return upload(ctx, buf, a);
}

int ef_hash_records(ef_ctx* ctx, const uint32_t* slots, uint32_t n, uint64_t* hashes) {
  EF_REQUIRE(!ctx->dirty, "tables not committed (call ef_tables_commit)");
  if (n == 0) return EF_OK;
  int rc = stage_addrs(ctx, ctx->d_addr_a, slots, n);
  if (rc) return rc;
  EF_CUDA(ctx->d_hash_out.reserve(n, ctx->st));
  if ((rc = hash_records_full(ctx, ctx->sc[0], ctx->st, ctx->d_addr_a.p, n, ctx->d_hash_out.p))) return rc;
  EF_CUDA(cudaMemcpyAsync(hashes, ctx->d_hash_out.p, n * 8, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_price_records(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const ef_price_params* pp, ef_cand_result* out) {
  EF_REQUIRE(!ctx->dirty, "tables not committed (call ef_tables_commit)");
  if (n == 0) return EF_OK;
  int rc = stage_addrs(ctx, ctx->d_addr_a, slots, n);
  if (rc) return rc;
  EF_CUDA(ctx->d_res_aux.reserve(n, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_res_aux.p, 0, n * sizeof(ef_cand_result), ctx->st));
  PriceArgs Pa{};
  Pa.g = ctx->geo;
  Pa.T = make_tables(ctx);
  Pa.pp = *pp;
  Pa.n = n;
  Pa.rec = ctx->d_addr_a.p;
  Pa.res = ctx->d_res_aux.p;
  ++ctx->kcount, k_price<<<(n + kPriceThreads - 1) / kPriceThreads, kPriceThreads, 0, ctx->st>>>(Pa);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaMemcpyAsync(out, ctx->d_res_aux.p, n * sizeof(ef_cand_result), cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

// ---------------------------------------------------------------------------------------------
// visited set
// ---------------------------------------------------------------------------------------------

static constexpr uint64_t kVisMaxSlots = 1ull << 31;  // 16 GiB of keys; the mask is 32-bit

int ef_visited_reset(ef_ctx* ctx, uint64_t capacity) {
  EF_REQUIRE(capacity <= kVisMaxSlots, "ef_visited_reset: capacity above 2^31 slots");
  uint32_t cap = pow2_at_least(std::max<uint64_t>(capacity, 1024));
  if (!ctx->h_vis) EF_CUDA(cudaMallocHost(&ctx->h_vis, 16));
  EF_CUDA(ctx->d_vis.reserve(cap, ctx->st));
  EF_CUDA(ctx->d_vis_count.reserve(1, ctx->st));
  EF_CUDA(ctx->d_vis_err.reserve(1, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_vis.p, 0, (size_t)cap * 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_vis_count.p, 0, 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_vis_err.p, 0, 4, ctx->st));
  ctx->vis_mask = cap - 1;
  ctx->vis_bound = 0;
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

// after a synchronised insert: exact count, and a full table is an error (never with vis_reserve)
static int vis_settle(ef_ctx* ctx) {
  EF_CUDA(cudaMemcpyAsync(ctx->h_vis, ctx->d_vis_count.p, 8, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaMemcpyAsync(ctx->h_vis + 1, ctx->d_vis_err.p, 4, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  ctx->vis_bound = ctx->h_vis[0];
  EF_REQUIRE(!((uint32_t)ctx->h_vis[1] & 8u), "visited set full");
  return EF_OK;
}

// Room for `more` insertions at a load factor of at most 1/2: the table doubles (or more) by
// rehashing every stored key on the device.  Between synchronised inserts vis_bound is an upper
// bound, so this costs a host round trip only when the bound says the table may be filling up.
static int vis_reserve(ef_ctx* ctx, uint64_t more) {
  const uint64_t cap = (uint64_t)ctx->vis_mask + 1;
  if (2 * (ctx->vis_bound + more) <= cap) return EF_OK;
  int rc = vis_settle(ctx);
  if (rc) return rc;
  const uint64_t need = ctx->vis_bound + more;
  if (2 * need <= cap) return EF_OK;
  uint64_t ncap = cap;
  while (2 * need > ncap) ncap *= 2;
  EF_REQUIRE(ncap <= kVisMaxSlots, "visited set above 2^30 hashes");
  unsigned long long* q = nullptr;
  EF_CUDA(cudaMalloc(&q, ncap * 8));
  EF_CUDA(cudaMemsetAsync(q, 0, ncap * 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_vis_count.p, 0, 8, ctx->st));
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((cap + 255) / 256, ctx->n_sm * 16ull));
  ++ctx->kcount, k_visited_rehash<<<grid, 256, 0, ctx->st>>>(ctx->d_vis.p, cap, q, (uint32_t)(ncap - 1), ctx->d_vis_count.p,
                                              ctx->d_vis_err.p);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  cudaFree(ctx->d_vis.p);
  ctx->d_vis.p = q;
  ctx->d_vis.cap = ncap;
  ctx->vis_mask = (uint32_t)(ncap - 1);
  return vis_settle(ctx);
}

int ef_visited_insert(ef_ctx* ctx, const uint64_t* hashes, uint32_t n) {
  EF_REQUIRE(ctx->vis_mask, "visited set not initialised");
  if (!n) return EF_OK;
  int rc = vis_reserve(ctx, n);
  if (rc) return rc;
  EF_CUDA(ctx->d_hash_out.reserve(n, ctx->st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_hash_out.p, hashes, n * 8, cudaMemcpyHostToDevice, ctx->st));
  ++ctx->kcount, k_visited_put<<<(n + 255) / 256, 256, 0, ctx->st>>>(ctx->d_vis.p, ctx->vis_mask, ctx->d_vis_count.p,
                                                       ctx->d_hash_out.p, n, ctx->d_vis_err.p);
  EF_CUDA(cudaGetLastError());
  return vis_settle(ctx);
}

int ef_visited_capacity(ef_ctx* ctx, uint64_t* capacity) {
  EF_REQUIRE(ctx->vis_mask && capacity, "visited set not initialised");
  *capacity = (uint64_t)ctx->vis_mask + 1;
  return EF_OK;
}

int ef_visited_count(ef_ctx* ctx, uint64_t* count) {
  EF_REQUIRE(ctx->vis_mask, "visited set not initialised");
  EF_CUDA(cudaMemcpyAsync(count, ctx->d_vis_count.p, 8, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

// ---------------------------------------------------------------------------------------------
// the frontier step
// ---------------------------------------------------------------------------------------------

// words per parent of k_match's tables (ef_kernels.cuh) plus k_reach's rows (ef_step.cuh)
static uint64_t pstride_of(const Geo& g) { return 10ull * g.cap_nodes + 1 + 2ull * g.cap_refs + kReachSlots * kReachWords; }

static int ensure_parent_buffers(ef_ctx* ctx, uint32_t n_parents) {
  const Geo& g = ctx->geo;
  if (ctx->site_cap == 0) ctx->site_cap = std::max<uint32_t>(4 * g.cap_nodes, 256);
  const uint64_t pstride = pstride_of(g);
  EF_CUDA(ctx->d_parent_addr.reserve(n_parents, ctx->st));
  EF_CUDA(ctx->d_pscratch.reserve(pstride * n_parents, ctx->st));
  EF_CUDA(ctx->d_sites.reserve((uint64_t)ctx->site_cap * n_parents, ctx->st));
  EF_CUDA(ctx->d_site_count.reserve(n_parents, ctx->st));
  EF_CUDA(ctx->d_cand_off.reserve(n_parents + 1, ctx->st));
  EF_CUDA(ctx->d_scalars.reserve(16, ctx->st));
  return EF_OK;
}

// candidate-level buffers of a step
static int ensure_step_cand(ef_ctx* ctx, uint32_t total, uint32_t S) {
  const uint64_t tcap = pow2_at_least(2ull * std::max<uint32_t>(total, 1024));
  EF_CUDA(ctx->d_res.reserve(std::max<uint32_t>(total, 1), ctx->st));
  EF_CUDA(ctx->d_plan.reserve(std::max<uint32_t>(total, 1), ctx->st));
  EF_CUDA(ctx->d_plist.reserve(std::max<uint32_t>(total, 1), ctx->st));
  EF_CUDA(ctx->d_alg8.reserve((uint64_t)std::max<uint32_t>(total, 1) * S, ctx->st));
  EF_CUDA(ctx->d_step_key.reserve(2 * tcap, ctx->st));  // step table + per-parent table
  EF_CUDA(ctx->d_step_seq.reserve(2 * tcap, ctx->st));
  EF_CUDA(ctx->d_req_sig.reserve(ctx->req_cap, ctx->st));
  EF_CUDA(ctx->d_req_dv.reserve(4 * ctx->req_cap, ctx->st));
  return EF_OK;
}

// per-chunk hashing scratch for rows of S node slots and Rs ref slots: bounded (half the free
// HBM, at most 96 GiB) so graphs of any size stream through; a chunk that holds the whole step
// keeps every candidate in flight (large graphs have few parents: chunking starves the GPU)
// lean (step rows beyond kFastRows with k_dirty_big and the merged stream): no didx / sort
// value rows, and the merged key stream reuses the jobs row (dead after the node keys), so a
// chunk holds 1.4x the candidates (DAG-20k: 98 -> 70 bytes per candidate slot)
static bool lean_rows(ef_ctx* ctx, uint32_t S) { return S > kFastRows && ctx->big_merge && ctx->dirty_big; }

static int ensure_chunk(ef_ctx* ctx, Scratch& sc, cudaStream_t st, uint32_t items, uint32_t S, uint32_t Rs, uint32_t* chunk,
                        bool lean) {
  const bool big = S > kFastRows && ctx->big_merge && !lean;  // + the merged key stream
  const uint64_t per = (uint64_t)S * (4 + sizeof(Job) + 16 + 16 + 8 + 8 + (S > kFastRows ? 2 : 0) +
                                      (lean ? 0 : 4 + 4 + 4) + (big ? 16 : 0)) +
                       4ull * Rs + 4ull * (S + 31) / 32 + 32;
  if (!ctx->chunk_mib) {  // a share of the HBM free when the first chunk is sized (EF_CHUNK_MIB overrides)
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    ctx->chunk_mib = std::min<uint64_t>(144ull << 10, std::max<uint64_t>(1024, (uint64_t)(0.8 * (double)fr) >> 20));
  }
  uint64_t ch = std::max<uint64_t>(256, (ctx->chunk_mib << 20) / per);
  ch = std::min<uint64_t>(ch, (uint64_t)INT32_MAX / S);
  // equal chunks: a full chunk and a small remainder would run the remainder's kernels at a
  // fraction of the GPU for a whole per-candidate latency (DAG-20k, 9 parents: 84k + 7.5k)
  const uint64_t nch = (std::max<uint32_t>(items, 1) + ch - 1) / ch;
  ch = (std::max<uint32_t>(items, 1) + nch - 1) / nch;
  *chunk = (uint32_t)ch;
  if (!lean) {
    EF_CUDA(sc.didx.reserve(ch * S, st));
    EF_CUDA(sc.sval2.reserve(ch * S, st));
  }
  if (S > kFastRows) EF_CUDA(sc.jlvl.reserve(ch * S, st));
  if (big) EF_CUDA(sc.merged.reserve(ch * S * 2, st));
  EF_CUDA(sc.jv.reserve(ch * S, st));
  EF_CUDA(sc.jobs.reserve(ch * S, st));
  EF_CUDA(sc.refsrc.reserve(ch * Rs, st));
  EF_CUDA(sc.fresh.reserve(2 * ch * S, st));
  EF_CUDA(sc.fresh2.reserve(2 * ch * S, st));
  EF_CUDA(sc.rmask.reserve(ch * ((S + 31) / 32), st));
  EF_CUDA(sc.skey.reserve(ch * S, st));
  EF_CUDA(sc.skey2.reserve(ch * S, st));
  EF_CUDA(sc.dcount.reserve(ch, st));
  EF_CUDA(sc.dorder.reserve(ch, st));
  EF_CUDA(sc.seg_b.reserve(ch, st));
  EF_CUDA(sc.seg_e.reserve(ch, st));
  EF_CUDA(sc.cbins.reserve(S + 2, st));
  return EF_OK;
}

static VArgs chunk_args(ef_ctx* ctx, Scratch& sc, uint32_t S, uint32_t Rs, bool lean) {
  VArgs V{};
  V.g = ctx->geo;
  V.T = make_tables(ctx);
  V.plan = ctx->d_plan.p;
  V.res = ctx->d_res.p;
  V.S = S;
  V.Rs = Rs;
  V.didx = lean ? nullptr : sc.didx.p;
  V.jobs = sc.jobs.p;
  V.refsrc = sc.refsrc.p;
  V.fresh = sc.fresh.p;
  V.dcount = sc.dcount.p;
  V.order = sc.dorder.p;
  V.skey = sc.skey.p;
  V.skey_sorted = sc.skey2.p;
  V.sval_sorted = lean ? nullptr : sc.sval2.p;  // full mode only
  V.seg_begin = sc.seg_b.p;
  V.seg_end = sc.seg_e.p;
  V.W = (S + 31) / 32;
  V.rmask = sc.rmask.p;
  V.fresh_sorted = sc.fresh2.p;
  V.input_words = reinterpret_cast<const uint64_t*>(ctx->d_input_text.p);
  V.err = ctx->d_scalars.p + 1;
  V.jv = sc.jv.p;
  V.jlvl = nullptr;
  V.wide_min = 0;
  V.kstream = lean ? reinterpret_cast<uint64_t*>(sc.jobs.p)  // the jobs rows are dead by the merge
                   : (S > kFastRows && ctx->big_merge) ? sc.merged.p : sc.fresh2.p;
  return V;
}

// every candidate's fresh keys in ascending order: warp bitonic sort in shared memory for
// rows up to 1024 keys, k_sortbig (a CTA per candidate) beyond
static int sort_fresh_keys(ef_ctx* ctx, Scratch& sc, cudaStream_t st, const VArgs& V) {
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 7) / 8, ctx->n_sm * 32));
  if (V.S <= 128) {
    ++ctx->kcount, k_sortkeys<128, 8><<<grid, 256, 0, st>>>(V);
  } else if (V.S <= 256) {
    ++ctx->kcount, k_sortkeys<256, 8><<<grid, 256, 0, st>>>(V);
  } else if (V.S <= 512) {
    ++ctx->kcount, k_sortkeys<512, 8><<<grid, 256, 0, st>>>(V);
  } else if (V.S <= 1024) {
    ++ctx->kcount, k_sortkeys<1024, 4><<<std::max<uint32_t>(1, std::min<uint32_t>((V.n + 3) / 4, ctx->n_sm * 32)), 128, 0, st>>>(V);
  } else {  // a CTA per candidate: shared-memory bucket sort up to 8192 keys, runs merged beyond
    uint32_t R = 1024;
    while (R < V.S && R < 8192u) R <<= 1;
    const size_t smem = 12ull * R;  // R sort words + R bucket counters
    EF_CUDA(cudaFuncSetAttribute(k_sortbig<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++ctx->kcount, k_sortbig<512><<<std::max<uint32_t>(1, std::min<uint32_t>(V.n, ctx->n_sm * 4)), 512, smem, st>>>(V, R);
  }
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}


// ---- step phases --------------------------------------------------------------------------

static int launch_spec_price(ef_ctx* ctx, uint32_t total);

// 1-3: match, plans, per chunk dirty walk / node keys / key sort / graph digest.  Leaves the
// candidates' hashes in d_res; no synchronisation at the end.
static int step_hash(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                     uint32_t n_rules, uint32_t* n_total) {
  Scratch& sc = ctx->sc[0];
  for (int attempt = 0; attempt < 8; ++attempt) {
    int rc = ensure_parent_buffers(ctx, std::max<uint32_t>(n_parents, 1));
    if (rc) return rc;
    const Geo& g = ctx->geo;
    if ((rc = stage_addrs(ctx, ctx->d_parent_addr, parent_slots, n_parents))) return rc;
    EF_CUDA(cudaMemsetAsync(ctx->d_scalars.p, 0, 16 * 4, ctx->st));
    EF_CUDA(ctx->d_stats.reserve(8, ctx->st));
    EF_CUDA(cudaMemsetAsync(ctx->d_stats.p, 0, 8 * 8, ctx->st));
    StepArgs A{};
    A.g = g;
    A.T = make_tables(ctx);
    A.parent_addr = ctx->d_parent_addr.p;
    A.n_parents = n_parents;
    A.pscratch = ctx->d_pscratch.p;
    A.pstride = pstride_of(g);
    for (uint32_t i = 0; i < n_rules; ++i) A.rules[i] = rules[i];
    A.n_rules = (int32_t)n_rules;
    A.sites = ctx->d_sites.p;
    A.site_cap = ctx->site_cap;
    A.site_count = ctx->d_site_count.p;
    A.cand_off = ctx->d_cand_off.p;
    A.total = ctx->d_scalars.p + 0;
    A.err = ctx->d_scalars.p + 1;
    A.n_req_sig = ctx->d_scalars.p + 2;
    A.n_req_dv = ctx->d_scalars.p + 3;
    A.cand_cap = 0xffffffffu;

    // 1) match every rule at every node of every parent; candidate offsets; parent sizes
    cudaEventRecord(ctx->ev[0], ctx->st);
    if (n_parents) {
      ++ctx->kcount, k_match<kMatchThreads><<<std::min<uint32_t>(n_parents, ctx->n_sm * 8), kMatchThreads, 0, ctx->st>>>(A);
      EF_CUDA(cudaGetLastError());
    }
    ++ctx->kcount, k_offsets<1024><<<1, 1024, 0, ctx->st>>>(A);
    EF_CUDA(cudaGetLastError());
    cudaEventRecord(ctx->ev[1], ctx->st);
    EF_CUDA(cudaMemcpyAsync(ctx->h_scalars, ctx->d_scalars.p, 16 * 4, cudaMemcpyDeviceToHost, ctx->st));
    EF_CUDA(cudaStreamSynchronize(ctx->st));
    if (ctx->h_scalars[1] & 1u) {  // site buffer too small
      ctx->site_cap *= 4;
      continue;
    }
    const uint32_t total = ctx->h_scalars[0];
    const uint32_t S = (std::max<uint32_t>(ctx->h_scalars[5], 1) + 2 + 3) & ~3u;
    const uint32_t Rs = ctx->h_scalars[6] + 4;
    uint32_t chunk = 0;
    const bool lean = lean_rows(ctx, S);
    if ((rc = ensure_step_cand(ctx, total, S)) || (rc = ensure_chunk(ctx, sc, ctx->st, total, S, Rs, &chunk, lean)))
      return rc;
    ctx->step_S = S;
    ctx->step_Rs = Rs;
    ctx->step_n_parents = n_parents;
    A.res = ctx->d_res.p;
    A.req_sig = ctx->d_req_sig.p;
    A.req_sig_cap = ctx->req_cap;
    A.req_dv = ctx->d_req_dv.p;
    A.req_dv_cap = ctx->req_cap;

    // 2) rewrite plans; 3) per chunk: dirty walk, node keys, key sort, graph digest
    const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
    if (total && S <= kFastRows) {  // per-parent reach rows for k_dirty_warp
      const uint32_t rmax = ctx->h_scalars[6];
      const size_t smem = 2ull * 4 * (256 + 260 + ((rmax + 3) & ~3u) + kReachSlots * kReachWords);
      EF_CUDA(cudaFuncSetAttribute(k_reach, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ++ctx->kcount, k_reach<<<std::max<uint32_t>(1, (n_parents + 1) / 2), 64, smem, ctx->st>>>(A, rmax);
      EF_CUDA(cudaGetLastError());
    }
    if (total) {
      ++ctx->kcount, k_plan<<<grid_t, 256, 0, ctx->st>>>(A, ctx->d_plan.p);
      EF_CUDA(cudaGetLastError());
    }
    ctx->spec_live = false;
    ctx->spec_mode = !ctx->spec_pp ? 0
                     : ctx->spec_price > 0 ? ctx->spec_price
                     : total < ctx->spec_min_cands ? 0
                     : S > 4 * ctx->spec_min_rows ? 4  // DAG-20k per step: 183.5 (node keys), 183.5 (digest), 179.9 ms (key sort)
                     : S > ctx->spec_min_rows ? 2
                     : (S > kFastRows && total <= ctx->spec_max_cands) ? 1 : 0;
    if (ctx->spec_mode == 2 && (rc = launch_spec_price(ctx, total))) return rc;
    cudaEventRecord(ctx->ev[2], ctx->st);
    VArgs V = chunk_args(ctx, sc, S, Rs, lean);
    V.parent_addr = A.parent_addr;
    V.stats = ctx->d_stats.p;
    V.pscratch = A.pscratch;
    V.pstride = A.pstride;
    V.Os = ctx->h_scalars[8] + 2;
    EF_CUDA(sc.outsrc.reserve((uint64_t)chunk * V.Os, ctx->st));
    V.outsrc = sc.outsrc.p;
    // graphs with many outputs (large rows): the digest's prefix built by k_prefix
    const bool pfx = S > kFastRows && ctx->big_merge && !ctx->fuse_merge && ctx->digest_pf && ctx->h_scalars[8] >= kPrefixMinOuts;
    V.pfx = nullptr;
    if (pfx) {
      V.pfx_stride = (uint32_t)(((uint64_t)ctx->input_text.size() + 18ull * ctx->h_scalars[8] + 7) / 8 + 2) & ~1u;
      EF_CUDA(sc.pfx.reserve((uint64_t)chunk * V.pfx_stride, ctx->st));
      V.pfx = sc.pfx.p;
      if (ctx->pfx_share && ctx->dirty_big) {  // (k_dirty_big finds the first changed output)  // the parents' prefix chains, once per step
        const uint32_t li = (uint32_t)ctx->input_text.size();
        V.pfx_nst = ((li + 18u * ctx->h_scalars[8]) >> 7) + 1;
        EF_CUDA(sc.pfx_state.reserve((uint64_t)n_parents * V.pfx_nst * 8, ctx->st));
        EF_CUDA(sc.pfx_first.reserve(chunk, ctx->st));
        V.pfx_state = sc.pfx_state.p;
        V.pfx_first = sc.pfx_first.p;
        // on the wide-key stream: a one-warp-per-parent chain that runs beside the dirty walk
        EF_CUDA(cudaEventRecord(ctx->ev_pf0, ctx->st));
        EF_CUDA(cudaStreamWaitEvent(ctx->st_wide, ctx->ev_pf0, 0));
        ++ctx->kcount, k_pfx_chain<<<std::max<uint32_t>(1, n_parents), 32, 0, ctx->st_wide>>>(
            A.parent_addr, ctx->geo, n_parents, reinterpret_cast<const uint64_t*>(ctx->d_input_text.p), li, V.pfx_nst,
            sc.pfx_state.p);
        EF_CUDA(cudaGetLastError());
        EF_CUDA(cudaEventRecord(ctx->ev_pf1, ctx->st_wide));
      }
    }
    // k_merge_scatter: the parents' top-bit directories, once per step
    const bool ms16 = S < 65536u;  // positions as 16-bit words
    const bool ms_sort = ms16 && S > ctx->ms_sort_min_rows;  // the merge sorts the fresh keys too (k_sortkeys below)
    const size_t ms_smem =
        4ull * (2ull * V.W + 3) + (ms_sort ? 4ull * (1u << kDirBits) + 6ull * kMsDcap : (ms16 ? 2ull : 4ull) * S);
    V.pdir = nullptr;
    if (total && S > kFastRows && S > ctx->ms_min_rows && ctx->big_merge && !ctx->fuse_merge && ctx->merge_scatter &&
        ms_smem <= 200ull * 1024) {
      EF_CUDA(sc.pdir.reserve((uint64_t)kDirN * n_parents, ctx->st));
      V.pdir = sc.pdir.p;
      ++ctx->kcount, k_merge_dir<<<std::max<uint32_t>(1, std::min<uint32_t>(n_parents, ctx->n_sm * 8)), 256, 0, ctx->st>>>(
          A.parent_addr, ctx->geo, n_parents, sc.pdir.p);
      EF_CUDA(cudaGetLastError());
    }
    ctx->n_chunks = 0;
    for (uint32_t c0 = 0; c0 < total; c0 += chunk) {
      V.c0 = c0;
      V.n = std::min(chunk, total - c0);
      const uint32_t gd = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 127) / 128, ctx->n_sm * 16));
      while (ctx->ev_chunk.size() < 5ull * (ctx->n_chunks + 1)) {
        cudaEvent_t e;
        EF_CUDA(cudaEventCreate(&e));
        ctx->ev_chunk.push_back(e);
      }
      cudaEvent_t* ce = ctx->ev_chunk.data() + 5 * ctx->n_chunks++;
      cudaEventRecord(ce[0], ctx->st);
      // rows <= kFastRows: slot walk, warp merge, streaming digest (the 32-word slot walk and
      // the shared-memory merge also handle rows <= 1024, but measured slower than the general
      // kernels there: NasNet-A 15.1 vs 13.8 ms per 1024-parent step)
      V.slots = S <= kFastRows;
      const bool big_walk = !V.slots && ctx->dirty_big && ctx->big_merge;  // (k_digest reads didx rows)
      V.osrc = V.slots || big_walk;
      V.wide_min = (V.slots || S < ctx->wide_min) ? 0u : ctx->wide_min;  // no candidate can reach it otherwise
      V.jlvl = V.wide_min ? sc.jlvl.p : nullptr;
      if (V.slots) {
        const uint32_t gw = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 3) / 4, ctx->n_sm * 16));
        ++ctx->kcount, k_dirty_warp<4><<<gw, 128, 0, ctx->st>>>(V);
      } else if (big_walk) {
        const size_t smem = 4ull * 4 * (3ull * V.W + 1);
        EF_CUDA(cudaFuncSetAttribute(k_dirty_big<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const uint32_t gw = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 3) / 4, ctx->n_sm * 32));
        ++ctx->kcount, k_dirty_big<4><<<gw, 128, smem, ctx->st>>>(V);
      } else {
        ++ctx->kcount, k_dirty<<<gd, 128, 0, ctx->st>>>(V);
      }
      EF_CUDA(cudaGetLastError());
      if ((rc = order_by_count(ctx, sc, ctx->st, V.n, S))) return rc;
      if (ctx->spec_mode == 3 && (rc = launch_spec_price(ctx, total))) return rc;  // beside the node keys
      cudaEventRecord(ce[1], ctx->st);
      if ((rc = launch_keys(ctx, ctx->st, V))) return rc;
      cudaEventRecord(ce[2], ctx->st);
      if (S <= kFastRows) {  // slot-space walk, warp merge into a contiguous key stream, streaming digest
        uint32_t rows = 32;
        while (rows < S) rows <<= 1;
        const int warps = rows <= 256 ? 4 : 2;
        const size_t smem = (size_t)warps * rows * 32;
        const uint32_t gm = std::max<uint32_t>(1, std::min<uint32_t>((V.n + warps - 1) / warps, ctx->n_sm * 32));
        if (warps == 4) {
          EF_CUDA(cudaFuncSetAttribute(k_merge<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          ++ctx->kcount, k_merge<8, 4><<<gm, 128, smem, ctx->st>>>(V, rows);
        } else {
          EF_CUDA(cudaFuncSetAttribute(k_merge<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          ++ctx->kcount, k_merge<8, 2><<<gm, 64, smem, ctx->st>>>(V, rows);
        }
        EF_CUDA(cudaGetLastError());
        cudaEventRecord(ce[3], ctx->st);
        ++ctx->kcount, k_digest_pm<kHashThreads, false, EF_DIGEST_MINB><<<gd, kHashThreads, 0, ctx->st>>>(V);
      } else {
        if (ctx->spec_mode == 4 && (rc = launch_spec_price(ctx, total))) return rc;  // beside the key sort
        if (!(V.pdir && ms_sort) && (rc = sort_fresh_keys(ctx, sc, ctx->st, V))) return rc;  // (k_merge_scatter sorts)
        if (ctx->spec_mode && (rc = launch_spec_price(ctx, total))) return rc;  // under the digest
        if (ctx->big_merge && ctx->fuse_merge) {  // the digest merges the two sorted streams itself
          cudaEventRecord(ce[3], ctx->st);
          ++ctx->kcount, k_digest_mg<kHashThreads, 2><<<gd, kHashThreads, 0, ctx->st>>>(V);
        } else if (ctx->big_merge) {  // merged key stream, then the streaming digest
          if (V.pdir) {
            const uint32_t per_sm = std::max<uint32_t>(1, std::min<uint32_t>(8, (uint32_t)((220ull * 1024) / (ms_smem + 2048))));
            const uint32_t gm = std::max<uint32_t>(1, std::min<uint32_t>(V.n, ctx->n_sm * per_sm));
            if (ms_sort) {
              EF_CUDA(cudaFuncSetAttribute(k_merge_scatter<256, uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
              ++ctx->kcount, k_merge_scatter<256, uint16_t, true><<<gm, 256, ms_smem, ctx->st>>>(V);
            } else if (ms16) {
              EF_CUDA(cudaFuncSetAttribute(k_merge_scatter<256, uint16_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
              ++ctx->kcount, k_merge_scatter<256, uint16_t, false><<<gm, 256, ms_smem, ctx->st>>>(V);
            } else {
              EF_CUDA(cudaFuncSetAttribute(k_merge_scatter<256, uint32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ms_smem));
              ++ctx->kcount, k_merge_scatter<256, uint32_t, false><<<gm, 256, ms_smem, ctx->st>>>(V);
            }
          } else {
            const size_t smem = 4ull * (2560 + 4 * (2 * V.W + 2));  // per warp: the output stage, kept counts, removed mask
            EF_CUDA(cudaFuncSetAttribute(k_merge_big<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const uint32_t gm = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 3) / 4, ctx->n_sm * 16));
            ++ctx->kcount, k_merge_big<4><<<gm, 128, smem, ctx->st>>>(V);
          }
          EF_CUDA(cudaGetLastError());
          if (V.pfx) {
            if (V.pfx_state && c0 == 0) EF_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_pf1, 0));  // the parents' chains
            const uint32_t gpx = std::max<uint32_t>(1, std::min<uint32_t>((V.n + 3) / 4, ctx->n_sm * 16));
            ++ctx->kcount, k_prefix<<<gpx, 128, 0, ctx->st>>>(V);
          }
          cudaEventRecord(ce[3], ctx->st);
          if (ctx->digest_pf) ++ctx->kcount, k_digest_pm<kHashThreads, true, EF_DIGEST_PF_MINB><<<gd, kHashThreads, 0, ctx->st>>>(V);
          else ++ctx->kcount, k_digest_pm<kHashThreads, false, EF_DIGEST_MINB><<<gd, kHashThreads, 0, ctx->st>>>(V);
        } else {
          cudaEventRecord(ce[3], ctx->st);
          ++ctx->kcount, k_digest<kHashThreads><<<gd, kHashThreads, 0, ctx->st>>>(V);
        }
      }
      EF_CUDA(cudaGetLastError());
      cudaEventRecord(ce[4], ctx->st);
    }
    cudaEventRecord(ctx->ev[3], ctx->st);
    ctx->last_total = total;
    ctx->last_step = A;
    *n_total = total;
    return EF_OK;
  }
  ctx->err = "ef_expand: buffers did not converge";
  return EF_ERR_CAPACITY;
}

static DedupArgs dedup_args(ef_ctx* ctx, const ef_price_params* pp, int insert_visited, uint32_t table_items) {
  const uint32_t tcap = pow2_at_least(2ull * std::max<uint32_t>(table_items, 1024));
  DedupArgs D{};
  D.res = ctx->d_res.p;
  D.total = ctx->d_scalars.p + 0;
  D.step_key = ctx->d_step_key.p;
  D.step_seq = ctx->d_step_seq.p;
  D.step_mask = tcap - 1;
  D.vis_key = ctx->d_vis.p;
  D.vis_mask = ctx->vis_mask;
  D.vis_count = ctx->d_vis_count.p;
  D.insert_visited = insert_visited;
  D.node_cap = pp ? pp->node_cap : 0;
  D.plist = ctx->d_plist.p;
  D.plist_n = ctx->d_scalars.p + 7;
  D.err = ctx->d_vis_err.p;
  D.per_parent = pp ? pp->per_parent : 0;
  return D;
}

// 4) dedup inside the step and against the visited set (single rank)
static int step_dedup_local(ef_ctx* ctx, const ef_price_params* pp) {
  const uint32_t total = ctx->last_total;
  DedupArgs D = dedup_args(ctx, pp, 0, total);
  const size_t tables = D.per_parent ? 2 : 1;
  EF_CUDA(cudaMemsetAsync(ctx->d_step_key.p, 0, tables * (D.step_mask + 1) * 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_step_seq.p, 0xff, tables * (D.step_mask + 1) * 4, ctx->st));
  const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
  ++ctx->kcount, k_dedup_claim<<<grid_t, 256, 0, ctx->st>>>(D);
  ++ctx->kcount, k_dedup_resolve<<<grid_t, 256, 0, ctx->st>>>(D);
  EF_CUDA(cudaGetLastError());
  cudaEventRecord(ctx->ev[4], ctx->st);
  return EF_OK;
}

// the inner search kernel over a candidate list (pl, *pn) on stream st; results into out (null:
// the step's results)
static int launch_price(ef_ctx* ctx, const ef_price_params* pp, uint32_t total, cudaStream_t st, const uint32_t* pl,
                        const uint32_t* pn, ef_cand_result* out) {
  VPriceArgs Pv{};
  Pv.pa.g = ctx->geo;
  Pv.pa.T = make_tables(ctx);
  Pv.pa.pp = *pp;
  Pv.pa.total = ctx->d_scalars.p + 0;
  Pv.pa.res = ctx->d_res.p;
  Pv.pa.step_mode = 1;
  Pv.plan = ctx->d_plan.p;
  Pv.parent_addr = ctx->d_parent_addr.p;
  Pv.pscratch = ctx->d_pscratch.p;
  Pv.pstride = pstride_of(ctx->geo);
  Pv.alg8 = ctx->d_alg8.p;
  Pv.S = ctx->step_S;
  Pv.out = out;
  const uint32_t gp = std::max<uint32_t>(1, std::min<uint32_t>((total + kPriceThreads - 1) / kPriceThreads, ctx->n_sm * (1024 / kPriceThreads)));
  const bool fast = pp->use_inner && pp->d == 1;
  const bool sm = ctx->step_S <= kFastRows;  // the sweep's algorithm row in shared memory
  Pv.algt = nullptr;
  if (!sm && ctx->step_S <= 2048) {  // the interleaved sweep rows of k_price_v, one per thread of
                                     // the grid (beyond 2k-slot rows the scratch outgrows L2: slower)
    EF_CUDA(ctx->d_algt.reserve((uint64_t)gp * kPriceThreads * ctx->step_S, st));
    Pv.algt = ctx->d_algt.p;
  }
  const size_t smem = sm ? (size_t)ctx->step_S * kPriceThreads : 0;
#define EF_PRICE(K)                                                                                        \
  do {                                                                                                     \
    if (sm) {                                                                                              \
      EF_CUDA(cudaFuncSetAttribute(k_price_v<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      ++ctx->kcount, k_price_v<K, true><<<gp, kPriceThreads, smem, st>>>(Pv, pl, pn);                             \
    } else {                                                                                               \
      ++ctx->kcount, k_price_v<K, false><<<gp, kPriceThreads, 0, st>>>(Pv, pl, pn);                                \
    }                                                                                                      \
  } while (0)
  ctx->alg_rows = fast;  // price_d1 leaves row indices (k_keep_alg reads the ids)
  const uint32_t lanes = ctx->price_lanes_env ? ctx->price_lanes : total < ctx->lanes_max_cands ? 2u : ctx->price_lanes;
  if (fast && lanes >= 2 && !out && ctx->step_S <= 2048) {  // a lane group per candidate (price_d1_lanes)
    const uint32_t PL = lanes;
    const uint32_t gl = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)(((uint64_t)total * PL + kPriceThreads - 1) / kPriceThreads),
                                                                 ctx->n_sm * 32));
    const size_t rows = (size_t)(kPriceThreads / PL) * ctx->step_S;
    const int smrow = rows <= 48 * 1024 ? 1 : 0;
    const size_t lsm = smrow ? rows : 0;
#define EF_PRICE_L(K, PLC) \
    ++ctx->kcount, k_price_lanes<K, PLC><<<gl, kPriceThreads, lsm, st>>>(Pv, pl, pn, smrow)
#define EF_PRICE_LK(K) \
    do { if (PL == 2) EF_PRICE_L(K, 2); else if (PL == 4) EF_PRICE_L(K, 4); else EF_PRICE_L(K, 8); } while (0)
    if (pp->kind == EF_C_ENERGY) EF_PRICE_LK(EF_C_ENERGY);
    else if (pp->kind == EF_C_TIME) EF_PRICE_LK(EF_C_TIME);
    else if (pp->kind == EF_C_LINEAR) EF_PRICE_LK(EF_C_LINEAR);
    else EF_PRICE_LK(EF_C_MIX + 1);
#undef EF_PRICE_LK
#undef EF_PRICE_L
    EF_CUDA(cudaGetLastError());
    return EF_OK;
  }
  if (fast && !sm && !Pv.algt)  // the global rows start at row 0 (price_d1 writes changes only)
    EF_CUDA(cudaMemsetAsync(ctx->d_alg8.p, 0, (uint64_t)std::max<uint32_t>(total, 1) * ctx->step_S, st));
  if (fast && ctx->sparse_sweep && ctx->step_n_parents) {  // the parents' movable-node bits (sparse sweeps)
    const uint32_t W = (ctx->geo.cap_nodes + 31) / 32;
    EF_CUDA(ctx->d_nsk.reserve((uint64_t)ctx->step_n_parents * W, st));
    Pv.nsk = ctx->d_nsk.p;
    Pv.nsk_W = W;
    const uint32_t gn = std::min<uint32_t>(ctx->step_n_parents, ctx->n_sm * 8);
    if (pp->kind == EF_C_ENERGY) ++ctx->kcount, k_price_nsk<EF_C_ENERGY><<<gn, 256, 0, st>>>(Pv.pa, ctx->d_parent_addr.p, ctx->d_pscratch.p, Pv.pstride, ctx->step_n_parents, W, ctx->d_nsk.p);
    else if (pp->kind == EF_C_TIME) ++ctx->kcount, k_price_nsk<EF_C_TIME><<<gn, 256, 0, st>>>(Pv.pa, ctx->d_parent_addr.p, ctx->d_pscratch.p, Pv.pstride, ctx->step_n_parents, W, ctx->d_nsk.p);
    else if (pp->kind == EF_C_LINEAR) ++ctx->kcount, k_price_nsk<EF_C_LINEAR><<<gn, 256, 0, st>>>(Pv.pa, ctx->d_parent_addr.p, ctx->d_pscratch.p, Pv.pstride, ctx->step_n_parents, W, ctx->d_nsk.p);
    else ++ctx->kcount, k_price_nsk<EF_C_MIX + 1><<<gn, 256, 0, st>>>(Pv.pa, ctx->d_parent_addr.p, ctx->d_pscratch.p, Pv.pstride, ctx->step_n_parents, W, ctx->d_nsk.p);
    EF_CUDA(cudaGetLastError());
  }
  if (fast && pp->kind == EF_C_ENERGY) EF_PRICE(EF_C_ENERGY);
  else if (fast && pp->kind == EF_C_TIME) EF_PRICE(EF_C_TIME);
  else if (fast && pp->kind == EF_C_LINEAR) EF_PRICE(EF_C_LINEAR);
  else if (fast) EF_PRICE(EF_C_MIX + 1);
  else ++ctx->kcount, k_price_v<-1, false><<<gp, kPriceThreads, 0, st>>>(Pv, pl, pn);
#undef EF_PRICE
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

// speculative pricing of every complete candidate on st_price, from where the main stream has
// got to (step_hash calls it once per step, when ctx->spec_pp is set)
static int launch_spec_price(ef_ctx* ctx, uint32_t total) {
  if (!ctx->spec_pp || !ctx->spec_mode || ctx->spec_live || !total) return EF_OK;
  EF_CUDA(ctx->d_spec.reserve(total, ctx->st));
  EF_CUDA(ctx->d_spec_list.reserve(total + 1, ctx->st));
  EF_CUDA(cudaEventRecord(ctx->ev_sp0, ctx->st));
  EF_CUDA(cudaStreamWaitEvent(ctx->st_price, ctx->ev_sp0, 0));
  uint32_t* list_n = ctx->d_spec_list.p + total;
  EF_CUDA(cudaMemsetAsync(list_n, 0, 4, ctx->st_price));
  const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
  ++ctx->kcount, k_spec_list<<<grid_t, 256, 0, ctx->st_price>>>(ctx->d_res.p, total, ctx->spec_pp->node_cap,
                                                                  ctx->d_spec_list.p, list_n, ctx->d_spec.p);
  EF_CUDA(cudaGetLastError());
  int rc = launch_price(ctx, ctx->spec_pp, total, ctx->st_price, ctx->d_spec_list.p, list_n, ctx->d_spec.p);
  if (rc) return rc;
  EF_CUDA(cudaEventRecord(ctx->ev_sp1, ctx->st_price));
  ctx->spec_live = true;
  return EF_OK;
}

// 5) inner search on every survivor (the compacted list of step 4), or, when the step priced
// speculatively, the survivors' prices taken from the speculative results
static int step_price(ef_ctx* ctx, const ef_price_params* pp) {
  const uint32_t total = ctx->last_total;
  if (ctx->spec_live) {
    ctx->spec_live = false;
    EF_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_sp1, 0));
    const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
    ++ctx->kcount, k_spec_commit<<<grid_t, 256, 0, ctx->st>>>(ctx->d_res.p, ctx->d_spec.p, total,
                                                              ctx->spec_sharded ? 0 : pp->per_parent);
    EF_CUDA(cudaGetLastError());
  } else {
    int rc = launch_price(ctx, pp, total, ctx->st, ctx->d_plist.p, ctx->d_scalars.p + 7, nullptr);
    if (rc) return rc;
  }
  cudaEventRecord(ctx->ev[5], ctx->st);
  return EF_OK;
}

// 6) the alpha-prune flags over the priced candidates (search.py:258-267), in step order
static int step_prune(ef_ctx* ctx, const ef_price_params* pp) {
  const uint32_t total = ctx->last_total;
  if (!(pp->alpha > 0.0) || !total) return EF_OK;
  constexpr int BT = 512;
  const uint32_t tiles = (total + BT - 1) / BT;
  EF_CUDA(ctx->d_tile.reserve(tiles, ctx->st));
  ++ctx->kcount, k_prune_tiles<BT><<<tiles, BT, 0, ctx->st>>>(ctx->d_res.p, total, ctx->d_tile.p);
  ++ctx->kcount, k_prune_scan<BT><<<1, BT, 0, ctx->st>>>(ctx->d_tile.p, tiles, pp->best);
  ++ctx->kcount, k_prune_flags<BT><<<tiles, BT, 0, ctx->st>>>(ctx->d_res.p, total, ctx->d_tile.p, pp->alpha);
  EF_CUDA(cudaGetLastError());
  cudaEventRecord(ctx->ev[5], ctx->st);  // the price stage includes the prune
  return EF_OK;
}

// synchronise; EF_NEED_RESOLVE when the plans asked for signatures / weight sets
static int step_sync(ef_ctx* ctx, bool timings) {
  EF_CUDA(cudaMemcpyAsync(ctx->h_scalars, ctx->d_scalars.p, 16 * 4, cudaMemcpyDeviceToHost, ctx->st));
  if (timings) EF_CUDA(cudaMemcpyAsync(ctx->last_stats, ctx->d_stats.p, 2 * 8, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));  // one round trip for the scalars and the counters
  const uint32_t err = ctx->h_scalars[1];
  ctx->last_req_sig = ctx->h_scalars[2];
  ctx->last_req_dv = ctx->h_scalars[3];
  if (timings) {  // match, plan, dirty, keys, sort, digest, dedup, price
    float ms[5];
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&ms[k], ctx->ev[k], ctx->ev[k + 1]);
    float sub[4] = {0, 0, 0, 0};
    for (uint32_t c = 0; c < ctx->n_chunks; ++c) {
      cudaEvent_t* ce = ctx->ev_chunk.data() + 5 * c;
      for (int k = 0; k < 4; ++k) {
        float x = 0;
        cudaEventElapsedTime(&x, ce[k], ce[k + 1]);
        sub[k] += x;
      }
    }
    ctx->last_ms[0] = ms[0];
    ctx->last_ms[1] = ms[1];
    for (int k = 0; k < 4; ++k) ctx->last_ms[2 + k] = sub[k];
    ctx->last_ms[6] = ms[3];
    ctx->last_ms[7] = ms[4];
    cudaEventElapsedTime(&ctx->last_ms[8], ctx->ev[0], ctx->ev[5]);  // the whole step (incl. any exchange)
    ctx->last_stats[2] = ctx->last_total;
    ctx->last_stats[3] = ctx->h_scalars[7];
    ctx->last_stats[4] = ctx->kcount - ctx->kcount_step0;
  }
  EF_REQUIRE(!(err & 4u), "candidate exceeds record capacity (raise cap_nodes/cap_refs)");
  if (err & 16u) {
    char buf[160];
    snprintf(buf, sizeof buf, "k_keys_wide: job levels out of range (chunk candidate %u: %u jobs, level %u)",
             ctx->h_scalars[10], ctx->h_scalars[11], ctx->h_scalars[12]);
    ctx->err = buf;
    return EF_ERR_INTERNAL;
  }
  if (ctx->last_req_sig || ctx->last_req_dv) return EF_NEED_RESOLVE;
  return EF_OK;
}

static int insert_firsts(ef_ctx* ctx) {
  int rc = vis_reserve(ctx, ctx->last_total);
  if (rc) return rc;
  DedupArgs D = dedup_args(ctx, nullptr, 1, ctx->last_total);
  const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((ctx->last_total + 255) / 256, ctx->n_sm * 8));
  ++ctx->kcount, k_visited_insert<<<grid_t, 256, 0, ctx->st>>>(D);
  EF_CUDA(cudaGetLastError());
  return vis_settle(ctx);
}

static int step_begin(ef_ctx* ctx, uint32_t* n_candidates, uint32_t n_rules) {
  EF_REQUIRE(n_candidates, "null n_candidates");
  *n_candidates = 0;
  EF_REQUIRE(!ctx->dirty, "tables not committed (call ef_tables_commit)");
  EF_REQUIRE(ctx->vis_mask, "visited set not initialised");
  EF_REQUIRE(n_rules <= 8, "at most 8 rules");
  cudaSetDevice(ctx->dev);
  ctx->kcount_step0 = ctx->kcount;
  return EF_OK;
}

int ef_expand(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules, uint32_t n_rules,
              const ef_price_params* pp, int insert_visited, uint32_t* n_candidates) {
  int rc = step_begin(ctx, n_candidates, n_rules);
  if (rc) return rc;
  uint32_t total = 0;
  // large graphs: price every candidate on a second stream while the chunks hash (their
  // pricing does not depend on the hashes, only which of them survive the dedup does)
  ctx->spec_pp = ctx->spec_price && pp && pp->use_inner ? pp : nullptr;
  ctx->spec_sharded = false;
  rc = step_hash(ctx, parent_slots, n_parents, rules, n_rules, &total);
  ctx->spec_pp = nullptr;
  if (rc) return rc;
  if ((rc = step_dedup_local(ctx, pp)) || (rc = step_price(ctx, pp)) || (rc = step_prune(ctx, pp))) return rc;
  rc = step_sync(ctx, true);
  *n_candidates = total;
  if (rc) return rc;
  if (insert_visited && (rc = insert_firsts(ctx))) return rc;
  return EF_OK;
}

// ---- hash-owner sharding ---------------------------------------------------------------------

int ef_expand_hashes(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                     uint32_t n_rules, uint32_t* n_candidates) {
  int rc = step_begin(ctx, n_candidates, n_rules);
  if (rc) return rc;
  uint32_t total = 0;
  if ((rc = step_hash(ctx, parent_slots, n_parents, rules, n_rules, &total))) return rc;
  rc = step_sync(ctx, false);
  *n_candidates = total;
  return rc;
}

int ef_expand_hashes_spec(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                          uint32_t n_rules, const ef_price_params* pp, uint32_t* n_candidates) {
  int rc = step_begin(ctx, n_candidates, n_rules);
  if (rc) return rc;
  uint32_t total = 0;
  // speculative pricing as in ef_expand; ef_expand_finish(_padded) commits the survivors (the
  // owners' verdicts: first occurrences, FIRST)
  ctx->spec_pp = ctx->spec_price && pp && pp->use_inner ? pp : nullptr;
  rc = step_hash(ctx, parent_slots, n_parents, rules, n_rules, &total);
  ctx->spec_pp = nullptr;
  ctx->spec_sharded = true;
  if (rc) return rc;
  rc = step_sync(ctx, false);
  *n_candidates = total;
  return rc;
}

int ef_route_owners(ef_ctx* ctx, uint32_t world, uint64_t order_base, uint64_t* d_send, uint32_t* counts) {
  EF_REQUIRE(world >= 1 && world <= 1024 && counts && d_send, "ef_route_owners: bad arguments");
  const uint32_t total = ctx->last_total;
  EF_CUDA(ctx->d_route.reserve(2 * (size_t)world + 2, ctx->st));
  EF_CUDA(ctx->d_perm.reserve(std::max<uint32_t>(total, 1), ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_route.p, 0, (2 * (size_t)world + 2) * 4, ctx->st));
  const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
  RouteArgs R{ctx->d_res.p, total, world, order_base, ctx->d_route.p, ctx->d_route.p + world, d_send, ctx->d_perm.p};
  ++ctx->kcount, k_route_count<<<grid_t, 256, world * 4, ctx->st>>>(R);
  EF_CUDA(cudaGetLastError());
  std::vector<uint32_t> cnt(world), off(world);
  EF_CUDA(cudaMemcpyAsync(cnt.data(), ctx->d_route.p, world * 4, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  uint32_t run = 0;
  for (uint32_t w = 0; w < world; ++w) {
    off[w] = run;
    run += cnt[w];
    counts[w] = cnt[w];
  }
  ctx->n_send = run;
  EF_CUDA(cudaMemcpyAsync(ctx->d_route.p + world, off.data(), world * 4, cudaMemcpyHostToDevice, ctx->st));
  ++ctx->kcount, k_route_scatter<<<grid_t, 256, world * 8, ctx->st>>>(R);
  EF_CUDA(cudaGetLastError());
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_owner_mark(ef_ctx* ctx, const uint64_t* d_recv, uint32_t n_recv, uint32_t* d_verdict, int insert_visited) {
  EF_REQUIRE(ctx->vis_mask, "visited set not initialised");
  if (!n_recv) return EF_OK;
  if (insert_visited) {
    int rc = vis_reserve(ctx, n_recv);
    if (rc) return rc;
  }
  const uint32_t tcap = pow2_at_least(2ull * std::max<uint32_t>(n_recv, 1024));
  EF_CUDA(ctx->d_step_key.reserve(tcap, ctx->st));
  EF_CUDA(ctx->d_step_ord.reserve(tcap, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_step_key.p, 0, (size_t)tcap * 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_step_ord.p, 0xff, (size_t)tcap * 8, ctx->st));
  OwnerArgs O{d_recv, n_recv, d_verdict, ctx->d_step_key.p, ctx->d_step_ord.p, tcap - 1, ctx->d_vis.p, ctx->vis_mask,
              ctx->d_vis_count.p, ctx->d_vis_err.p};
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((n_recv + 255) / 256, ctx->n_sm * 8));
  ++ctx->kcount, k_owner_claim<<<grid, 256, 0, ctx->st>>>(O);
  ++ctx->kcount, k_owner_resolve<<<grid, 256, 0, ctx->st>>>(O);
  if (insert_visited) ++ctx->kcount, k_owner_insert<<<grid, 256, 0, ctx->st>>>(O);
  EF_CUDA(cudaGetLastError());
  return insert_visited ? vis_settle(ctx) : (cudaStreamSynchronize(ctx->st) == cudaSuccess ? EF_OK : EF_ERR_CUDA);
}

int ef_expand_finish(ef_ctx* ctx, const uint32_t* d_verdict_back, const ef_price_params* pp) {
  const uint32_t total = ctx->last_total;
  EF_CUDA(cudaMemsetAsync(ctx->d_scalars.p + 7, 0, 4, ctx->st));
  cudaEventRecord(ctx->ev[3], ctx->st);
  if (ctx->n_send) {
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((ctx->n_send + 255) / 256, ctx->n_sm * 8));
    ++ctx->kcount, k_apply_verdicts<<<grid, 256, 0, ctx->st>>>(ctx->d_res.p, ctx->d_perm.p, d_verdict_back, ctx->n_send,
                                                pp->node_cap);
    const uint32_t gc = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
    ++ctx->kcount, k_compact_survivors<<<gc, 256, 0, ctx->st>>>(ctx->d_res.p, total, ctx->d_plist.p, ctx->d_scalars.p + 7);
    EF_CUDA(cudaGetLastError());
  }
  cudaEventRecord(ctx->ev[4], ctx->st);
  int rc = step_price(ctx, pp);
  if (rc || (rc = step_prune(ctx, pp))) return rc;
  return step_sync(ctx, true);
}

// ---- the padded exchange: no count goes through the host -------------------------------------

int ef_route_owners_padded(ef_ctx* ctx, uint32_t world, uint64_t order_base, uint32_t cap, uint64_t* d_send,
                           uint32_t* d_counts) {
  EF_REQUIRE(world >= 1 && world <= 1024 && d_counts && d_send, "ef_route_owners_padded: bad arguments");
  const uint32_t total = ctx->last_total;
  EF_REQUIRE(cap >= total, "ef_route_owners_padded: cap below this rank's candidate count");
  EF_CUDA(ctx->d_perm.reserve(std::max<uint64_t>((uint64_t)world * cap, 1), ctx->st));
  EF_CUDA(cudaMemsetAsync(d_counts, 0, world * 4, ctx->st));
  const uint32_t grid_t = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
  RouteArgs R{ctx->d_res.p, total, world, order_base, d_counts, nullptr, d_send, ctx->d_perm.p};
  if (total) ++ctx->kcount, k_route_pad<<<grid_t, 256, 0, ctx->st>>>(R, cap);
  EF_CUDA(cudaGetLastError());
  ctx->pad_counts = d_counts;
  return EF_OK;
}

int ef_owner_mark_padded(ef_ctx* ctx, const uint64_t* d_recv, const uint32_t* d_recv_counts, uint32_t world,
                         uint32_t cap, uint32_t* d_verdict, int insert_visited) {
  EF_REQUIRE(ctx->vis_mask, "visited set not initialised");
  EF_REQUIRE(world >= 1 && world <= 1024 && d_recv && d_recv_counts && d_verdict, "ef_owner_mark_padded: bad arguments");
  const uint64_t n = (uint64_t)world * cap;
  if (!n) return EF_OK;
  EF_REQUIRE(n < (1ull << 31), "ef_owner_mark_padded: world * cap above 2^31");
  if (insert_visited) {
    int rc = vis_reserve(ctx, n);  // an upper bound: no host round trip unless the table may fill
    if (rc) return rc;
  }
  const uint32_t tcap = pow2_at_least(2ull * std::max<uint64_t>(n, 1024));
  EF_CUDA(ctx->d_step_key.reserve(tcap, ctx->st));
  EF_CUDA(ctx->d_step_ord.reserve(tcap, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_step_key.p, 0, (size_t)tcap * 8, ctx->st));
  EF_CUDA(cudaMemsetAsync(ctx->d_step_ord.p, 0xff, (size_t)tcap * 8, ctx->st));
  OwnerArgs O{d_recv, (uint32_t)n, d_verdict, ctx->d_step_key.p, ctx->d_step_ord.p, tcap - 1, ctx->d_vis.p,
              ctx->vis_mask, ctx->d_vis_count.p, ctx->d_vis_err.p};
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, ctx->n_sm * 8ull));
  ++ctx->kcount, k_owner_claim_pad<<<grid, 256, 0, ctx->st>>>(O, d_recv_counts, cap);
  ++ctx->kcount, k_owner_resolve_pad<<<grid, 256, 0, ctx->st>>>(O, d_recv_counts, cap);
  if (insert_visited) {
    ++ctx->kcount, k_owner_insert_pad<<<grid, 256, 0, ctx->st>>>(O, d_recv_counts, cap);
    ctx->vis_bound += n;  // stays an upper bound without reading the count back
  }
  EF_CUDA(cudaGetLastError());
  return EF_OK;
}

int ef_expand_finish_padded(ef_ctx* ctx, const uint32_t* d_verdict_back, uint32_t world, uint32_t cap,
                            const ef_price_params* pp) {
  EF_REQUIRE(ctx->pad_counts, "ef_expand_finish_padded: no ef_route_owners_padded before it");
  const uint32_t total = ctx->last_total;
  EF_CUDA(cudaMemsetAsync(ctx->d_scalars.p + 7, 0, 4, ctx->st));
  cudaEventRecord(ctx->ev[3], ctx->st);
  if (total) {
    const uint64_t n = (uint64_t)world * cap;
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, ctx->n_sm * 8ull));
    ++ctx->kcount, k_apply_verdicts_pad<<<grid, 256, 0, ctx->st>>>(ctx->d_res.p, ctx->d_perm.p, ctx->pad_counts,
                                                                   d_verdict_back, world, cap, pp->node_cap);
    const uint32_t gc = std::max<uint32_t>(1, std::min<uint32_t>((total + 255) / 256, ctx->n_sm * 8));
    ++ctx->kcount, k_compact_survivors<<<gc, 256, 0, ctx->st>>>(ctx->d_res.p, total, ctx->d_plist.p, ctx->d_scalars.p + 7);
    EF_CUDA(cudaGetLastError());
  }
  ctx->pad_counts = nullptr;
  cudaEventRecord(ctx->ev[4], ctx->st);
  int rc = step_price(ctx, pp);
  if (rc || (rc = step_prune(ctx, pp))) return rc;
  return step_sync(ctx, true);
}

int ef_commit_bytes(ef_ctx* ctx, uint64_t* bytes) {
  EF_REQUIRE(bytes, "ef_commit_bytes: null out");
  *bytes = ctx->commit_bytes;
  return EF_OK;
}

int ef_stream(ef_ctx* ctx, void** stream) {
  EF_REQUIRE(stream, "ef_stream: null out");
  *stream = (void*)ctx->st;
  return EF_OK;
}

int ef_reprune(ef_ctx* ctx, double best, double alpha) {
  ef_price_params pp{};
  pp.best = best;
  pp.alpha = alpha;
  int rc = step_prune(ctx, &pp);
  if (rc) return rc;
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_pending(ef_ctx* ctx, ef_sig_desc* sigs, uint32_t sig_cap, uint32_t* n_sigs, int32_t* derives, uint32_t derive_cap,
               uint32_t* n_derives) {
  uint32_t ns = std::min(ctx->last_req_sig, ctx->req_cap), nd = std::min(ctx->last_req_dv, ctx->req_cap);
  if (n_sigs) *n_sigs = ns;
  if (n_derives) *n_derives = nd;
  if (sigs && ns) EF_CUDA(cudaMemcpyAsync(sigs, ctx->d_req_sig.p, std::min(ns, sig_cap) * sizeof(ef_sig_desc), cudaMemcpyDeviceToHost, ctx->st));
  if (derives && nd) EF_CUDA(cudaMemcpyAsync(derives, ctx->d_req_dv.p, std::min(nd, derive_cap) * 16, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_results(ef_ctx* ctx, ef_cand_result* out, uint32_t n) {
  EF_REQUIRE(n <= ctx->last_total, "ef_results: more than the last step produced");
  if (!n) return EF_OK;
  EF_CUDA(cudaMemcpyAsync(out, ctx->d_res.p, n * sizeof(ef_cand_result), cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_results_async(ef_ctx* ctx, ef_cand_result* out, uint32_t n) {
  EF_REQUIRE(n <= ctx->last_total, "ef_results_async: more than the last step produced");
  if (!n) return EF_OK;
  EF_CUDA(cudaEventSynchronize(ctx->ev_copy));  // the previous copy still reads the snapshot
  EF_CUDA(ctx->d_res_snap.reserve(n, ctx->st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_res_snap.p, ctx->d_res.p, n * sizeof(ef_cand_result), cudaMemcpyDeviceToDevice,
                          ctx->st));
  EF_CUDA(cudaEventRecord(ctx->ev_snap, ctx->st));
  EF_CUDA(cudaStreamWaitEvent(ctx->st_copy, ctx->ev_snap, 0));
  EF_CUDA(cudaMemcpyAsync(out, ctx->d_res_snap.p, n * sizeof(ef_cand_result), cudaMemcpyDeviceToHost, ctx->st_copy));
  EF_CUDA(cudaEventRecord(ctx->ev_copy, ctx->st_copy));
  return EF_OK;
}

int ef_results_wait(ef_ctx* ctx) {
  EF_CUDA(cudaEventSynchronize(ctx->ev_copy));
  return EF_OK;
}

int ef_keep(ef_ctx* ctx, const uint32_t* cand_idx, uint32_t n, const uint32_t* slots) {
  if (!n) return EF_OK;
  const Geo& g = ctx->geo;
  std::vector<unsigned long long> dst(n);
  for (uint32_t i = 0; i < n; ++i) {
    EF_REQUIRE(cand_idx[i] < ctx->last_total, "ef_keep: bad candidate index");
    EF_REQUIRE(slots[i] < ctx->n_slots, "ef_keep: bad slot");
    dst[i] = (unsigned long long)slot_addr(ctx, slots[i]);
  }
  std::vector<uint32_t> sel(cand_idx, cand_idx + n);
  int rc;
  if ((rc = upload(ctx, ctx->d_dst, dst)) || (rc = upload(ctx, ctx->d_sel, sel))) return rc;
  // the step's parents, sites and plans are still in place: materialise the chosen candidates
  StepArgs A = ctx->last_step;
  A.sel = ctx->d_sel.p;
  A.n_sel = n;
  A.dst = ctx->d_dst.p;
  ++ctx->kcount, k_materialise<kMatThreads><<<std::min<uint32_t>(n, ctx->n_sm * 8), kMatThreads, 0, ctx->st>>>(A);
  EF_CUDA(cudaGetLastError());
  ++ctx->kcount, k_keep_alg<<<std::min<uint32_t>(n, ctx->n_sm * 8), 128, 0, ctx->st>>>(ctx->d_alg8.p, ctx->step_S, ctx->d_sel.p,
                                                                      ctx->d_dst.p, n, g, make_tables(ctx),
                                                                      (int)ctx->alg_rows);
  EF_CUDA(cudaGetLastError());
  // node keys, sorted order and ranks of the new records (every parent carries them)
  EF_CUDA(ctx->d_hash_out.reserve(n, ctx->st));
  if ((rc = hash_records_full(ctx, ctx->sc[0], ctx->st, ctx->d_dst.p, n, ctx->d_hash_out.p))) return rc;
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  return EF_OK;
}

int ef_materialise(ef_ctx* ctx, const uint32_t* parent_slots, uint32_t n_parents, const int32_t* rules,
                   uint32_t n_rules, const uint32_t* cand_parent, const uint32_t* cand_local, uint32_t n,
                   const uint32_t* slots) {
  EF_REQUIRE(!ctx->dirty, "tables not committed (call ef_tables_commit)");
  EF_REQUIRE(n_rules <= 8, "at most 8 rules");
  if (!n) return EF_OK;
  EF_REQUIRE(n_parents, "ef_materialise: no parents");
  cudaSetDevice(ctx->dev);
  const Geo& g = ctx->geo;
  std::vector<unsigned long long> dst(n);
  for (uint32_t i = 0; i < n; ++i) {
    EF_REQUIRE(cand_parent[i] < n_parents, "ef_materialise: bad parent index");
    EF_REQUIRE(slots[i] < ctx->n_slots, "ef_materialise: bad slot");
    dst[i] = (unsigned long long)slot_addr(ctx, slots[i]);
  }
  for (int attempt = 0; attempt < 8; ++attempt) {
    int rc = ensure_parent_buffers(ctx, n_parents);
    if (rc || (rc = stage_addrs(ctx, ctx->d_parent_addr, parent_slots, n_parents))) return rc;
    EF_CUDA(cudaMemsetAsync(ctx->d_scalars.p, 0, 16 * 4, ctx->st));
    StepArgs A{};
    A.g = g;
    A.T = make_tables(ctx);
    A.parent_addr = ctx->d_parent_addr.p;
    A.n_parents = n_parents;
    A.pscratch = ctx->d_pscratch.p;
    A.pstride = pstride_of(g);
    for (uint32_t i = 0; i < n_rules; ++i) A.rules[i] = rules[i];
    A.n_rules = (int32_t)n_rules;
    A.sites = ctx->d_sites.p;
    A.site_cap = ctx->site_cap;
    A.site_count = ctx->d_site_count.p;
    A.cand_off = ctx->d_cand_off.p;
    A.total = ctx->d_scalars.p + 0;
    A.err = ctx->d_scalars.p + 1;
    A.n_req_sig = ctx->d_scalars.p + 2;
    A.n_req_dv = ctx->d_scalars.p + 3;
    A.cand_cap = 0xffffffffu;
    EF_CUDA(ctx->d_req_sig.reserve(ctx->req_cap, ctx->st));
    EF_CUDA(ctx->d_req_dv.reserve(4 * ctx->req_cap, ctx->st));
    A.req_sig = ctx->d_req_sig.p;
    A.req_dv = ctx->d_req_dv.p;
    A.req_sig_cap = A.req_dv_cap = ctx->req_cap;
    ++ctx->kcount, k_match<kMatchThreads><<<std::min<uint32_t>(n_parents, ctx->n_sm * 8), kMatchThreads, 0, ctx->st>>>(A);
    ++ctx->kcount, k_offsets<1024><<<1, 1024, 0, ctx->st>>>(A);
    EF_CUDA(cudaGetLastError());
    std::vector<uint32_t> coff(n_parents + 1);
    EF_CUDA(cudaMemcpyAsync(ctx->h_scalars, ctx->d_scalars.p, 16 * 4, cudaMemcpyDeviceToHost, ctx->st));
    EF_CUDA(cudaMemcpyAsync(coff.data(), ctx->d_cand_off.p, (n_parents + 1) * 4, cudaMemcpyDeviceToHost, ctx->st));
    EF_CUDA(cudaStreamSynchronize(ctx->st));
    if (ctx->h_scalars[1] & 1u) {  // site buffer too small
      ctx->site_cap *= 4;
      continue;
    }
    std::vector<uint32_t> sel(n);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t p = cand_parent[i];
      EF_REQUIRE(cand_local[i] < coff[p + 1] - coff[p], "ef_materialise: candidate index beyond its parent's sites");
      sel[i] = coff[p] + cand_local[i];
    }
    if ((rc = upload(ctx, ctx->d_dst, dst)) || (rc = upload(ctx, ctx->d_sel, sel))) return rc;
    A.sel = ctx->d_sel.p;
    A.n_sel = n;
    A.dst = ctx->d_dst.p;
    ++ctx->kcount, k_materialise<kMatThreads><<<std::min<uint32_t>(n, ctx->n_sm * 8), kMatThreads, 0, ctx->st>>>(A);
    EF_CUDA(cudaGetLastError());
    EF_CUDA(cudaMemcpyAsync(ctx->h_scalars, ctx->d_scalars.p, 16 * 4, cudaMemcpyDeviceToHost, ctx->st));
    EF_CUDA(cudaStreamSynchronize(ctx->st));
    ctx->last_total = 0;  // the step state now describes these parents: ef_keep is invalid
    EF_REQUIRE(!(ctx->h_scalars[1] & 4u), "candidate exceeds record capacity (raise cap_nodes/cap_refs)");
    // a rewrite whose signature / weight set this context has not interned yet (another rank's
    // step resolved it): the records hold unresolved ids, so they are not hashed; the caller
    // resolves (ef_pending) and calls again
    ctx->last_req_sig = ctx->h_scalars[2];
    ctx->last_req_dv = ctx->h_scalars[3];
    if (ctx->last_req_sig || ctx->last_req_dv) return EF_NEED_RESOLVE;
    EF_CUDA(ctx->d_hash_out.reserve(n, ctx->st));
    if ((rc = hash_records_full(ctx, ctx->sc[0], ctx->st, ctx->d_dst.p, n, ctx->d_hash_out.p))) return rc;
    EF_CUDA(cudaStreamSynchronize(ctx->st));
    return EF_OK;
  }
  ctx->err = "ef_materialise: site buffer did not converge";
  return EF_ERR_CAPACITY;
}

int ef_last_timing(ef_ctx* ctx, float* ms, uint32_t n) {
  for (uint32_t k = 0; k < n && k < 9; ++k) ms[k] = ctx->last_ms[k];
  return EF_OK;
}

int ef_last_stats(ef_ctx* ctx, uint64_t* out, uint32_t n) {
  for (uint32_t k = 0; k < n && k < 5; ++k) out[k] = ctx->last_stats[k];
  return EF_OK;
}

int ef_records_write_packed_async(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host,
                                  const uint64_t* offsets, uint64_t bytes) {
  EF_REQUIRE(!ctx->dirty, "tables not committed (call ef_tables_commit)");
  if (!n) return EF_OK;
  // record sizes from the host copy: no device round trip before the hashing is queued
  const uint8_t* hb = reinterpret_cast<const uint8_t*>(host);
  uint32_t max_n = 0, max_refs = 0;
  ctx->h_up_off.assign(offsets, offsets + n);
  ctx->h_up_dst.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    EF_REQUIRE(slots[i] < ctx->n_slots, "ef_records_write_packed: bad slot");
    EF_REQUIRE(offsets[i] % 4 == 0 && offsets[i] + 16 <= bytes, "ef_records_write_packed: bad offset");
    const uint32_t* h = reinterpret_cast<const uint32_t*>(hb + offsets[i]);
    EF_REQUIRE(h[0] <= ctx->geo.cap_nodes && h[1] <= ctx->geo.cap_refs && h[2] <= ctx->geo.cap_outs,
               "ef_records_write_packed: record exceeds the geometry");
    max_n = std::max(max_n, h[0]);
    max_refs = std::max(max_refs, h[1]);
    ctx->h_up_dst[i] = (unsigned long long)slot_addr(ctx, slots[i]);
  }
  cudaStream_t st = ctx->st_up;
  // the slots may still be read by queued main-stream work: the upload starts after it
  EF_CUDA(cudaEventRecord(ctx->ev_main, ctx->st));
  EF_CUDA(cudaStreamWaitEvent(st, ctx->ev_main, 0));
  EF_CUDA(ctx->d_up_stage.reserve(bytes, st));
  EF_CUDA(ctx->d_up_off.reserve(n, st));
  EF_CUDA(ctx->d_up_dst.reserve(n, st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_up_stage.p, host, bytes, cudaMemcpyHostToDevice, st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_up_off.p, ctx->h_up_off.data(), n * 8ull, cudaMemcpyHostToDevice, st));
  EF_CUDA(cudaMemcpyAsync(ctx->d_up_dst.p, ctx->h_up_dst.data(), n * 8ull, cudaMemcpyHostToDevice, st));
  ++ctx->kcount, k_unpack<<<std::min<uint32_t>(n, ctx->n_sm * 8), 256, 0, st>>>(reinterpret_cast<const uint8_t*>(ctx->d_up_stage.p),
                                                                 ctx->d_up_off.p, ctx->d_up_dst.p, n, ctx->geo);
  EF_CUDA(cudaGetLastError());
  int rc = hash_records_full(ctx, ctx->sc[1], st, ctx->d_up_dst.p, n, nullptr, max_n, max_refs);
  if (rc) return rc;
  EF_CUDA(cudaEventRecord(ctx->ev_up, st));
  return EF_OK;
}

int ef_upload_fence(ef_ctx* ctx) {
  EF_CUDA(cudaStreamWaitEvent(ctx->st, ctx->ev_up, 0));
  return EF_OK;
}

int ef_records_write_packed(ef_ctx* ctx, const uint32_t* slots, uint32_t n, const void* host, const uint64_t* offsets,
                            uint64_t bytes) {
  int rc = ef_records_write_packed_async(ctx, slots, n, host, offsets, bytes);
  if (rc) return rc;
  EF_CUDA(cudaStreamSynchronize(ctx->st_up));
  return EF_OK;
}

int ef_check_division(ef_ctx* ctx, const double* divisors, uint32_t n_divisors, uint64_t per_divisor, uint64_t seed,
                      uint64_t* mismatches) {
  EF_REQUIRE(divisors && n_divisors && mismatches, "ef_check_division: bad arguments");
  cudaSetDevice(ctx->dev);
  DevBuf<double> ys;
  DevBuf<unsigned long long> bad;
  EF_CUDA(ys.reserve(n_divisors, ctx->st));
  EF_CUDA(bad.reserve(1, ctx->st));
  EF_CUDA(cudaMemcpyAsync(ys.p, divisors, n_divisors * 8ull, cudaMemcpyHostToDevice, ctx->st));
  EF_CUDA(cudaMemsetAsync(bad.p, 0, 8, ctx->st));
  ++ctx->kcount, k_div_check<<<ctx->n_sm * 8, 256, 0, ctx->st>>>(ys.p, n_divisors, per_divisor, seed, bad.p);
  EF_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  EF_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, ctx->st));
  EF_CUDA(cudaStreamSynchronize(ctx->st));
  *mismatches = h;
  return EF_OK;
}

int ef_b2b_peak(ef_ctx* ctx, double* compress_per_s) {
  cudaSetDevice(ctx->dev);
  const int blocks = ctx->n_sm * 16, threads = 128, iters = 1000;
  DevBuf<uint64_t> out;
  EF_CUDA(out.reserve((size_t)blocks * threads, ctx->st));
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(ctx->ev[0], ctx->st);
    ++ctx->kcount, k_b2b_peak<<<blocks, threads, 0, ctx->st>>>(out.p, iters);
    cudaEventRecord(ctx->ev[1], ctx->st);
    EF_CUDA(cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    const double r = (double)blocks * threads * iters / (ms * 1e-3);
    if (rep > 0 && r > best) best = r;
  }
  out.release();
  *compress_per_s = best;
  return EF_OK;
}

