// The frontier step on *virtual candidates*.
//
// A candidate is never written out as a record during the step: it is its parent record
// (resident in HBM, shared by all of the parent's candidates, so L1/L2 serve it) plus a
// small rewrite plan (VPlan, ~100 bytes).  Only the candidates the search keeps are
// materialised afterwards (ef_keep).  Per step:
//
//   k_plan    thread/candidate  the rewrite plan of rules.py:164-331 in parent coordinates
//   k_reach   warp/parent       (parents <= 256 nodes) downstream-closure rows of every slot
//   k_dirty_warp warp/candidate one "job" per node whose Merkle key (graph.py:530-540)
//                               changes: its signature, weight set and the source of every
//                               producer key (parent key or fresh key j); the dirty set is an
//                               OR of reach rows.  k_dirty (thread/candidate, a walk of the
//                               topological order) serves larger parents.
//   sort      cub radix         candidates by job count, so the lanes of a warp run the same
//                               number of compressions
//   k_keys    thread/candidate  one BLAKE2b-128 per job; the message is built in registers /
//                               a per-thread shared-memory column, compressed at ONE call site
//   k_keys_wide warp/candidate  (large graphs) candidates with >= 512 jobs, a level of their
//                               key DAG per round, on a side stream beside k_keys
//   k_keys_quad 4 lanes/cand.   launches too small to fill the GPU (uploads, kept records)
//   rows <= 256: k_merge (warp/candidate: fresh keys sorted in registers, merged by rank
//                with the parent's sorted keys minus removed ranks into a key stream)
//   rows > 256:  k_sortkeys / cub segmented sort of the fresh keys, then k_merge_big
//                (warp/candidate merge path) into the key stream
//   k_digest_pm thread/candidate BLAKE2b-64 over input text, output keys and the key stream
//                               (graph.py:541-549)
// followed by the dedup kernels and k_price_v on the virtual view.
#pragma once
#include "ef_kernels.cuh"

// minimum resident CTAs per SM for the step's throughput kernels (register budgets; tuned on
// the ResNet-50 frontier)
#ifndef EF_PRICE_THREADS
#define EF_PRICE_THREADS 64  // k_price_v block size (one survivor per thread)
#endif
#ifndef EF_MERGE_MINB
#define EF_MERGE_MINB 6
#endif
#ifndef EF_DIGEST_MINB
#define EF_DIGEST_MINB 4
#endif
#ifndef EF_DIGEST_PF_MINB  // the prefetching digest of large rows (k_digest_pm<.., true, ..>)
#define EF_DIGEST_PF_MINB 3  // 3 CTAs per SM without spills (DAG-20k digest 62.6 -> 56.5 ms; 4 spills: 89 ms)
#endif
#ifndef EF_KEYS_MINB
#define EF_KEYS_MINB 4
#endif

namespace ef {

constexpr uint32_t kFresh = 0x80000000u;  // refsrc: key comes from the candidate's fresh keys
constexpr int kKeyMaxW = 32;              // message words a job may use in the fast path (256 bytes)

// rewrite plan in parent coordinates (positions >= pn are the new nodes pn, pn + 1)
struct VPlan {
  int32_t drop0, drop1;  // removed parent positions, ascending (-1: none)
  int32_t mod;           // parent position rewritten in place (-1: none)
  uint32_t mod_sig, mod_aux;
  int32_t live[2];
  uint32_t new_sig[2], new_aux[2], new_ref[2];
  int32_t n_rm;
  uint32_t rm_from[2], rm_to[2];
  int32_t ins_slot;   // parent topo slot where the new nodes are emitted (-1: none)
  int32_t ins_after;  // 1: after the node at ins_slot, 0: in place of it (that node is dropped)
  int32_t first;      // first parent topo slot whose key can change
  int32_t pn, n_keep, n_live;
  uint32_t parent;
};

struct Job {
  uint32_t sig, aux, roff, nin;
};

struct VArgs {
  Geo g;
  Tables T;
  const unsigned long long* parent_addr;
  const VPlan* plan;  // whole step
  ef_cand_result* res;
  uint32_t c0, n;     // chunk: candidates [c0, c0 + n)
  uint32_t S, Rs;     // per-candidate strides: node slots, ref slots
  uint32_t* didx;     // [n][S]  fresh index + 1 of a dirty node (0: key unchanged)
  Job* jobs;          // [n][S]
  uint32_t* refsrc;   // [n][Rs]
  uint64_t* fresh;    // [n][S][2]
  uint32_t* dcount;   // [n]
  uint16_t* jlvl;     // [n][S] job level in the candidate's key DAG (k_dirty; null: not computed)
  uint32_t wide_min;  // > 0: candidates with at least this many jobs go to k_keys_wide, not k_keys
  const uint32_t* order;  // [n] chunk-local candidate per lane (k_keys)
  uint64_t* skey;     // [n][S] sort keys (first key word, big endian)
  const uint64_t* skey_sorted;
  uint32_t* sval_sorted;
  int32_t* seg_begin;  // [n]
  int32_t* seg_end;    // [n]
  const uint32_t* pscratch;  // per-parent tables of k_match and k_reach
  uint64_t pstride;
  uint32_t Os;         // words per output-source row
  uint32_t* outsrc;    // [n][Os] key source of every (remapped) graph output (k_dirty_warp)
  int slots;           // 1: rows <= kFastRows (k_dirty_warp, k_merge)
  int osrc;            // 1: the dirty kernel wrote outsrc (graph output key sources) instead of didx rows
  uint32_t W;          // words per removed-mask row
  uint32_t* rmask;     // [n][W] parent keys (by sorted rank) absent from the candidate: dropped or dirty
  uint64_t* fresh_sorted;  // [n][S][2] the fresh keys in ascending byte order
  uint64_t* kstream;       // [n][S][2] the merged key stream k_digest_pm hashes (k_merge: fresh_sorted)
  const uint32_t* pdir;    // [parent][kDirN] first sorted rank per top-12-bit prefix (k_merge_dir), or null
  const uint64_t* input_words;  // input text, 8-byte words, zero padded
  uint64_t* pfx;       // [n][pfx_stride] the digest's prefix (input text, output keys and ports) as
                       // little-endian words (k_prefix), or null: the digest assembles it itself
  uint32_t pfx_stride;
  uint32_t* pfx_first;        // [n] first graph output whose (key, port) differs from the parent's (k_dirty_big)
  const uint64_t* pfx_state;  // [parent][pfx_nst][8] BLAKE2b state of the parent's digest after b prefix blocks
  uint32_t pfx_nst;           //   (k_pfx_chain), or null: every digest starts from block 0
  uint32_t* err;
  // full mode (whole records: uploads, kept candidates): parent_addr[c] is record c itself,
  // every node is a job, jv[c][j] = position of job j; graph hashes go to hash_out[c]
  int full;
  uint32_t* jv;
  uint64_t* hash_out;
  unsigned long long* stats;  // [0] k_keys compressions, [1] k_digest compressions (may be null)
};

constexpr uint32_t kInputJob = 0x80000000u;  // Job.nin flag: input node, aux = input-name id

// ------------------------------------------------------------------------------------------
// k_plan
// ------------------------------------------------------------------------------------------

__global__ void k_plan(StepArgs A, VPlan* plans) {
  const Geo& G = A.g;
  const uint32_t total = min(A.total[0], A.cand_cap);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = A.n_parents;  // parent: last pi with cand_off[pi] <= c
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (A.cand_off[mid] <= c) lo = mid;
      else hi = mid;
    }
    const uint32_t pi = lo;
    const unsigned long long site = A.sites[(uint64_t)pi * A.site_cap + (c - A.cand_off[pi])];
    const uint32_t rule = (uint32_t)(site >> 56), sa = (uint32_t)(site >> 28) & 0xfffffffu, sb = (uint32_t)site & 0xfffffffu;
    Rec R{reinterpret_cast<char*>(A.parent_addr[pi])};
    const int n = R.h().n, n_refs = R.h().n_refs;
    const uint32_t* u0 = A.pscratch + (uint64_t)pi * A.pstride;
    const uint32_t* u1 = u0 + G.cap_nodes;
    const uint32_t* tslot = u0 + 4 * G.cap_nodes + 1 + G.cap_refs;
    Plan P;
    plan_rewrite(A, P, R, n, rule, sa, sb, u0, u1);
    VPlan V;
    V.drop0 = P.drop[0];
    V.drop1 = P.drop[1];
    V.mod = P.mod;
    V.mod_sig = P.mod_sig;
    V.mod_aux = P.mod_aux;
    for (int k = 0; k < 2; ++k) {
      V.live[k] = k < P.n_new ? P.live[k] : 0;
      V.new_sig[k] = P.new_sig[k];
      V.new_aux[k] = P.new_aux[k];
      V.new_ref[k] = P.new_ref[k];
      V.rm_from[k] = P.rm_from[k];
      V.rm_to[k] = P.rm_to[k];
    }
    V.n_rm = P.n_rm;
    // insertion point of the new nodes (same placement as k_materialise)
    const int s0 = V.drop0 >= 0 ? (int)tslot[V.drop0] : n;
    const int s1 = V.drop1 >= 0 ? (int)tslot[V.drop1] : n;
    V.ins_slot = -1;
    V.ins_after = 0;
    if (P.n_new > 0) {
      if (rule == EF_R_MERGE_CONVS) {
        V.ins_slot = min(s0, s1);
      } else if (P.topo_node >= 0) {
        V.ins_slot = (int)tslot[P.topo_node];
        V.ins_after = P.topo_mode == 1 ? 1 : 0;
      }
    }
    int first = min(s0, s1);
    if (V.mod >= 0) first = min(first, (int)tslot[V.mod]);
    if (V.ins_slot >= 0) first = min(first, V.ins_slot);
    V.first = first;
    V.pn = n;
    V.n_keep = n - (V.drop0 >= 0) - (V.drop1 >= 0);
    V.n_live = V.live[0] + V.live[1];
    V.parent = pi;
    plans[c] = V;

    int drop_refs = 0;
    if (V.drop0 >= 0) drop_refs += (int)R.nin(G)[V.drop0];
    if (V.drop1 >= 0) drop_refs += (int)R.nin(G)[V.drop1];
    const int n_child = V.n_keep + V.n_live;
    const int n_refs_child = n_refs - drop_refs + V.n_live;
    ef_cand_result* res = A.res + c;
    uint32_t flags = P.incomplete ? EF_F_INCOMPLETE : 0u;
    if (n_child > (int)G.cap_nodes || n_refs_child > (int)G.cap_refs) {
      atomicOr(A.err, 4u);
      flags = EF_F_INCOMPLETE;
    }
    res->flags = flags;
    res->parent = pi;
    res->rule = rule;
    res->site_a = sa;
    res->site_b = sb;
    res->touched_sig[0] = P.touched[0];
    res->touched_sig[1] = P.touched[1];
    res->n_compute = R.h().n_compute - (n - V.n_keep) + V.n_live;
    res->n_nodes = (uint32_t)n_child;
    res->hash = 0;
    res->cost = res->time_ms = res->energy = 0.0;
    res->evals = 0;
    res->sweeps = 0;
  }
}

// ------------------------------------------------------------------------------------------
// k_dirty
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t vremap(const VPlan& P, uint32_t r) {
  for (int k = 0; k < P.n_rm; ++k)
    if (r == P.rm_from[k]) return P.rm_to[k];
  return r;
}

// Lanes of a warp hold neighbouring candidates (mostly of one parent) and walk the same
// warp-uniform range of topological slots in lockstep, so the parent's arrays are read as
// broadcasts and the warp never splits.
__global__ void k_dirty(VArgs A) {
  const Geo& G = A.g;
  const uint32_t span = (A.n + 31) / 32 * 32;
  for (uint32_t lc = blockIdx.x * blockDim.x + threadIdx.x; lc < span; lc += gridDim.x * blockDim.x) {
    const uint32_t c = A.c0 + lc;
    const bool incomplete = lc >= A.n || (A.res[c].flags & EF_F_INCOMPLETE);
    const unsigned mask = __ballot_sync(0xffffffffu, !incomplete);
    if (incomplete) {
      if (lc < A.n) {
        A.dcount[lc] = 0;
        A.seg_begin[lc] = A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S);
      }
      continue;
    }
    const VPlan P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint32_t* topo = R.topo(G);
    const uint32_t* psig = R.sig(G);
    const uint32_t* paux = R.aux(G);
    const uint32_t* pnin = R.nin(G);
    const uint32_t* pinoff = R.inoff(G);
    const uint32_t* prefs = R.refs(G);
    const int pn = P.pn;
    uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    Job* jobs = A.jobs + (uint64_t)lc * A.S;
    uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    for (int i = 0; i < (pn + 2 + 3) / 4; ++i) reinterpret_cast<uint4*>(didx)[i] = make_uint4(0, 0, 0, 0);
    const uint32_t* srank = R.srank(G);
    uint32_t* rm = A.rmask + (uint64_t)lc * A.W;
    for (int w = 0; w < (pn + 31) / 32; ++w) rm[w] = 0;
    auto remove = [&](int v) {
      const uint32_t k = srank[v];
      rm[k >> 5] |= 1u << (k & 31);
    };
    if (P.drop0 >= 0) remove(P.drop0);
    if (P.drop1 >= 0) remove(P.drop1);
    uint32_t j = 0, r = 0;
    // levels for k_keys_wide (only when this candidate can reach its job threshold): by job in
    // jlvl, by parent position in the (step-mode idle) jv row, read beside didx so the level
    // costs no extra dependent load
    const bool levels = A.jlvl && (uint32_t)(pn - max(P.first, 0)) + 2u >= A.wide_min;  // jobs <= slots from first on
    uint16_t* lv = levels ? A.jlvl + (uint64_t)lc * A.S : nullptr;
    uint32_t* plv = A.jv + (uint64_t)lc * A.S;
    uint32_t lvl = 0;  // level of the job being emitted
    auto src_of = [&](uint32_t ref) -> uint32_t {
      const uint32_t p = ref >> 8, port = ref & 255u;
      const uint32_t fi = didx[p];
      if (levels && fi) lvl = max(lvl, plv[p] + 1u);
      return fi ? (kFresh | (port << 23) | (fi - 1)) : ((port << 23) | p);
    };
    auto emit_new = [&]() {
      for (int k = 0; k < 2; ++k) {
        if (!P.live[k]) continue;
        lvl = 0;
        rs[r] = src_of(P.new_ref[k]);  // new nodes are exempt from the remap (rules.py:186-188)
        jobs[j] = Job{P.new_sig[k], P.new_aux[k], r, 1u};
        if (levels) {
          lv[j] = (uint16_t)min(lvl, 65535u);
          plv[pn + k] = lvl;
        }
        r += 1;
        didx[pn + k] = ++j;
      }
    };
    const int s_lo = (int)__reduce_min_sync(mask, (unsigned)P.first);
    const int s_hi = (int)__reduce_max_sync(mask, (unsigned)pn);
    for (int s = s_lo; s < s_hi; ++s) {
      if (s < P.first || s >= pn) continue;
      const int v = (int)topo[s];
      if (v == P.drop0 || v == P.drop1) {
        if (s == P.ins_slot && !P.ins_after) emit_new();
        continue;
      }
      bool dirty = v == P.mod;
      const uint32_t r0 = pinoff[v], nr = pnin[v];
      lvl = 0;
      for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t ref = prefs[r0 + k];
        const uint32_t ref2 = vremap(P, ref);
        const uint32_t sv = src_of(ref2);
        dirty |= (ref2 != ref) || (sv & kFresh);
        rs[r + k] = sv;
      }
      if (dirty) {
        jobs[j] = Job{v == P.mod ? P.mod_sig : psig[v], v == P.mod ? P.mod_aux : paux[v], r, nr};
        if (levels) {
          lv[j] = (uint16_t)min(lvl, 65535u);
          plv[v] = lvl;
        }
        r += nr;
        didx[v] = ++j;
        remove(v);
      }
      if (s == P.ins_slot && P.ins_after) emit_new();
    }
    A.dcount[lc] = j;
    A.seg_begin[lc] = (int32_t)((uint64_t)lc * A.S);
    A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S + j);
  }
}

// ------------------------------------------------------------------------------------------
// k_reach + k_dirty_warp (parents of <= 256 topological slots)
//
// A node's Merkle key changes iff its own (sig, aux) or one of its input refs changes, or a
// producer's key changes (graph.py:528-540), so a candidate's dirty set is the downstream
// closure of its seeds: the node rewritten in place and the owners of remapped refs.
// k_reach gives every parent, once per step, reach[s] = the slots reachable from topological
// slot s (itself included) as 8 words.  k_dirty_warp then takes one warp per candidate: the
// dirty mask is an OR of a few reach rows, job indices are prefix popcounts of the mask, and
// the lanes emit the jobs of 32 slots at a time with no sequential walk.
// ------------------------------------------------------------------------------------------

constexpr uint32_t kReachSlots = 256;
constexpr uint32_t kReachWords = kReachSlots / 32;  // words per reach row

// offset (words) of the parent's reach rows inside its pscratch row (after k_match's tables)
__device__ __forceinline__ uint64_t reach_off(const Geo& G) { return 10ull * G.cap_nodes + 1 + 2ull * G.cap_refs; }

// one warp per parent; dynamic shared memory per warp: s_v[256], coff[257], consumer slots
// [max refs], rows [256 x 8]
__global__ void __launch_bounds__(64) k_reach(StepArgs A, uint32_t rmax) {
  extern __shared__ uint32_t sh_reach[];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint32_t per = 256 + 260 + ((rmax + 3) & ~3u) + kReachSlots * kReachWords;
  uint32_t* sv = sh_reach + wid * per;
  uint32_t* cof = sv + 256;
  uint32_t* cls = cof + 260;
  uint32_t* rows = cls + ((rmax + 3) & ~3u);
  const Geo& G = A.g;
  for (uint32_t pi = blockIdx.x * 2 + wid; pi < A.n_parents; pi += gridDim.x * 2) {
    Rec R{reinterpret_cast<char*>(A.parent_addr[pi])};
    const int n = R.h().n;
    const uint32_t* ps = A.pscratch + (uint64_t)pi * A.pstride;
    const uint32_t* coff = ps + 2 * G.cap_nodes;
    const uint32_t* clist = coff + 2 * G.cap_nodes + 1;
    const uint32_t* tslot = clist + G.cap_refs;
    const uint32_t* s_v = tslot + G.cap_nodes;
    const uint32_t ncons = coff[n];
    for (int i = lane; i < n; i += 32) sv[i] = s_v[i];
    for (int i = lane; i <= n; i += 32) cof[i] = coff[i];
    for (uint32_t x = lane; x < ncons; x += 32) cls[x] = tslot[clist[x]];
    __syncwarp();
    // reverse topological order; lane w owns word w of every row, so there is no cross-lane
    // dependency: a row only reads rows of later slots, written by the same lane
    const int nw = (n + 31) >> 5;
    if ((int)lane < nw) {
      for (int s = n - 1; s >= 0; --s) {
        const uint32_t v = sv[s];
        uint32_t acc = ((s >> 5) == (int)lane) ? 1u << (s & 31) : 0u;
        for (uint32_t x = cof[v]; x < cof[v + 1]; ++x) acc |= rows[cls[x] * kReachWords + lane];
        rows[s * kReachWords + lane] = acc;
      }
    }
    __syncwarp();
    uint32_t* out = A.pscratch + (uint64_t)pi * A.pstride + reach_off(G);
    for (int i = lane; i < n * (int)kReachWords; i += 32) out[i] = rows[i];
    __syncwarp();
  }
}

// position of the r-th (0-based) set bit of x (r < popc(x))
__device__ __forceinline__ uint32_t nth_bit(uint32_t x, uint32_t r) {
  uint32_t pos = 0, c;
  c = __popc(x & 0xffffu);
  if (r >= c) { r -= c; x >>= 16; pos += 16; }
  c = __popc(x & 0xffu);
  if (r >= c) { r -= c; x >>= 8; pos += 8; }
  c = __popc(x & 0xfu);
  if (r >= c) { r -= c; x >>= 4; pos += 4; }
  c = __popc(x & 0x3u);
  if (r >= c) { r -= c; x >>= 2; pos += 2; }
  c = x & 1u;
  if (r >= c) pos += 1;
  return pos;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_dirty_warp(VArgs A) {
  __shared__ uint32_t sh_dm[WARPS][kReachWords], sh_cum[WARPS][kReachWords + 1], sh_rk[WARPS][kReachWords];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t* dm = sh_dm[wid];
  uint32_t* cum = sh_cum[wid];
  uint32_t* rk = sh_rk[wid];
  const Geo& G = A.g;
  for (uint32_t lc = blockIdx.x * WARPS + wid; lc < A.n; lc += gridDim.x * WARPS) {  // warp-uniform
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) {
      if (lane == 0) {
        A.dcount[lc] = 0;
        A.seg_begin[lc] = A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S);
      }
      continue;
    }
    const VPlan P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint32_t* ps = A.pscratch + (uint64_t)P.parent * A.pstride;
    const uint32_t* coff = ps + 2 * G.cap_nodes;
    const uint32_t* clist = coff + 2 * G.cap_nodes + 1;
    const uint32_t* tslot = clist + G.cap_refs;
    const uint32_t* s_v = tslot + G.cap_nodes;
    const uint32_t* s_pk = s_v + G.cap_nodes;
    const uint32_t* rslot = s_pk + G.cap_nodes;
    const uint32_t* reach = ps + reach_off(G);
    const uint32_t* psig = R.sig(G);
    const uint32_t* paux = R.aux(G);
    const uint32_t* pinoff = R.inoff(G);
    const uint32_t* pnin = R.nin(G);
    const uint32_t* prefs = R.refs(G);
    const uint32_t* srank = R.srank(G);
    const int pn = P.pn;
    const int nw = (pn + 31) >> 5;
    if (lane < kReachWords) dm[lane] = rk[lane] = 0;
    __syncwarp();
    // seeds: the node rewritten in place, the owners of remapped refs (dropped nodes excluded)
    const int ms = P.mod >= 0 ? (int)tslot[P.mod] : -1;
    const int ds0 = P.drop0 >= 0 ? (int)tslot[P.drop0] : -1, ds1 = P.drop1 >= 0 ? (int)tslot[P.drop1] : -1;
    auto seed = [&](uint32_t t) {
      for (int w = 0; w < nw; ++w) atomicOr(&dm[w], reach[t * kReachWords + w]);
    };
    if (ms >= 0 && lane == 0) seed((uint32_t)ms);
    uint32_t rf[2] = {0xffffffffu, 0xffffffffu};
    for (int k = 0; k < P.n_rm; ++k) {
      const uint32_t from = P.rm_from[k], p = from >> 8;
      rf[k] = (tslot[p] << 8) | (from & 255u);
      for (uint32_t x = coff[p] + lane; x < coff[p + 1]; x += 32) {
        const uint32_t q = clist[x];
        if ((int)q == P.drop0 || (int)q == P.drop1) continue;
        bool hit = false;
        for (uint32_t r = pinoff[q]; r < pinoff[q] + pnin[q]; ++r) hit |= prefs[r] == from;
        if (hit) seed(tslot[q]);
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (ds0 >= 0) dm[ds0 >> 5] &= ~(1u << (ds0 & 31));
      if (ds1 >= 0) dm[ds1 >> 5] &= ~(1u << (ds1 & 31));
    }
    __syncwarp();
    {  // exclusive prefix popcounts of the mask words
      const uint32_t x = lane < (uint32_t)nw ? (uint32_t)__popc(dm[lane]) : 0u;
      uint32_t inc = x;
#pragma unroll
      for (int o = 1; o < (int)kReachWords; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += y;
      }
      if (lane < kReachWords) cum[lane] = inc - x;
      if (lane == kReachWords - 1) cum[kReachWords] = inc;
    }
    __syncwarp();
    const int ins = P.ins_slot;
    auto popc_below = [&](uint32_t t) -> uint32_t {
      return cum[t >> 5] + __popc(dm[t >> 5] & ((1u << (t & 31)) - 1u));
    };
    auto dirty_at = [&](uint32_t t) -> bool { return (dm[t >> 5] >> (t & 31)) & 1u; };
    auto fidx = [&](uint32_t t) -> uint32_t { return popc_below(t) + ((int)t > ins && ins >= 0 ? P.n_live : 0); };
    auto fnew = [&](int k) -> uint32_t {
      return popc_below((uint32_t)(ins + (P.ins_after ? 1 : 0))) + (k == 1 ? (uint32_t)P.live[0] : 0u);
    };
    auto src_pos = [&](uint32_t ref) -> uint32_t {  // a ref in parent-position space -> key source
      const uint32_t p = ref >> 8, port = ref & 255u;
      if ((int)p >= pn) return kFresh | (port << 23) | fnew((int)p - pn);
      const uint32_t t = tslot[p];
      return dirty_at(t) ? (kFresh | (port << 23) | fidx(t)) : ((port << 23) | p);
    };
    Job* jobs = A.jobs + (uint64_t)lc * A.S;
    uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    // jobs of the dirty slots: lane q takes the q-th dirty slot (32 jobs per round); a job's
    // sources sit at its parent ref offset
    const uint32_t nd = cum[kReachWords];
    for (uint32_t q = lane; q < nd; q += 32) {
      uint32_t w = 0;
      while (cum[w + 1] <= q) ++w;
      const uint32_t t = 32u * w + nth_bit(dm[w], q - cum[w]);
      const uint32_t v = s_v[t], pk = s_pk[t];
      const uint32_t r0 = pk & 0xffffffu, nr = pk >> 24;
      for (uint32_t k = 0; k < nr; ++k) {
        const uint32_t rsl = rslot[r0 + k];
        uint32_t sv;
        if (rsl == rf[0] || rsl == rf[1]) {  // the owner now consumes another producer (a remap)
          sv = src_pos(rsl == rf[0] ? P.rm_to[0] : P.rm_to[1]);
        } else {
          const uint32_t tp = rsl >> 8, port = rsl & 255u;
          sv = dirty_at(tp) ? (kFresh | (port << 23) | fidx(tp)) : ((port << 23) | (prefs[r0 + k] >> 8));
        }
        rs[r0 + k] = sv;
      }
      const bool m = (int)t == ms;
      jobs[q + ((int)t > ins && ins >= 0 ? P.n_live : 0)] = Job{m ? P.mod_sig : psig[v], m ? P.mod_aux : paux[v], r0, nr};
      const uint32_t k = srank[v];
      atomicOr(&rk[k >> 5], 1u << (k & 31));
    }
    const uint32_t pref = R.h().n_refs;
    if (lane < 2 && P.live[lane]) {  // the new nodes, exempt from the remap (rules.py:186-188)
      rs[pref + lane] = src_pos(P.new_ref[lane]);
      jobs[fnew((int)lane)] = Job{P.new_sig[lane], P.new_aux[lane], pref + lane, 1u};
    }
    if (lane == 0) {
      if (P.drop0 >= 0) atomicOr(&rk[srank[P.drop0] >> 5], 1u << (srank[P.drop0] & 31));
      if (P.drop1 >= 0) atomicOr(&rk[srank[P.drop1] >> 5], 1u << (srank[P.drop1] & 31));
    }
    // graph outputs (remapped) -> key sources, for the digest
    const uint32_t* pouts = R.outs(G);
    uint32_t* os = A.outsrc + (uint64_t)lc * A.Os;
    for (int o = lane; o < R.h().n_out; o += 32) os[o] = src_pos(vremap(P, pouts[o]));
    __syncwarp();
    uint32_t* grm = A.rmask + (uint64_t)lc * A.W;
    if ((int)lane < nw) grm[lane] = rk[lane];
    if (lane == 0) {
      const uint32_t j = cum[kReachWords] + (uint32_t)P.n_live;
      A.dcount[lc] = j;
      A.seg_begin[lc] = (int32_t)((uint64_t)lc * A.S);
      A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S + j);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// k_dirty_big (parents beyond 256 slots): one warp per candidate walks the topological slots
// 32 at a time from its first touched slot.  Lane i holds slot 32w + i, which is dirty iff it
// is a seed (the node rewritten in place, an owner of a remapped ref) or one of its producers
// is dirty: producers in earlier windows are final (shared-memory mask), producers inside the
// window are resolved by iterating the window's ballot to a fixed point (the dirty set only
// grows).  Job indices are prefix popcounts (the running count + the window's ballot), so the
// jobs, their key sources and the removed ranks are emitted in the same pass, in the layout
// k_dirty_warp produces from reach rows (sources at the parent's ref offsets, output sources
// in outsrc).  The slot tables are the parent's (k_match), shared by its candidates through
// L1/L2; per window a lane issues independent loads only.  Dynamic shared memory per warp:
// dm[W], cum[W + 1], rk[W].
// ------------------------------------------------------------------------------------------

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_dirty_big(VArgs A) {
  extern __shared__ uint32_t db_smem[];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  const uint32_t W = A.W;
  uint32_t* dm = db_smem + (uint64_t)wid * (3 * W + 1);
  uint32_t* cum = dm + W;
  uint32_t* rk = cum + W + 1;
  const Geo& G = A.g;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t lc = blockIdx.x * WARPS + wid; lc < A.n; lc += gridDim.x * WARPS) {  // warp-uniform
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) {
      if (lane == 0) {
        A.dcount[lc] = 0;
        A.seg_begin[lc] = A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S);
      }
      continue;
    }
    const VPlan P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint32_t* ps = A.pscratch + (uint64_t)P.parent * A.pstride;
    const uint32_t* coff = ps + 2 * G.cap_nodes;
    const uint32_t* clist = coff + 2 * G.cap_nodes + 1;
    const uint32_t* tslot = clist + G.cap_refs;
    const uint32_t* s_v = tslot + G.cap_nodes;
    const uint32_t* s_pk = s_v + G.cap_nodes;
    const uint32_t* rslot = s_pk + G.cap_nodes;
    const uint32_t* psig = R.sig(G);
    const uint32_t* paux = R.aux(G);
    const uint32_t* pinoff = R.inoff(G);
    const uint32_t* pnin = R.nin(G);
    const uint32_t* prefs = R.refs(G);
    const uint32_t* srank = R.srank(G);
    const int pn = P.pn;
    const uint32_t nw = ((uint32_t)pn + 31) >> 5;
    for (uint32_t w = lane; w < nw; w += 32) dm[w] = rk[w] = cum[w] = 0;
    __syncwarp();
    const int ms = P.mod >= 0 ? (int)tslot[P.mod] : -1;
    const int ds0 = P.drop0 >= 0 ? (int)tslot[P.drop0] : -1, ds1 = P.drop1 >= 0 ? (int)tslot[P.drop1] : -1;
    if (ms >= 0 && lane == 0) atomicOr(&dm[ms >> 5], 1u << (ms & 31));
    uint32_t rf[2] = {0xffffffffu, 0xffffffffu};
    for (int k = 0; k < P.n_rm; ++k) {  // owners of remapped refs (dropped nodes excluded)
      const uint32_t from = P.rm_from[k], p = from >> 8;
      rf[k] = (tslot[p] << 8) | (from & 255u);
      for (uint32_t x = coff[p] + lane; x < coff[p + 1]; x += 32) {
        const uint32_t q = clist[x];
        if ((int)q == P.drop0 || (int)q == P.drop1) continue;
        bool hit = false;
        for (uint32_t r = pinoff[q]; r < pinoff[q] + pnin[q]; ++r) hit |= prefs[r] == from;
        if (hit) {
          const uint32_t t = tslot[q];
          atomicOr(&dm[t >> 5], 1u << (t & 31));
        }
      }
    }
    __syncwarp();
    const int ins = P.ins_slot;
    auto popc_below = [&](uint32_t t) -> uint32_t {  // dirty slots before t (t = pn: all; set at the end)
      return t >= (uint32_t)pn ? cum[nw] : cum[t >> 5] + __popc(dm[t >> 5] & ((1u << (t & 31)) - 1u));
    };
    auto dirty_at = [&](uint32_t t) -> bool { return (dm[t >> 5] >> (t & 31)) & 1u; };
    auto fidx = [&](uint32_t t) -> uint32_t { return popc_below(t) + ((int)t > ins && ins >= 0 ? P.n_live : 0); };
    auto fnew = [&](int k) -> uint32_t {
      return popc_below((uint32_t)(ins + (P.ins_after ? 1 : 0))) + (k == 1 ? (uint32_t)P.live[0] : 0u);
    };
    auto src_pos = [&](uint32_t ref) -> uint32_t {  // a ref in parent-position space -> key source
      const uint32_t p = ref >> 8, port = ref & 255u;
      if ((int)p >= pn) return kFresh | (port << 23) | fnew((int)p - pn);
      const uint32_t t = tslot[p];
      return dirty_at(t) ? (kFresh | (port << 23) | fidx(t)) : ((port << 23) | p);
    };
    Job* jobs = A.jobs + (uint64_t)lc * A.S;
    uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    // levels of the key DAG for k_keys_wide: by job in jlvl, by slot in the (step-mode idle) jv row
    const bool levels = A.jlvl != nullptr;
    uint16_t* lv = levels ? A.jlvl + (uint64_t)lc * A.S : nullptr;
    uint32_t* plv = A.jv + (uint64_t)lc * A.S;
    auto new_level = [&](int k) -> uint32_t {  // a new node: 1 + its producer's level if that is fresh
      uint32_t extra = 0, p = P.new_ref[k] >> 8;
      if ((int)p >= pn) {  // the other new node
        extra = 1;
        p = P.new_ref[(int)p - pn] >> 8;
        if ((int)p >= pn) return extra;
      }
      const uint32_t tq = tslot[p];
      return extra + (dirty_at(tq) ? plv[tq] + 1u : 0u);
    };
    uint32_t run = 0;
    const uint32_t w0 = (uint32_t)max(P.first, 0) >> 5;
    // the first window's slot table entries, then one window ahead
    uint32_t t = 32u * w0 + lane;
    uint32_t pk = t < (uint32_t)pn ? s_pk[t] : 0u;
    for (uint32_t w = w0; w < nw; ++w) {
      const bool live = t < (uint32_t)pn;
      const uint32_t tn = t + 32u;
      const uint32_t pk_next = tn < (uint32_t)pn ? s_pk[tn] : 0u;
      const uint32_t r0 = pk & 0xffffffu, nr = pk >> 24;
      const bool dropped = (int)t == ds0 || (int)t == ds1;
      const uint32_t word = dm[w];
      bool d = false;
      uint32_t inmask = 0;
      if (live && !dropped) {
        d = (word >> lane) & 1u;
        for (uint32_t k = 0; k < nr && !d; ++k) {
          const uint32_t rsl = rslot[r0 + k], tp = rsl >> 8;
          if (rsl == rf[0] || rsl == rf[1]) continue;  // remapped: its owner is a seed
          if ((tp >> 5) == w) inmask |= 1u << (tp & 31u);
          else d = dirty_at(tp);
        }
      }
      uint32_t cur = __ballot_sync(full, d);
      while (true) {  // producers inside the window: to the fixed point
        d = d || (inmask & cur) != 0u;
        const uint32_t nxt = __ballot_sync(full, d);
        if (nxt == cur) break;
        cur = nxt;
      }
      if (lane == 0) {
        dm[w] = cur;
        cum[w] = run;
      }
      __syncwarp();
      const uint32_t j = run + __popc(cur & lt) + ((int)t > ins && ins >= 0 ? (uint32_t)P.n_live : 0u);
      // level: the deepest fresh producer + 1.  A producer in this window is resolved by the
      // shuffle pass below (in[k]: lanes whose level + k + 1 bounds this one: k = 1, 2 through
      // one or two new nodes, whose level is their producer's + 1)
      uint32_t lvl = 0, in1 = 0, in2 = 0, in3 = 0;
      if (d) {
        const uint32_t v = s_v[t];
        auto dep = [&](uint32_t tq, uint32_t plus) {
          if ((tq >> 5) == w) {
            const uint32_t bit = 1u << (tq & 31u);
            if (plus == 1u) in1 |= bit;
            else if (plus == 2u) in2 |= bit;
            else in3 |= bit;
          } else {
            lvl = max(lvl, plv[tq] + plus);
          }
        };
        auto lvl_of = [&](uint32_t tq) { dep(tq, 1u); };
        auto new_dep = [&](int k) {  // a fresh new node as a producer: its level is its producer's + 1
          uint32_t plus = 2, p = P.new_ref[k] >> 8;
          if ((int)p >= pn) {  // the other new node
            plus = 3;
            p = P.new_ref[(int)p - pn] >> 8;
            if ((int)p >= pn) {
              lvl = max(lvl, 2u);
              return;
            }
          }
          const uint32_t tq = tslot[p];
          if (dirty_at(tq)) dep(tq, plus);
          else lvl = max(lvl, plus - 1u);
        };
        for (uint32_t k = 0; k < nr; ++k) {
          const uint32_t rsl = rslot[r0 + k];
          uint32_t sv;
          if (rsl == rf[0] || rsl == rf[1]) {  // the owner now consumes another producer (a remap)
            const uint32_t to = rsl == rf[0] ? P.rm_to[0] : P.rm_to[1];
            sv = src_pos(to);
            if (levels) {
              const uint32_t p = to >> 8;
              if ((int)p >= pn) new_dep((int)p - pn);
              else if (sv & kFresh) lvl_of(tslot[p]);
            }
          } else {
            const uint32_t tp = rsl >> 8, port = rsl & 255u;
            const bool f = dirty_at(tp);
            sv = f ? (kFresh | (port << 23) | fidx(tp)) : ((port << 23) | (prefs[r0 + k] >> 8));
            if (levels && f) lvl_of(tp);
          }
          rs[r0 + k] = sv;
        }
        const bool m = (int)t == ms;
        jobs[j] = Job{m ? P.mod_sig : psig[v], m ? P.mod_aux : paux[v], r0, nr};
        const uint32_t k = srank[v];
        atomicOr(&rk[k >> 5], 1u << (k & 31));
      }
      if (levels) {
        // in-window producers sit on lower lanes: one ascending pass over the lanes some lane
        // depends on (a producer's own in-window producers are lower still, so it is final
        // when it is read)
        for (uint32_t u = __reduce_or_sync(full, in1 | in2 | in3); u; u &= u - 1u) {  // warp-uniform
          const int b = __ffs(u) - 1;
          const uint32_t x = __shfl_sync(full, lvl, b);
          if ((in1 >> b) & 1u) lvl = max(lvl, x + 1u);
          if ((in2 >> b) & 1u) lvl = max(lvl, x + 2u);
          if ((in3 >> b) & 1u) lvl = max(lvl, x + 3u);
        }
        if (d) {
          plv[t] = lvl;
          lv[j] = (uint16_t)min(lvl, 65535u);
        }
      }
      run += __popc(cur);
      t = tn;
      pk = pk_next;
    }
    if (lane == 0) cum[nw] = run;
    __syncwarp();
    const uint32_t pref = R.h().n_refs;
    if (lane < 2 && P.live[lane]) {  // the new nodes, exempt from the remap (rules.py:186-188)
      rs[pref + lane] = src_pos(P.new_ref[lane]);
      jobs[fnew((int)lane)] = Job{P.new_sig[lane], P.new_aux[lane], pref + lane, 1u};
      if (levels) lv[fnew((int)lane)] = (uint16_t)min(new_level((int)lane), 65535u);
    }
    if (lane == 0) {
      if (P.drop0 >= 0) atomicOr(&rk[srank[P.drop0] >> 5], 1u << (srank[P.drop0] & 31));
      if (P.drop1 >= 0) atomicOr(&rk[srank[P.drop1] >> 5], 1u << (srank[P.drop1] & 31));
    }
    const uint32_t* pouts = R.outs(G);
    uint32_t* os = A.outsrc + (uint64_t)lc * A.Os;
    uint32_t o_first = 0xffffffffu;
    for (int o = lane; o < R.h().n_out; o += 32) {
      const uint32_t ref = pouts[o], sv = src_pos(vremap(P, ref));
      os[o] = sv;
      if (sv != (((ref & 255u) << 23) | (ref >> 8))) o_first = min(o_first, (uint32_t)o);  // not the parent's own key
    }
    if (A.pfx_first) {
      o_first = __reduce_min_sync(full, o_first);
      if (lane == 0) A.pfx_first[lc] = min(o_first, (uint32_t)R.h().n_out);
    }
    __syncwarp();
    uint32_t* grm = A.rmask + (uint64_t)lc * A.W;
    for (uint32_t w = lane; w < nw; w += 32) grm[w] = rk[w];
    if (lane == 0) {
      const uint32_t j = run + (uint32_t)P.n_live;
      A.dcount[lc] = j;
      A.seg_begin[lc] = (int32_t)((uint64_t)lc * A.S);
      A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S + j);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// message assembly: a byte stream packed into aligned 64-bit words of a per-thread column
// (word q of thread t at col[q * BT]), so the message can be indexed dynamically while the
// compression itself runs on registers
// ------------------------------------------------------------------------------------------

template <int BT>
struct WordSink {
  uint64_t* col;
  uint64_t acc;
  uint32_t accb;  // bytes pending in acc (0..7)
  uint32_t q;     // words written
  __device__ __forceinline__ void init(uint64_t* c) {
    col = c;
    acc = 0;
    accb = 0;
    q = 0;
  }
  // append nb (1..8) bytes given as the low bytes of w (higher bytes zero)
  __device__ __forceinline__ void push(uint64_t w, uint32_t nb) {
    if (accb == 0) {
      if (nb == 8) {
        col[(q++) * BT] = w;
      } else {
        acc = w;
        accb = nb;
      }
      return;
    }
    acc |= w << (8 * accb);
    const uint32_t tot = accb + nb;
    if (tot >= 8) {
      col[(q++) * BT] = acc;
      acc = w >> (8 * (8 - accb));
      accb = tot - 8;
    } else {
      accb = tot;
    }
  }
  __device__ __forceinline__ void flush() {
    if (accb) {
      col[(q++) * BT] = acc;
      acc = 0;
      accb = 0;
    }
  }
};

__device__ __forceinline__ uint64_t port_be(uint32_t port) { return (uint64_t)((port >> 8) & 255u) | ((uint64_t)(port & 255u) << 8); }

// Message of a non-input job with <= 2 inputs, written straight into the column: the text
// words (8-byte aligned, zero padded in the table) are copied, and the suffix
//   digest[16] | key0[16] port0[2] | key1[16] port1[2]
// is built as aligned words in registers and funnel-shifted by the text's tail length.
// Returns the number of words written (ceil(len / 8)).
template <int BT>
__device__ __forceinline__ uint32_t msg_fast(uint64_t* col, const uint64_t* tw, uint32_t tlen, uint64_t d0, uint64_t d1,
                                             uint32_t nin, uint64_t k00, uint64_t k01, uint32_t p0, uint64_t k10,
                                             uint64_t k11, uint32_t p1) {
  const uint32_t fw = tlen >> 3, r = tlen & 7u;
#pragma unroll 4
  for (uint32_t i = 0; i < fw; ++i) col[i * BT] = __ldg(tw + i);
  uint64_t sw[7];
  sw[0] = d0;
  sw[1] = d1;
  sw[2] = nin > 0 ? k00 : 0;
  sw[3] = nin > 0 ? k01 : 0;
  const uint64_t pb0 = nin > 0 ? port_be(p0) : 0, pb1 = nin > 1 ? port_be(p1) : 0;
  const uint64_t a0 = nin > 1 ? k10 : 0, a1 = nin > 1 ? k11 : 0;
  sw[4] = pb0 | (a0 << 16);
  sw[5] = (a0 >> 48) | (a1 << 16);
  sw[6] = (a1 >> 48) | (pb1 << 16);
  const uint32_t len = tlen + 16u + 18u * nin;
  const uint32_t nout = ((len + 7u) >> 3) - fw;  // words from the tail word on
  const uint64_t tail = r ? __ldg(tw + fw) : 0ull;
  const uint32_t sl = 8u * r, sr = 64u - sl;
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j) {
    if (j < nout) {
      const uint64_t lo = j == 0 ? tail : (r ? sw[j - 1] >> sr : 0ull);
      const uint64_t hi = j < 7 ? sw[j] << sl : 0ull;
      col[(fw + j) * BT] = lo | hi;
    }
  }
  return fw + nout;
}

__device__ __forceinline__ void b2b_start(uint64_t* h, int outlen) {
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = b2b_iv(i);
  h[0] ^= 0x01010000ULL ^ (uint64_t)outlen;
}

// node key of a job too long for the fast path (rare: many-input concats); streaming BLAKE2b
struct TextTables {  // what job_key_slow reads, by value (a Tables& copies the parameter block to the stack)
  const uint8_t* sig_text;
  const uint32_t *sig_text_off, *sig_text_len;
  const uint8_t* names;
  const uint32_t *name_off, *name_len;
  const uint64_t* ws_digest;
};
__device__ __forceinline__ TextTables text_tables(const Tables& T) {
  return TextTables{T.sig_text, T.sig_text_off, T.sig_text_len, T.names, T.name_off, T.name_len, T.ws_digest};
}
struct Key128 {
  uint64_t a, b;
};

__device__ __noinline__ Key128 job_key_slow(const TextTables T, const Job jb, const uint32_t* rs, const uint64_t* pkeys,
                                            const uint64_t* fresh) {
  B2b st;
  st.init(16);
  const uint32_t off = T.sig_text_off[jb.sig], len = T.sig_text_len[jb.sig];
  const uint64_t* tw = reinterpret_cast<const uint64_t*>(T.sig_text + off);
  for (uint32_t i = 0; i < (len >> 3); ++i) st.word_le(tw[i]);
  const uint8_t* tail = T.sig_text + off + 8 * (len >> 3);
  for (uint32_t i = 0; i < (len & 7u); ++i) st.byte(tail[i]);
  const bool input = jb.nin & 0x80000000u;
  if (input) {
    const uint8_t* nm = T.names + T.name_off[jb.aux];
    for (uint32_t i = 0; i < T.name_len[jb.aux]; ++i) st.byte(nm[i]);
  }
  const uint32_t ws = input ? 0u : jb.aux;
  st.word_le(T.ws_digest[2 * ws]);
  st.word_le(T.ws_digest[2 * ws + 1]);
  for (uint32_t k = 0; k < (input ? 0u : jb.nin); ++k) {
    const uint32_t sv = rs[jb.roff + k];
    const uint32_t idx = sv & 0x7fffffu, port = (sv >> 23) & 255u;
    const uint64_t* kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
    st.word_le(kp[0]);
    st.word_le(kp[1]);
    st.u16_be(port);
  }
  st.final();
  return Key128{st.h[0], st.h[1]};
}

// ------------------------------------------------------------------------------------------
// k_keys
// ------------------------------------------------------------------------------------------

template <int BT>
__global__ void __launch_bounds__(BT, EF_KEYS_MINB) k_keys(VArgs A) {
  __shared__ uint64_t msg[kKeyMaxW * BT];
  const Geo& G = A.g;
  const Tables& T = A.T;
  uint64_t* col = msg + threadIdx.x;
  for (uint32_t l = blockIdx.x * BT + threadIdx.x; l < A.n; l += gridDim.x * BT) {
    const uint32_t lc = A.order[l];
    const uint32_t d = A.dcount[lc];
    if (d == 0 || (A.wide_min && d >= A.wide_min)) continue;  // (the wide ones: k_keys_wide)
    const uint32_t c = A.c0 + lc;
    const uint64_t* pkeys = A.full ? nullptr : Rec{reinterpret_cast<char*>(A.parent_addr[A.plan[c].parent])}.keys(G);
    const Job* jobs = A.jobs + (uint64_t)lc * A.S;
    const uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    uint64_t* skey = A.skey + (uint64_t)lc * A.S;
    uint32_t ncomp = 0;
    uint64_t last0 = 0, last1 = 0;
    // the next job's descriptor and text metadata are fetched one job ahead (their dependent
    // loads run under the current compression)
    Job jn = jobs[0];
    uint32_t tl_n = T.sig_text_len[jn.sig], to_n = T.sig_text_off[jn.sig];
    for (uint32_t jj = 0; jj < d; ++jj) {
      const Job jb = jn;
      const uint32_t tlen = tl_n, toff = to_n;
      if (jj + 1 < d) jn = jobs[jj + 1];
      const bool input = jb.nin & kInputJob;
      const uint32_t nin = input ? 0u : jb.nin;
      const uint32_t nlen = input ? T.name_len[jb.aux] : 0u;
      const uint32_t len = tlen + nlen + 16u + 18u * nin;
      uint64_t h[8];
      if (len > 8u * kKeyMaxW) {
        const Key128 ks = job_key_slow(text_tables(T), jb, rs, pkeys, fresh);
        h[0] = ks.a;
        h[1] = ks.b;
      } else {
        const uint64_t* tw = reinterpret_cast<const uint64_t*>(T.sig_text + toff);
        const uint32_t ws = input ? kEmptyWset : jb.aux;
        auto src = [&](uint32_t k, uint64_t& k0, uint64_t& k1) -> uint32_t {
          const uint32_t sv = rs[jb.roff + k];
          const uint32_t idx = sv & 0x7fffffu;
          if ((sv & kFresh) && idx + 1 == jj) {  // the previous job's key, still in registers
            k0 = last0;
            k1 = last1;
          } else {
            const uint64_t* kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
            k0 = kp[0];
            k1 = kp[1];
          }
          return (sv >> 23) & 255u;
        };
        uint32_t nw;
        if (!input && nin <= 2u) {
          uint64_t k00 = 0, k01 = 0, k10 = 0, k11 = 0;
          uint32_t p0 = 0, p1 = 0;
          if (nin > 0u) p0 = src(0, k00, k01);
          if (nin > 1u) p1 = src(1, k10, k11);
          nw = msg_fast<BT>(col, tw, tlen, __ldg(T.ws_digest + 2 * ws), __ldg(T.ws_digest + 2 * ws + 1), nin, k00, k01,
                            p0, k10, k11, p1);
        } else {
          WordSink<BT> sk;
          sk.init(col);
          const uint32_t full = tlen >> 3;
          for (uint32_t i = 0; i < full; ++i) sk.push(__ldg(tw + i), 8);
          if (tlen & 7u) sk.push(__ldg(tw + full), tlen & 7u);
          if (input) {  // graph.py:534-535: the input's name follows its signature text
            const uint8_t* nm = T.names + T.name_off[jb.aux];
            for (uint32_t i = 0; i < nlen; ++i) sk.push(nm[i], 1);
          }
          sk.push(__ldg(T.ws_digest + 2 * ws), 8);
          sk.push(__ldg(T.ws_digest + 2 * ws + 1), 8);
          for (uint32_t k = 0; k < nin; ++k) {
            uint64_t k0, k1;
            const uint32_t port = src(k, k0, k1);
            sk.push(k0, 8);
            sk.push(k1, 8);
            sk.push(port_be(port), 2);
          }
          sk.flush();
          nw = sk.q;
        }
        const uint32_t nb = (len + 127u) >> 7;
        for (uint32_t q = nw; q < 16u * nb; ++q) col[q * BT] = 0;
        if (jj + 1 < d) {
          tl_n = T.sig_text_len[jn.sig];
          to_n = T.sig_text_off[jn.sig];
        }
        b2b_start(h, 16);
        ncomp += nb;
        for (uint32_t b = 0; b < nb; ++b)
          b2b_compress_col<BT>(h, col + 16 * b * BT, (uint64_t)min(len, 128u * (b + 1)), b + 1 == nb);
      }
      if (len > 8u * kKeyMaxW && jj + 1 < d) {
        tl_n = T.sig_text_len[jn.sig];
        to_n = T.sig_text_off[jn.sig];
      }
      fresh[2 * jj] = h[0];
      fresh[2 * jj + 1] = h[1];
      last0 = h[0];
      last1 = h[1];
      skey[jj] = B2b::bswap64(h[0]);
    }
    if (A.stats) atomicAdd(A.stats, (unsigned long long)ncomp);
  }
}

// ------------------------------------------------------------------------------------------
// k_keys_wide: one warp per candidate with many jobs (large graphs).  A candidate's node keys
// form a DAG: a job needs the keys of its fresh producers only.  k_dirty records each job's
// level (one past its deepest fresh producer); the warp counting-sorts its jobs by level and
// hashes a level at a time, 32 jobs per round, so a long dependency chain is no longer one
// thread's sequential walk (the tail that bounded k_keys on 5k-20k-node graphs).
// The candidate's skey row is scratch for the level sort until the keys are done.
// ------------------------------------------------------------------------------------------

#ifndef EF_WIDE_MINB  // CTAs per SM the wide-key kernel's register budget is sized for
#define EF_WIDE_MINB 1
#endif
template <int BT, int LPC>
__global__ void __launch_bounds__(BT, EF_WIDE_MINB) k_keys_wide(VArgs A) {
  constexpr int WPB = BT / 32;
  constexpr int GPW = 32 / LPC;  // candidates per warp
  __shared__ uint64_t msg[kKeyMaxW * BT];
  const Geo& G = A.g;
  const Tables& T = A.T;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const uint32_t sl = lane % LPC, grp = lane / LPC;
  const unsigned gmask = LPC == 32 ? 0xffffffffu : (((1u << LPC) - 1u) << (grp * LPC));
  uint64_t* col = msg + threadIdx.x;
  const unsigned full = 0xffffffffu;
  for (uint32_t base = (blockIdx.x * WPB + wid) * GPW; base < A.n; base += gridDim.x * WPB * GPW) {  // warp-uniform
    const uint32_t l = base + grp;
    const uint32_t lc = l < A.n ? A.order[l] : 0u;
    const uint32_t d = l < A.n ? A.dcount[lc] : 0u;
    const bool has = l < A.n && d >= A.wide_min;
    if (!__any_sync(full, has)) break;  // sorted by job count: the rest belong to k_keys
    uint32_t nl = 0, ncomp = 0;
    const uint32_t c = A.c0 + lc;
    const uint64_t* pkeys = nullptr;
    const uint16_t* lv = A.jlvl + (uint64_t)lc * A.S;
    uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    uint64_t* skey = A.skey + (uint64_t)lc * A.S;
    uint32_t* ord = reinterpret_cast<uint32_t*>(skey);  // [S] jobs by level
    uint32_t* cnt = ord + A.S;                          // [S] per level: count -> start -> end
    if (has) {  // group-uniform: the counting sort of the candidate's jobs by level
      pkeys = Rec{reinterpret_cast<char*>(A.parent_addr[A.plan[c].parent])}.keys(G);
      uint32_t L = 0;
      for (uint32_t j = sl; j < d; j += LPC) L = max(L, (uint32_t)lv[j]);
      L = __reduce_max_sync(gmask, L);
      if (L < 65535u && L >= d) {  // a level is at most the job count - 1: report, hash in job order
        if (sl == 0 && atomicOr(A.err, 16u) == 0u) {
          A.err[9] = lc;
          A.err[10] = d;
          A.err[11] = L;
        }
        L = 65535u;
      }
      nl = L + 1;
      if (L >= 65535u) {  // levels saturated (a > 65k-deep key chain): one job per "level", in index order
        nl = d;
        for (uint32_t x = sl; x < d; x += LPC) {
          ord[x] = x;
          cnt[x] = x + 1;
        }
        __syncwarp(gmask);
      } else {
        for (uint32_t x = sl; x < nl; x += LPC) cnt[x] = 0;
        __syncwarp(gmask);
        for (uint32_t j = sl; j < d; j += LPC) atomicAdd(&cnt[lv[j]], 1u);
        __syncwarp(gmask);
        uint32_t run = 0;
        for (uint32_t x0 = 0; x0 < nl; x0 += LPC) {
          const uint32_t x = x0 + sl;
          const uint32_t v = x < nl ? cnt[x] : 0u;
          uint32_t inc = v;
#pragma unroll
          for (int o = 1; o < LPC; o <<= 1) {
            const uint32_t y = __shfl_up_sync(gmask, inc, o, LPC);
            if ((int)sl >= o) inc += y;
          }
          if (x < nl) cnt[x] = run + inc - v;
          run += __shfl_sync(gmask, inc, LPC - 1, LPC);
        }
        __syncwarp(gmask);
        for (uint32_t j = sl; j < d; j += LPC) ord[atomicAdd(&cnt[lv[j]], 1u)] = j;
        __syncwarp(gmask);  // cnt[level] is now the end of the level's run in ord
      }
    }
    // rounds: a level's keys are visible to the next level's lanes after the round's
    // __syncwarp.  Lanes are dealt per round: every group first gets up to LPC lanes for its
    // current level's remaining jobs, the lanes still idle then go to the groups with more than
    // that (in group order), so a narrow level of one candidate lends its lanes to a wide level
    // of another (fixed LPC-lane groups left 7.4 of 32 lanes idle per instruction on DAG-20k).
    uint32_t lev = 0, pos = 0, e = has ? cnt[0] : 0u;  // the group's state, in each of its lanes
    const uint64_t pk_bits = reinterpret_cast<uint64_t>(pkeys);
    while (__any_sync(full, lev < nl)) {
      const uint32_t avail = lev < nl ? e - pos : 0u;
      uint32_t av[GPW], tb = 0, te = 0;
#pragma unroll
      for (int g = 0; g < GPW; ++g) {
        av[g] = __shfl_sync(full, avail, g * LPC);
        tb += min(av[g], (uint32_t)LPC);
      }
      // this lane's job: (group g, index within the level's remaining jobs k)
      int g_sel = -1;
      uint32_t k_sel = 0, taken_mine = 0;
      {
        uint32_t bpre = 0, epre = 0;
#pragma unroll
        for (int g = 0; g < GPW; ++g) {
          const uint32_t base = min(av[g], (uint32_t)LPC), extra = av[g] - base;
          const uint32_t room = 32u > tb + epre ? 32u - tb - epre : 0u;
          const uint32_t ex_taken = min(extra, room);
          if (lane >= bpre && lane < bpre + base) {
            g_sel = g;
            k_sel = lane - bpre;
          } else if (lane >= tb + epre && lane < tb + epre + ex_taken) {
            g_sel = g;
            k_sel = base + (lane - tb - epre);
          }
          if ((uint32_t)g == grp) taken_mine = base + ex_taken;
          bpre += base;
          epre += extra;
        }
        te = epre;
      }
      (void)te;
      // the selected group's candidate, parent keys and position (from its lanes)
      const int src_lane = (g_sel < 0 ? (int)grp : g_sel) * LPC;
      const uint32_t lc_g = __shfl_sync(full, lc, src_lane);
      const uint32_t pos_g = __shfl_sync(full, pos, src_lane);
      const uint64_t pk_g = ((uint64_t)__shfl_sync(full, (uint32_t)(pk_bits >> 32), src_lane) << 32) |
                            __shfl_sync(full, (uint32_t)pk_bits, src_lane);
      if (g_sel >= 0) {
        const uint64_t* pkeys = reinterpret_cast<const uint64_t*>(pk_g);
        const Job* jobs = A.jobs + (uint64_t)lc_g * A.S;
        const uint32_t* rs = A.refsrc + (uint64_t)lc_g * A.Rs;
        uint64_t* fresh = A.fresh + 2ull * lc_g * A.S;
        const uint32_t* ord = reinterpret_cast<const uint32_t*>(A.skey + (uint64_t)lc_g * A.S);
        const uint32_t jj = ord[pos_g + k_sel];
        const Job jb = jobs[jj];
        const bool input = jb.nin & kInputJob;
        const uint32_t nin = input ? 0u : jb.nin;
        const uint32_t tlen = T.sig_text_len[jb.sig];
        const uint32_t nlen = input ? T.name_len[jb.aux] : 0u;
        const uint32_t len = tlen + nlen + 16u + 18u * nin;
        uint64_t h0, h1;
        if (len > 8u * kKeyMaxW) {
          const Key128 ks = job_key_slow(text_tables(T), jb, rs, pkeys, fresh);
          h0 = ks.a;
          h1 = ks.b;
        } else {
          const uint64_t* tw = reinterpret_cast<const uint64_t*>(T.sig_text + T.sig_text_off[jb.sig]);
          const uint32_t ws = input ? kEmptyWset : jb.aux;
          auto src = [&](uint32_t k, uint64_t& k0, uint64_t& k1) -> uint32_t {
            const uint32_t sv = rs[jb.roff + k];
            const uint32_t idx = sv & 0x7fffffu;
            const uint64_t* kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
            k0 = kp[0];
            k1 = kp[1];
            return (sv >> 23) & 255u;
          };
          uint32_t nw;
          if (!input && nin <= 2u) {
            uint64_t k00 = 0, k01 = 0, k10 = 0, k11 = 0;
            uint32_t p0 = 0, p1 = 0;
            if (nin > 0u) p0 = src(0, k00, k01);
            if (nin > 1u) p1 = src(1, k10, k11);
            nw = msg_fast<BT>(col, tw, tlen, __ldg(T.ws_digest + 2 * ws), __ldg(T.ws_digest + 2 * ws + 1), nin, k00,
                              k01, p0, k10, k11, p1);
          } else {
            WordSink<BT> sk;
            sk.init(col);
            const uint32_t fw = tlen >> 3;
            for (uint32_t i = 0; i < fw; ++i) sk.push(__ldg(tw + i), 8);
            if (tlen & 7u) sk.push(__ldg(tw + fw), tlen & 7u);
            if (input) {  // graph.py:534-535: the input's name follows its signature text
              const uint8_t* nm = T.names + T.name_off[jb.aux];
              for (uint32_t i = 0; i < nlen; ++i) sk.push(nm[i], 1);
            }
            sk.push(__ldg(T.ws_digest + 2 * ws), 8);
            sk.push(__ldg(T.ws_digest + 2 * ws + 1), 8);
            for (uint32_t k = 0; k < nin; ++k) {
              uint64_t k0, k1;
              const uint32_t port = src(k, k0, k1);
              sk.push(k0, 8);
              sk.push(k1, 8);
              sk.push(port_be(port), 2);
            }
            sk.flush();
            nw = sk.q;
          }
          const uint32_t nb = (len + 127u) >> 7;
          for (uint32_t q = nw; q < 16u * nb; ++q) col[q * BT] = 0;
          uint64_t h[8];
          b2b_start(h, 16);
          ncomp += nb;
          for (uint32_t bk = 0; bk < nb; ++bk)
            b2b_compress_col_pf<BT>(h, col + 16 * bk * BT, (uint64_t)min(len, 128u * (bk + 1)), bk + 1 == nb);
          h0 = h[0];
          h1 = h[1];
        }
        fresh[2 * jj] = h0;
        fresh[2 * jj + 1] = h1;
      }
      if (lev < nl) {
        pos += taken_mine;
        if (pos >= e) {
          pos = e;
          if (++lev < nl) e = cnt[lev];
        }
      }
      __syncwarp();
    }
    if (has) {
      for (uint32_t j = sl; j < d; j += LPC) {  // the sort records (the level scratch is dead)
        skey[j] = B2b::bswap64(fresh[2 * j]);
      }
    }
    ncomp = __reduce_add_sync(full, ncomp);
    if (A.stats && lane == 0) atomicAdd(A.stats, (unsigned long long)ncomp);
  }
}

// Sort every candidate's fresh keys: one warp per candidate, bitonic network over M
// (a power of two >= the step's row length) in shared memory on the keys' first word
// (big endian), carrying the job index; runs of equal first words (a 2^-64 event unless
// the keys are identical) are then ordered by the second word.
template <int M, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_sortkeys(VArgs A) {
  __shared__ uint64_t sk_all[WARPS * M];
  __shared__ uint32_t sv_all[WARPS * M];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t* sk = sk_all + w * M;
  uint32_t* sv = sv_all + w * M;
  for (uint32_t lc = blockIdx.x * WARPS + w; lc < A.n; lc += gridDim.x * WARPS) {
    const uint32_t d = A.dcount[lc];
    if (d == 0) continue;
    uint32_t m = 2;
    while (m < d) m <<= 1;
    // sort value: the key's first 4 bytes (big endian) above the job index
    const uint64_t* src = A.skey + (uint64_t)lc * A.S;
    for (uint32_t i = lane; i < m; i += 32) sk[i] = i < d ? ((src[i] >> 32) << 32) | i : ~0ULL;
    __syncwarp();
    for (uint32_t k = 2; k <= m; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = lane; i < m; i += 32) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const uint64_t a = sk[i], b = sk[ixj];
            if ((a > b) == ((i & k) == 0)) {
              sk[i] = b;
              sk[ixj] = a;
            }
          }
        }
        __syncwarp();
      }
    }
    for (uint32_t i = lane; i < d; i += 32) sv[i] = (uint32_t)sk[i];
    __syncwarp();
    // equal first 4 bytes (p ~ d^2 / 2^33 per candidate): order those runs by the full key
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    bool tie = false;
    for (uint32_t i = lane; i + 1 < d; i += 32) tie |= (sk[i] >> 32) == (sk[i + 1] >> 32);
    if (__any_sync(0xffffffffu, tie)) {
      if (lane == 0) {
        auto less = [&](uint32_t x, uint32_t y) {
          const uint64_t a0 = B2b::bswap64(fresh[2 * x]), b0 = B2b::bswap64(fresh[2 * y]);
          if (a0 != b0) return a0 < b0;
          return B2b::bswap64(fresh[2 * x + 1]) < B2b::bswap64(fresh[2 * y + 1]);
        };
        for (uint32_t i = 0; i + 1 < d;) {
          uint32_t e = i + 1;
          while (e < d && (sk[e] >> 32) == (sk[i] >> 32)) ++e;
          for (uint32_t x = i + 1; x < e; ++x) {
            const uint32_t v = sv[x];
            uint32_t y = x;
            while (y > i && less(v, sv[y - 1])) {
              sv[y] = sv[y - 1];
              --y;
            }
            sv[y] = v;
          }
          i = e;
        }
      }
      __syncwarp();
    }
    uint64_t* dst = A.fresh_sorted + 2ull * lc * A.S;
    uint32_t* dsv = A.sval_sorted + (uint64_t)lc * A.S;
    for (uint32_t i = lane; i < d; i += 32) {
      const uint32_t v = sv[i];
      dst[2 * i] = fresh[2 * v];
      dst[2 * i + 1] = fresh[2 * v + 1];
      if (A.full) dsv[i] = v;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// k_keys_quad: the same jobs with four lanes per candidate, for launches too small to fill
// the GPU (uploads, kept records, single-parent expansions): lane q of a quad holds column q
// of the BLAKE2b state (v[q], v[q+4], v[q+8], v[q+12]) and computes one G of every half
// round; quad shuffles rotate b/c/d between the column and the diagonal step.  The message
// is assembled by the quad's lane 0 into the quad's shared-memory column.
// ------------------------------------------------------------------------------------------

// message-word indices of quad lane q in round r: bits [16k + 4q, +4) of kQuadSigma[r % 10]
// are sigma[r][2q + {0, 1, 8, 9}[k]] (the column and diagonal G's of the lane)
__constant__ uint64_t kQuadSigma[10] = {
    0xfdb9eca875316420ull, 0x372c5b016f8ad94eull, 0x416e973ad208f5cbull, 0x80a6f452ec19bd37ull,
    0xd8c136bef470a259ull, 0x9e5d1f743bac8062ull, 0xb2378960adf54e1cull, 0xa64028f591eb3c7dull,
    0x5472a1dc839f0be6ull, 0x0cebd39f5642178aull};

// One compression by the 4 lanes of a quad (lane q runs column G q and diagonal G q, the
// state rotates between them by shuffles).  The rounds are unrolled with the lane's message
// words of round r + 1 loaded during round r, so the chain is the G's and the shuffles only.
template <int QN>
__device__ __forceinline__ void b2b_compress_quad(uint64_t& h0, uint64_t& h1, const uint64_t* col, uint64_t t,
                                                  bool last, int q, int qbase) {
  uint64_t a = h0, b = h1, c = b2b_iv(q), d = b2b_iv(4 + q);
  if (q == 0) d ^= t;
  if (q == 2 && last) d = ~d;
  const unsigned full = 0xffffffffu;
  const uint32_t sh = 4u * (uint32_t)q;
  uint64_t x0, y0, x1, y1;
  {
    const uint64_t w = 0xfdb9eca875316420ull >> sh;
    x0 = col[(w & 15u) * QN];
    y0 = col[((w >> 16) & 15u) * QN];
    x1 = col[((w >> 32) & 15u) * QN];
    y1 = col[((w >> 48) & 15u) * QN];
  }
#pragma unroll
  for (int r = 0; r < 12; ++r) {
    uint64_t nx0 = 0, ny0 = 0, nx1 = 0, ny1 = 0;
    if (r + 1 < 12) {
      const uint64_t w = kQuadSigma[(r + 1) % 10] >> sh;
      nx0 = col[(w & 15u) * QN];
      ny0 = col[((w >> 16) & 15u) * QN];
      nx1 = col[((w >> 32) & 15u) * QN];
      ny1 = col[((w >> 48) & 15u) * QN];
    }
    EF_B2B_G(a, b, c, d, x0, y0);
    b = __shfl_sync(full, b, qbase | ((q + 1) & 3));
    c = __shfl_sync(full, c, qbase | ((q + 2) & 3));
    d = __shfl_sync(full, d, qbase | ((q + 3) & 3));
    EF_B2B_G(a, b, c, d, x1, y1);
    b = __shfl_sync(full, b, qbase | ((q + 3) & 3));
    c = __shfl_sync(full, c, qbase | ((q + 2) & 3));
    d = __shfl_sync(full, d, qbase | ((q + 1) & 3));
    x0 = nx0;
    y0 = ny0;
    x1 = nx1;
    y1 = ny1;
  }
  h0 ^= a ^ c;
  h1 ^= b ^ d;
}

// what lane 0 of a quad knows about a job before assembling its message: fetched one job
// ahead, so the dependent loads (descriptor -> text metadata / key sources -> producer keys)
// run under the previous job's compression
struct QuadJob {
  Job jb;
  uint32_t tlen, toff;
  uint32_t sv0, sv1;            // key sources of inputs 0 and 1
  uint64_t k00, k01, k10, k11;  // their keys, unless they are the previous job's
};

template <int BT>
__global__ void __launch_bounds__(BT) k_keys_quad(VArgs A) {
  constexpr int QN = BT / 4;  // quads per block
  __shared__ uint64_t msg[kKeyMaxW * QN];
  const Geo& G = A.g;
  const Tables& T = A.T;
  const int q = threadIdx.x & 3, quad = threadIdx.x >> 2;
  const int qbase = (threadIdx.x & 31) & ~3;
  uint64_t* col = msg + quad;
  const uint32_t nq = (A.n + QN - 1) / QN * QN;  // whole blocks iterate together
  for (uint32_t l = blockIdx.x * QN + quad; l < nq; l += gridDim.x * QN) {
    const bool live = l < A.n;
    const uint32_t lc = live ? A.order[l] : 0;
    uint32_t d = live ? A.dcount[lc] : 0;
    if (A.wide_min && d >= A.wide_min) d = 0;  // k_keys_wide's
    const uint32_t dmax = __reduce_max_sync(0xffffffffu, d);  // lanes of the warp loop together
    const uint32_t c = A.c0 + lc;
    const uint64_t* pkeys =
        (A.full || !live) ? nullptr : Rec{reinterpret_cast<char*>(A.parent_addr[A.plan[c].parent])}.keys(G);
    const Job* jobs = A.jobs + (uint64_t)lc * A.S;
    const uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    uint64_t* skey = A.skey + (uint64_t)lc * A.S;
    auto key_of = [&](uint32_t sv, uint64_t& k0, uint64_t& k1) {
      const uint32_t idx = sv & 0x7fffffu;
      const uint64_t* kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
      k0 = kp[0];
      k1 = kp[1];
    };
    auto fwd = [](uint32_t sv, uint32_t j) { return (sv & kFresh) && (sv & 0x7fffffu) + 1 == j; };
    auto stage1 = [&](QuadJob& J, const Job jb) {  // descriptor -> text metadata + key sources
      J.jb = jb;
      J.tlen = T.sig_text_len[jb.sig];
      J.toff = T.sig_text_off[jb.sig];
      const uint32_t nin = (jb.nin & kInputJob) ? 0u : jb.nin;
      J.sv0 = nin > 0 ? rs[jb.roff] : 0u;
      J.sv1 = nin > 1 ? rs[jb.roff + 1] : 0u;
    };
    auto stage2 = [&](QuadJob& J, uint32_t j) {  // producer keys other than job j - 1's
      const uint32_t nin = (J.jb.nin & kInputJob) ? 0u : J.jb.nin;
      J.k00 = J.k01 = J.k10 = J.k11 = 0;
      if (nin > 0 && !fwd(J.sv0, j)) key_of(J.sv0, J.k00, J.k01);
      if (nin > 1 && !fwd(J.sv1, j)) key_of(J.sv1, J.k10, J.k11);
    };
    QuadJob cur{}, nxt{};
    Job jnext{};
    if (q == 0 && d > 0) {
      stage1(cur, jobs[0]);
      stage2(cur, 0);
      if (d > 1) jnext = jobs[1];
    }
    uint64_t last0 = 0, last1 = 0;
    uint32_t ncomp = 0;
    for (uint32_t jj = 0; jj < dmax; ++jj) {
      const bool act = jj < d;
      uint32_t len = 0, nb = 0;
      bool slow = false;
      uint64_t sh0 = 0, sh1 = 0;
      if (act && q == 0) {
        const Job jb = cur.jb;
        const bool input = jb.nin & kInputJob;
        const uint32_t nin = input ? 0u : jb.nin;
        if (nin > 0 && fwd(cur.sv0, jj)) {
          cur.k00 = last0;
          cur.k01 = last1;
        }
        if (nin > 1 && fwd(cur.sv1, jj)) {
          cur.k10 = last0;
          cur.k11 = last1;
        }
        const bool more = jj + 1 < d;
        if (more) stage1(nxt, jnext);
        if (jj + 2 < d) jnext = jobs[jj + 2];
        const uint32_t nlen = input ? T.name_len[jb.aux] : 0u;
        len = cur.tlen + nlen + 16u + 18u * nin;
        if (len > 8u * kKeyMaxW) {
          const Key128 ks = job_key_slow(text_tables(T), jb, rs, pkeys, fresh);
          sh0 = ks.a;
          sh1 = ks.b;
          slow = true;
        } else {
          WordSink<QN> sk;
          sk.init(col);
          const uint64_t* tw = reinterpret_cast<const uint64_t*>(T.sig_text + cur.toff);
          const uint32_t fullw = cur.tlen >> 3;
          for (uint32_t i = 0; i < fullw; ++i) sk.push(__ldg(tw + i), 8);
          if (cur.tlen & 7u) sk.push(__ldg(tw + fullw), cur.tlen & 7u);
          const uint32_t ws = input ? kEmptyWset : jb.aux;
          if (input) {
            const uint8_t* nm = T.names + T.name_off[jb.aux];
            for (uint32_t i = 0; i < nlen; ++i) sk.push(nm[i], 1);
          }
          sk.push(__ldg(T.ws_digest + 2 * ws), 8);
          sk.push(__ldg(T.ws_digest + 2 * ws + 1), 8);
          for (uint32_t k = 0; k < nin; ++k) {
            uint64_t k0, k1;
            uint32_t sv;
            if (k == 0) {
              sv = cur.sv0;
              k0 = cur.k00;
              k1 = cur.k01;
            } else if (k == 1) {
              sv = cur.sv1;
              k0 = cur.k10;
              k1 = cur.k11;
            } else {
              sv = rs[jb.roff + k];
              if (fwd(sv, jj)) {
                k0 = last0;
                k1 = last1;
              } else {
                key_of(sv, k0, k1);
              }
            }
            sk.push(k0, 8);
            sk.push(k1, 8);
            sk.push(port_be((sv >> 23) & 255u), 2);
          }
          sk.flush();
          nb = (len + 127u) >> 7;
          for (uint32_t w = sk.q; w < 16u * nb; ++w) col[w * QN] = 0;
        }
        if (more) stage2(nxt, jj + 1);  // its loads run under the compression below
      }
      // broadcast the job shape within the quad, then compress cooperatively
      nb = __shfl_sync(0xffffffffu, nb, qbase);
      len = __shfl_sync(0xffffffffu, len, qbase);
      slow = __shfl_sync(0xffffffffu, (int)slow, qbase) != 0;
      __syncwarp();
      uint64_t h0 = b2b_iv(q), h1 = b2b_iv(4 + q);
      if (q == 0) h0 ^= 0x01010000ULL ^ 16ULL;
      const uint32_t nbmax = __reduce_max_sync(0xffffffffu, act && !slow ? nb : 0u);
      for (uint32_t bk = 0; bk < nbmax; ++bk) {
        const bool go = act && !slow && bk < nb;
        // every lane of the warp runs the shuffles; quads without a block keep their state
        uint64_t g0 = h0, g1 = h1;
        b2b_compress_quad<QN>(g0, g1, col + 16 * bk * QN, (uint64_t)min(len, 128u * (bk + 1)), bk + 1 == nb, q,
                              qbase);
        if (go) {
          h0 = g0;
          h1 = g1;
        }
      }
      // the 16-byte key is h[0] (lane 0) and h[1] (lane 1)
      uint64_t k0 = __shfl_sync(0xffffffffu, h0, qbase);
      uint64_t k1 = __shfl_sync(0xffffffffu, h0, qbase | 1);
      if (slow) {
        k0 = __shfl_sync(0xffffffffu, sh0, qbase);
        k1 = __shfl_sync(0xffffffffu, sh1, qbase);
      } else {
        sh0 = __shfl_sync(0xffffffffu, sh0, qbase);  // keep the shuffles warp-uniform
        sh1 = __shfl_sync(0xffffffffu, sh1, qbase);
      }
      if (act && q == 0) {
        fresh[2 * jj] = k0;
        fresh[2 * jj + 1] = k1;
        skey[jj] = B2b::bswap64(k0);
          ncomp += slow ? 0u : nb;
        if (jj + 1 < d) cur = nxt;
      }
      last0 = k0;
      last1 = k1;
      __syncwarp();
    }
    if (A.stats && q == 0 && live) atomicAdd(A.stats, (unsigned long long)ncomp);
  }
}

// Candidates ordered by job count, largest first (the lanes of a k_keys warp then run about
// the same number of compressions; k_keys_wide takes a prefix): a counting sort over the
// exact counts.  bins[S - count] is histogrammed, scanned by one CTA, then every candidate
// claims its position with one warp-aggregated atomic per distinct count in the warp.
__global__ void k_count_hist(const uint32_t* dcount, uint32_t n, uint32_t S, uint32_t* bins) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(bins + (S - min(dcount[i], S)), 1u);
}

template <int BT>
__global__ void __launch_bounds__(BT) k_count_scan(uint32_t* bins, uint32_t nb) {
  __shared__ uint32_t sh_scan[BT / 32 + 1];
  uint32_t run = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += BT) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? bins[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<BT>(v, &tot, sh_scan);
    if (b < nb) bins[b] = run + ex;
    run += tot;
    __syncthreads();
  }
}

__global__ void k_count_scatter(const uint32_t* dcount, uint32_t n, uint32_t S, uint32_t* bins, uint32_t* order) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t span = (n + 31) / 32 * 32;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < span; i += gridDim.x * blockDim.x) {
    const bool live = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (!live) continue;
    const uint32_t b = S - min(dcount[i], S);
    const unsigned peers = __match_any_sync(act, b);
    const uint32_t leader = (uint32_t)(__ffs(peers) - 1);
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(bins + b, (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    order[base + __popc(peers & ((1u << lane) - 1u))] = i;
  }
}

// Rows of more than 1024 fresh keys: one CTA per candidate (largest first), sorting on
// (first 4 key bytes, big endian) << 32 | job index by buckets: the keys are node-key hashes,
// uniform in their first bytes, so min(pow2(d), R) buckets on the top bits hold ~1-3 keys
// each -- a histogram, a block scan, a scatter and a per-bucket insertion sort: O(d) work and
// four barriers (bitonic runs and merges cost log^2 d stages: 21 of the 47 ms of the DAG-20k
// sort stage went there).  The sorted words live in shared memory up to R keys, beyond in the
// candidate's global sort row.  Runs of equal first 4 bytes (p ~ d^2 / 2^33 per candidate)
// are then ordered by the full key as in k_sortkeys, and the keys are gathered into
// fresh_sorted with 16-byte loads and coalesced 16-byte stores.  Dynamic shared memory: R
// words + R bucket counters.
// the end of a k_sortbig candidate: src holds (first 4 key bytes << 32 | job index) ascending;
// runs of equal first 4 bytes are ordered by the full key, then the keys are gathered into
// fresh_sorted (src may be shared or global memory)
template <int BT>
__device__ __forceinline__ void sort_finish(const VArgs& A, uint32_t lc, uint32_t d, uint64_t* src) {
  const uint32_t tid = threadIdx.x;
  const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
  int tie = 0;
  for (uint32_t i = tid; i + 1 < d; i += BT) tie |= (src[i] >> 32) == (src[i + 1] >> 32);
  if (__syncthreads_or(tie) && tid == 0) {
    auto less = [&](uint32_t x, uint32_t y) {
      const uint64_t a0 = B2b::bswap64(fresh[2 * x]), b0 = B2b::bswap64(fresh[2 * y]);
      if (a0 != b0) return a0 < b0;
      return B2b::bswap64(fresh[2 * x + 1]) < B2b::bswap64(fresh[2 * y + 1]);
    };
    for (uint32_t i = 0; i + 1 < d;) {
      uint32_t e = i + 1;
      while (e < d && (src[e] >> 32) == (src[i] >> 32)) ++e;
      for (uint32_t x = i + 1; x < e; ++x) {  // insertion sort of the run by the full key
        const uint64_t v = src[x];
        uint32_t y = x;
        while (y > i && less((uint32_t)v, (uint32_t)src[y - 1])) {
          src[y] = src[y - 1];
          --y;
        }
        src[y] = v;
      }
      i = e;
    }
  }
  __syncthreads();
  uint4* out = reinterpret_cast<uint4*>(A.fresh_sorted + 2ull * lc * A.S);
  const uint4* f4 = reinterpret_cast<const uint4*>(fresh);
  uint32_t* osv = A.sval_sorted + (uint64_t)lc * A.S;
  for (uint32_t i = tid; i < d; i += BT) {
    const uint32_t v = (uint32_t)src[i];
    out[i] = f4[v];
    if (A.full) osv[i] = v;
  }
  __syncthreads();
}

template <int BT>
__device__ __forceinline__ void block_excl_scan_inplace(uint32_t* cnt, uint32_t nb, uint32_t* wsum) {
  // each thread scans a contiguous stretch of nb / BT counters (nb is a power of two >= 32)
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t per = (nb + BT - 1) / BT;
  const uint32_t b0 = min(nb, tid * per), b1 = min(nb, b0 + per);
  uint32_t loc = 0;
  for (uint32_t b = b0; b < b1; ++b) loc += cnt[b];
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t v = lane < BT / 32 ? wsum[lane] : 0u, x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane < BT / 32) wsum[lane] = x - v;
  }
  __syncthreads();
  uint32_t run = wsum[w] + inc - loc;
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t c = cnt[b];
    cnt[b] = run;
    run += c;
  }
  __syncthreads();
}

template <int BT>
__global__ void __launch_bounds__(BT) k_sortbig(VArgs A, uint32_t R) {
  extern __shared__ uint64_t sbig[];
  __shared__ uint32_t wsum[BT / 32];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sbig + R);  // R bucket counters
  const uint32_t tid = threadIdx.x;
  for (uint32_t l = blockIdx.x; l < A.n; l += gridDim.x) {
    const uint32_t lc = A.order[l];
    const uint32_t d = A.dcount[lc];
    if (d == 0) continue;  // CTA-uniform
    const uint64_t* in = A.skey + (uint64_t)lc * A.S;  // first key words (big endian)
    // the sorted words: shared memory up to R keys, else the candidate's global sort row (L2)
    uint64_t* dst = d <= R ? sbig : const_cast<uint64_t*>(A.skey_sorted) + (uint64_t)lc * A.S;
    uint32_t nb = 32, lg = 5;
    while (nb < d && nb < R) nb <<= 1, ++lg;
    const uint32_t shift = 64 - lg;  // bucket = top lg bits of the first key word
    for (uint32_t b = tid; b < nb; b += BT) cnt[b] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < d; i += BT) atomicAdd(cnt + (uint32_t)(in[i] >> shift), 1u);
    __syncthreads();
    block_excl_scan_inplace<BT>(cnt, nb, wsum);
    for (uint32_t i = tid; i < d; i += BT) {
      const uint64_t v = in[i];
      const uint32_t pos = atomicAdd(cnt + (uint32_t)(v >> shift), 1u);
      dst[pos] = ((v >> 32) << 32) | i;
    }
    __syncthreads();
    // cnt[b] is now the end of bucket b: order each bucket (distinct values: the index)
    for (uint32_t b = tid; b < nb; b += BT) {
      const uint32_t e = cnt[b], s0 = b ? cnt[b - 1] : 0u;
      for (uint32_t x = s0 + 1; x < e; ++x) {
        const uint64_t v = dst[x];
        uint32_t y = x;
        while (y > s0 && dst[y - 1] > v) {
          dst[y] = dst[y - 1];
          --y;
        }
        dst[y] = v;
      }
    }
    __syncthreads();
    sort_finish<BT>(A, lc, d, dst);
  }
}

// ------------------------------------------------------------------------------------------
// k_digest
// ------------------------------------------------------------------------------------------

template <int BT>
__global__ void __launch_bounds__(BT) k_digest(VArgs A) {
  __shared__ uint64_t blk[16 * BT];
  const Geo& G = A.g;
  const Tables& T = A.T;
  uint64_t* col = blk + threadIdx.x;
  for (uint32_t lc = blockIdx.x * BT + threadIdx.x; lc < A.n; lc += gridDim.x * BT) {
    const uint32_t c = A.c0 + lc;
    VPlan P;
    if (A.full) {  // the record itself, everything fresh
      P.drop0 = P.drop1 = P.mod = -1;
      P.n_rm = 0;
      P.pn = 0;
      P.n_keep = Rec{reinterpret_cast<char*>(A.parent_addr[c])}.h().n;
      P.n_live = 0;
      P.parent = c;
    } else {
      if (A.res[c].flags & EF_F_INCOMPLETE) continue;
      P = A.plan[c];
    }
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pkeys = R.keys(G);
    const uint32_t* pouts = R.outs(G);
    const int n_out = R.h().n_out;
    const int pn = P.pn;
    const uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    const uint32_t d = A.dcount[lc];
    const uint32_t li = T.input_text_len;
    const uint32_t n_child = (uint32_t)(P.n_keep + P.n_live);
    const uint64_t len = (uint64_t)li + 18ull * n_out + 16ull * n_child;
    const uint32_t nblk = (uint32_t)((len + 127) >> 7);

    // generator state
    int phase = 0;
    uint32_t gi = 0, part = 0;
    uint64_t cw0 = 0, cw1 = 0;  // current key's raw words
    // merge streams: the parent's keys in sorted order minus the removed ranks, and the fresh
    // keys in sorted order; the heads are loaded as soon as a stream advances
    const uint64_t* pskeys = R.skeys(G);
    const uint32_t* rm = A.rmask + (uint64_t)lc * A.W;
    const uint64_t* fsk = A.fresh_sorted + 2ull * lc * A.S;
    uint32_t pi = 0, fk = 0, mw_idx = 0xffffffffu, mw = 0;
    uint64_t ph0 = 0, ph1 = 0, fh0 = 0, fh1 = 0;
    bool have_p = false, have_f = false;
    auto next_p = [&]() {
      while (pi < (uint32_t)pn) {
        if ((pi >> 5) != mw_idx) {
          mw_idx = pi >> 5;
          mw = rm[mw_idx];
        }
        const uint32_t rest = mw >> (pi & 31);
        if (rest == 0xffffffffu >> (pi & 31) && (pi | 31) < (uint32_t)pn) {  // whole tail removed
          pi = (pi | 31) + 1;
          continue;
        }
        if (!(rest & 1u)) break;
        ++pi;
      }
      have_p = pi < (uint32_t)pn;
      if (have_p) {
        ph0 = pskeys[2 * pi];
        ph1 = pskeys[2 * pi + 1];
      }
    };
    auto next_f = [&]() {
      have_f = fk < d;
      if (have_f) {
        fh0 = fsk[2 * fk];
        fh1 = fsk[2 * fk + 1];
      }
    };
    next_p();
    next_f();
    auto key_of = [&](uint32_t ref, uint64_t& w0, uint64_t& w1) {
      const uint32_t p = ref >> 8;
      const uint32_t fi = didx[p];
      if (fi) {
        w0 = fresh[2 * (fi - 1)];
        w1 = fresh[2 * (fi - 1) + 1];
      } else {
        w0 = pkeys[2 * p];
        w1 = pkeys[2 * p + 1];
      }
    };
    WordSink<BT> sk;
    sk.init(col);
    uint64_t h[8];
    b2b_start(h, 8);
    for (uint32_t b = 0; b < nblk; ++b) {
      sk.q = 0;
      while (sk.q < 16 && phase < 3) {
        if (phase == 0) {  // input declarations "name=dims;" (graph.py:542-543)
          if (gi * 8 < li) {
            const uint32_t nb = min(8u, li - gi * 8);
            sk.push(__ldg(A.input_words + gi), nb);
            ++gi;
          } else {
            phase = 1;
            gi = 0;
            part = 0;
          }
        } else if (phase == 1) {  // outputs: key + port (graph.py:544-546)
          if ((int)gi < n_out) {
            const uint32_t ref = vremap(P, pouts[gi]);
            if (part == 0) {
              key_of(ref, cw0, cw1);
              sk.push(cw0, 8);
              part = 1;
            } else if (part == 1) {
              sk.push(cw1, 8);
              part = 2;
            } else {
              sk.push(port_be(ref & 255u), 2);
              part = 0;
              ++gi;
            }
          } else {
            phase = 2;
            part = 0;
          }
        } else {  // sorted node keys (graph.py:547-548): merge of two ascending streams
          if (part == 0) {
            if (!have_p && !have_f) {
              phase = 3;
              continue;
            }
            bool take_f = !have_p;
            if (have_f && have_p) {
              const uint64_t a = B2b::bswap64(ph0), bb = B2b::bswap64(fh0);
              take_f = bb < a || (bb == a && B2b::bswap64(fh1) < B2b::bswap64(ph1));
            }
            if (take_f) {
              cw0 = fh0;
              cw1 = fh1;
              ++fk;
              next_f();
            } else {
              cw0 = ph0;
              cw1 = ph1;
              ++pi;
              next_p();
            }
            sk.push(cw0, 8);
            part = 1;
          } else {
            sk.push(cw1, 8);
            part = 0;
          }
        }
      }
      if (phase == 3) {
        sk.flush();
        for (uint32_t q = sk.q; q < 16; ++q) col[q * BT] = 0;
      }
      b2b_compress_col<BT>(h, col, len < 128ull * (b + 1) ? len : 128ull * (b + 1), b + 1 == nblk);
    }
    if (A.full) {
      if (A.hash_out) A.hash_out[c] = B2b::bswap64(h[0]);
    }
    else A.res[c].hash = B2b::bswap64(h[0]);
    if (A.stats) atomicAdd(A.stats + 1, (unsigned long long)nblk);
  }
}

// ------------------------------------------------------------------------------------------
// k_merge (rows of <= 32K keys): one warp per candidate builds the candidate's sorted key
// stream graph.py:547 sorted(keys) -- the fresh keys sorted in registers (bitonic network,
// K per lane, shuffles across lanes), the parent's pre-sorted keys compacted past the removed
// ranks (ballot), and both merged by rank (each key's position = own index + its count of
// smaller keys in the other list, by binary search in shared memory).  The stream is written
// contiguously, so k_digest_pm reads it with vector loads.
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ bool be_less(uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) {
  return a0 < b0 || (a0 == b0 && a1 < b1);
}

// sort the d (<= 32K) fresh keys of one candidate by the warp; writes them (big-endian word
// pairs) to sb in ascending order and returns whether two first words tied
template <int K>
__device__ __forceinline__ bool warp_sort_fresh(const uint64_t* fresh, uint32_t d, uint64_t* sb, int lane) {
  constexpr int M = 32 * K;
  uint64_t v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t i = lane * K + k;
    v[k] = i < d ? ((B2b::bswap64(fresh[2 * i]) >> 32) << 32) | i : ~0ULL;
  }
#pragma unroll
  for (int size = 2; size <= M; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j < K) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k & j) continue;
          const uint32_t i = lane * K + k;
          const bool up = (i & size) == 0;
          const uint64_t a = v[k], b = v[k | j];
          if ((a > b) == up) {
            v[k] = b;
            v[k | j] = a;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t i = lane * K + k;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[k], j / K);
          const bool up = (i & size) == 0, lower = (i & j) == 0;
          v[k] = (lower == up) ? (o < v[k] ? o : v[k]) : (o > v[k] ? o : v[k]);
        }
      }
    }
  }
  bool tie = false;
#pragma unroll
  for (int k = 0; k + 1 < K; ++k) tie |= (lane * K + k + 1 < d) && (v[k] >> 32) == (v[k + 1] >> 32);
  const uint64_t nxt = __shfl_down_sync(0xffffffffu, v[0], 1);
  tie |= lane < 31 && (uint32_t)((lane + 1) * K) < d && (v[K - 1] >> 32) == (nxt >> 32);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t i = lane * K + k;
    if (i < d) {
      const uint32_t jx = (uint32_t)v[k];
      sb[2 * i] = B2b::bswap64(fresh[2 * jx]);
      sb[2 * i + 1] = B2b::bswap64(fresh[2 * jx + 1]);
    }
  }
  return tie;
}

// smem bitonic sort of the packed values (first 4 key bytes << 32 | job) of one candidate, then
// its fresh keys in that order into sb; for candidates with more than 256 fresh keys
__device__ __forceinline__ bool warp_sort_fresh_smem(const uint64_t* fresh, uint32_t d, uint64_t* buf, uint64_t* sb,
                                                     int lane) {
  uint32_t m = 2;
  while (m < d) m <<= 1;
  for (uint32_t i = lane; i < m; i += 32) buf[i] = i < d ? ((B2b::bswap64(fresh[2 * i]) >> 32) << 32) | i : ~0ULL;
  __syncwarp();
  for (uint32_t k = 2; k <= m; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < m; i += 32) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = buf[i], b = buf[ixj];
          if ((a > b) == ((i & k) == 0)) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
  }
  bool tie = false;
  for (uint32_t i = lane; i + 1 < d; i += 32) tie |= (buf[i] >> 32) == (buf[i + 1] >> 32);
  // gather the keys in order (sb and buf may not alias: buf is the A area, sb the B area)
  for (uint32_t i = lane; i < d; i += 32) {
    const uint32_t jx = (uint32_t)buf[i];
    sb[2 * i] = B2b::bswap64(fresh[2 * jx]);
    sb[2 * i + 1] = B2b::bswap64(fresh[2 * jx + 1]);
  }
  return tie;
}

// dynamic shared memory: per warp two arrays of `rows` keys (A = parent, B = fresh)
template <int KMAX, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, EF_MERGE_MINB) k_merge(VArgs A, uint32_t rows) {
  extern __shared__ __align__(16) uint64_t merge_smem[];
  const Geo& G = A.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t* sa = merge_smem + (uint64_t)w * rows * 4;
  uint64_t* sb = sa + rows * 2;
  for (uint32_t lc = blockIdx.x * WARPS + w; lc < A.n; lc += gridDim.x * WARPS) {
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;
    const VPlan& P = A.plan[c];
    const int pn = P.pn;
    const uint32_t d = A.dcount[lc];
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    // 1) the fresh keys sorted, network sized to this candidate (warp-uniform branch)
    bool tie;
    if (d <= 32) tie = warp_sort_fresh<1>(fresh, d, sb, lane);
    else if (d <= 64 || KMAX < 4) tie = warp_sort_fresh<(KMAX < 2 ? KMAX : 2)>(fresh, d, sb, lane);
    else if (d <= 128 || KMAX < 8) tie = warp_sort_fresh<(KMAX < 4 ? KMAX : 4)>(fresh, d, sb, lane);
    else if (d <= 32u * KMAX) tie = warp_sort_fresh<KMAX>(fresh, d, sb, lane);
    else tie = warp_sort_fresh_smem(fresh, d, sa, sb, lane);
    __syncwarp();
    if (__any_sync(0xffffffffu, tie)) {  // p ~ d^2 / 2^33: insertion sort of the whole list by full key
      if (lane == 0) {
        for (uint32_t x = 1; x < d; ++x) {
          const uint64_t k0 = sb[2 * x], k1 = sb[2 * x + 1];
          uint32_t y = x;
          while (y > 0 && be_less(k0, k1, sb[2 * (y - 1)], sb[2 * (y - 1) + 1])) {
            sb[2 * y] = sb[2 * (y - 1)];
            sb[2 * y + 1] = sb[2 * (y - 1) + 1];
            --y;
          }
          sb[2 * y] = k0;
          sb[2 * y + 1] = k1;
        }
      }
      __syncwarp();
    }
    // 3) the parent's sorted keys minus removed ranks
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pskeys = R.skeys(G);
    const uint32_t* rm = A.rmask + (uint64_t)lc * A.W;
    uint32_t na = 0;
    for (int r0 = 0; r0 < pn; r0 += 32) {
      const int r = r0 + lane;
      const bool keep = r < pn && !((rm[r0 >> 5] >> lane) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const uint32_t at = na + __popc(bal & ((1u << lane) - 1u));
        sa[2 * at] = B2b::bswap64(pskeys[2 * r]);
        sa[2 * at + 1] = B2b::bswap64(pskeys[2 * r + 1]);
      }
      na += __popc(bal);
    }
    __syncwarp();
    // 4) merge by rank into the candidate's key stream (raw little-endian words)
    uint64_t* out = A.fresh_sorted + 2ull * lc * A.S;
    for (uint32_t i = lane; i < na; i += 32) {
      const uint64_t k0 = sa[2 * i], k1 = sa[2 * i + 1];
      uint32_t lo = 0, hi = d;  // fresh keys < this one
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (be_less(sb[2 * mid], sb[2 * mid + 1], k0, k1)) lo = mid + 1;
        else hi = mid;
      }
      out[2 * (i + lo)] = B2b::bswap64(k0);
      out[2 * (i + lo) + 1] = B2b::bswap64(k1);
    }
    for (uint32_t j = lane; j < d; j += 32) {
      const uint64_t k0 = sb[2 * j], k1 = sb[2 * j + 1];
      uint32_t lo = 0, hi = na;  // parent keys <= this one
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (!be_less(k0, k1, sa[2 * mid], sa[2 * mid + 1])) lo = mid + 1;
        else hi = mid;
      }
      out[2 * (j + lo)] = B2b::bswap64(k0);
      out[2 * (j + lo) + 1] = B2b::bswap64(k1);
    }
    __syncwarp();
  }
}

// The key stream of graphs beyond the shared-memory merge (rows > 256): the parent's sorted
// keys minus the removed ranks (A) merged with the candidate's sorted fresh keys (B, from the
// key sort), parent first on equal keys as in k_merge.  One warp per candidate, merge path:
// lane k finds where the k-th 1/32 of the output starts with one binary search on its
// diagonal (A addressed by kept index through per-word kept counts in shared memory), then
// merges its stretch sequentially.  O(n + d) per candidate instead of a binary search per key.
// The lanes' outputs go through a per-warp shared-memory stage, 4 keys per lane, and leave as
// 64-byte runs (eight lanes' stretches per store instruction) instead of 32 scattered 16-byte
// stores.  The candidate's removed-rank mask is copied to shared memory first: the lanes walk
// their kept ranks word by word, and a dependent global load per 32 ranks was the kernel's
// largest stall.  Dynamic shared memory: per warp, 2.5 KB of stage + 2 W + 2 words.
#ifndef EF_MERGE_BIG_MINB  // CTAs per SM the merge's register budget is sized for
#define EF_MERGE_BIG_MINB 1
#endif
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, EF_MERGE_BIG_MINB) k_merge_big(VArgs A) {
  extern __shared__ uint4 mb_stage[];
  const Geo& G = A.g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  constexpr uint32_t MK = 4, MS = MK + 1;  // keys per lane per flush; stage row stride (+1: conflict-free 16-byte stores)
  uint4* stage = mb_stage + (uint64_t)w * 32 * MS;  // [32 lanes][MK keys + pad]
  uint32_t* cumk = reinterpret_cast<uint32_t*>(mb_stage + (uint64_t)WARPS * 32 * MS) + (uint64_t)w * (2 * A.W + 2);
  uint32_t* rm = cumk + A.W + 1;  // the removed-rank mask, in shared memory
  for (uint32_t lc = blockIdx.x * WARPS + w; lc < A.n; lc += gridDim.x * WARPS) {  // warp-uniform
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;
    const VPlan& P = A.plan[c];
    const uint32_t pn = (uint32_t)P.pn;
    const uint32_t d = A.dcount[lc];
    const uint32_t* grm = A.rmask + (uint64_t)lc * A.W;
    const uint32_t nw = (pn + 31) >> 5;
    for (uint32_t x = lane; x < nw; x += 32) rm[x] = grm[x];
    rm[nw] = 0u;  // the walk may look one word past the last rank
    __syncwarp();
    // kept counts per word -> exclusive prefix
    uint32_t run = 0;
    for (uint32_t x0 = 0; x0 < nw; x0 += 32) {
      const uint32_t x = x0 + lane;
      uint32_t v = 0;
      if (x < nw) {
        const uint32_t valid = (x + 1 < nw || (pn & 31u) == 0) ? 0xffffffffu : ((1u << (pn & 31u)) - 1u);
        v = __popc(~rm[x] & valid);
      }
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(full, inc, o);
        if (lane >= o) inc += y;
      }
      if (x < nw) cumk[x] = run + inc - v;
      run += __shfl_sync(full, inc, 31);
    }
    if (lane == 0) cumk[nw] = run;
    __syncwarp();
    const uint32_t na = run;
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pskeys = R.skeys(G);
    const uint64_t* bs = A.fresh_sorted + 2ull * lc * A.S;  // B: the key sort's output
    uint64_t* out = A.kstream + 2ull * lc * A.S;
    // rank of the i-th kept parent key (i < na)
    auto select_kept = [&](uint32_t i) -> uint32_t {
      uint32_t lo = 0, hi = nw;  // last word with cumk <= i
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cumk[mid] <= i) lo = mid;
        else hi = mid;
      }
      return 32u * lo + nth_bit(~rm[lo], i - cumk[lo]);
    };
    auto a_raw = [&](uint32_t r) -> uint4 { return __ldg(reinterpret_cast<const uint4*>(pskeys) + r); };
    auto a_key = [&](uint32_t r, uint64_t& k0, uint64_t& k1) {  // big endian
      const uint4 x = a_raw(r);
      k0 = B2b::bswap64(((uint64_t)x.y << 32) | x.x);
      k1 = B2b::bswap64(((uint64_t)x.w << 32) | x.z);
    };
    auto b_key = [&](uint32_t j, uint64_t& k0, uint64_t& k1) {
      const uint4 x = *(reinterpret_cast<const uint4*>(bs) + j);
      k0 = B2b::bswap64(((uint64_t)x.y << 32) | x.x);
      k1 = B2b::bswap64(((uint64_t)x.w << 32) | x.z);
    };
    const uint32_t tot = na + d;
    const uint32_t per = (tot + 31) / 32;
    const uint32_t D = min(tot, per * (uint32_t)lane);
    // merge path: i = number of A elements among the first D outputs
    uint32_t lo = D > d ? D - d : 0u, hi = min(D, na);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      uint64_t a0, a1, b0, b1;
      a_key(select_kept(mid), a0, a1);
      b_key(D - mid - 1, b0, b1);
      if (!be_less(b0, b1, a0, a1)) lo = mid + 1;  // A[mid] <= B[D - mid - 1]
      else hi = mid;
    }
    uint32_t i = lo, j = D - lo;
    const uint32_t end = min(tot, D + per);
    // the A stream: kept ranks in order from the cached mask word, one key fetched ahead
    uint32_t r = i < na ? select_kept(i) : 0u;
    uint32_t wd = r >> 5, bits = (r & 31u) == 31u ? 0u : (~rm[wd] & ~((2u << (r & 31u)) - 1u));
    auto next_rank = [&]() -> uint32_t {  // the kept rank after the last one handed out
      while (!bits) bits = ~rm[++wd];
      const uint32_t x = 32u * wd + (uint32_t)(__ffs(bits) - 1);
      bits &= bits - 1u;
      return x;
    };
    uint64_t a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    if (i < na) a_key(r, a0, a1);
    // the next four A keys and the next B key in flight (independent loads under the merge)
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    uint4 an0 = i + 1 < na ? a_raw(next_rank()) : z4;
    uint4 an1 = i + 2 < na ? a_raw(next_rank()) : z4;
    uint4 an2 = i + 3 < na ? a_raw(next_rank()) : z4;
    uint4 an3 = i + 4 < na ? a_raw(next_rank()) : z4;
    const uint4* b4 = reinterpret_cast<const uint4*>(bs);
    if (j < d) b_key(j, b0, b1);
    uint4 bn0 = j + 1 < d ? b4[j + 1] : z4;
    uint4* o4 = reinterpret_cast<uint4*>(out);
    const uint32_t mine = end - D;  // this lane's outputs (per, or fewer at the tail)
    for (uint32_t t0 = 0; t0 < per; t0 += MK) {  // warp-uniform trip count
#pragma unroll
      for (uint32_t k = 0; k < MK; ++k) {
        if (t0 + k < mine) {
          const bool take_a = j >= d || (i < na && !be_less(b0, b1, a0, a1));
          if (take_a) {
            const uint64_t w0 = B2b::bswap64(a0), w1 = B2b::bswap64(a1);
            stage[lane * MS + k] = make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32));
            if (++i < na) {
              a0 = B2b::bswap64(((uint64_t)an0.y << 32) | an0.x);
              a1 = B2b::bswap64(((uint64_t)an0.w << 32) | an0.z);
              an0 = an1;
              an1 = an2;
              an2 = an3;
              an3 = i + 4 < na ? a_raw(next_rank()) : z4;
            }
          } else {
            const uint64_t w0 = B2b::bswap64(b0), w1 = B2b::bswap64(b1);
            stage[lane * MS + k] = make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32));
            if (++j < d) {
              b0 = B2b::bswap64(((uint64_t)bn0.y << 32) | bn0.x);
              b1 = B2b::bswap64(((uint64_t)bn0.w << 32) | bn0.z);
              bn0 = j + 1 < d ? b4[j + 1] : z4;
            }
          }
        }
      }
      __syncwarp();
      // the stage out: round q stores the 8 keys of lanes 4q .. 4q + 3, 128 contiguous bytes each
      const uint32_t cnt = mine > t0 ? min(MK, mine - t0) : 0u;
#pragma unroll
      for (uint32_t q = 0; q < MK; ++q) {
        const uint32_t src = (32 / MK) * q + (uint32_t)lane / MK, k = (uint32_t)lane % MK;
        const uint32_t c_src = __shfl_sync(full, cnt, src), o_src = __shfl_sync(full, D + t0, src);
        if (k < c_src) o4[o_src + k] = stage[src * MS + k];
      }
      __syncwarp();
    }
  }
}

// k_merge_dir + k_merge_scatter (rows > kFastRows, the default): the same key stream as
// k_merge_big without a serial per-lane merge.  The stream is the parent's sorted keys minus the
// removed ranks with the candidate's sorted fresh keys inserted (graph.py:547 sorts every node
// key), so a fresh key j lands at j + (kept parent keys <= it).  That count comes from a
// per-parent directory of the keys' top 12 bits (k_merge_dir, once per step) plus a search of
// the ~5 parent keys sharing them and the kept-rank prefix of the candidate's removed mask.
// The warps then fill 32 output positions per round: the fresh ones from a ballot of the
// positions in the round, the others from the parent's kept ranks in order (a 64-rank window
// of the removed mask), with one coalesced 16-byte load and store per lane.  A CTA per
// candidate; dynamic shared memory: the removed mask, its kept prefix and the S positions.
constexpr uint32_t kDirBits = 12, kDirN = (1u << kDirBits) + 1;

__device__ __forceinline__ uint32_t key_top(const uint2 x) {  // top kDirBits of the key's first word (big endian)
  return __byte_perm(x.x, 0, 0x0123) >> (32 - kDirBits);
}

__global__ void __launch_bounds__(256) k_merge_dir(const unsigned long long* parent_addr, const Geo G, uint32_t n_parents,
                                                  uint32_t* dir) {
  for (uint32_t pi = blockIdx.x; pi < n_parents; pi += gridDim.x) {
    Rec R{reinterpret_cast<char*>(parent_addr[pi])};
    const uint32_t n = (uint32_t)R.h().n;
    const uint2* sk = reinterpret_cast<const uint2*>(R.skeys(G));  // key r's first word: sk[2r]
    uint32_t* D = dir + (uint64_t)pi * kDirN;
    // D[b] = the first rank whose top bits are >= b: rank r owns (top(r - 1), top(r)], the
    // end sentinel rank n owns the rest up to D[2^bits]
    for (uint32_t r = threadIdx.x; r <= n; r += blockDim.x) {
      const uint32_t t1 = r < n ? key_top(sk[2 * r]) : (1u << kDirBits);
      const uint32_t t0 = r ? key_top(sk[2 * (r - 1)]) + 1u : 0u;
      for (uint32_t b = t0; b <= t1; ++b) D[b] = r;
    }
  }
}

__device__ __forceinline__ void be_key(const uint4 x, uint64_t& k0, uint64_t& k1) {
  k0 = B2b::bswap64(((uint64_t)x.y << 32) | x.x);
  k1 = B2b::bswap64(((uint64_t)x.w << 32) | x.z);
}

//
// SORT (16-bit positions only): the fresh keys are read unsorted from the node-key rows and
// ordered here, replacing k_sortbig: a histogram on the same top 12 bits as the directory, a
// block scan, a scatter of the job indices and an insertion sort inside each bucket (~1 key
// per bucket on DAG-20k).  Candidates with up to kMsDcap fresh keys keep the order and the
// positions in shared memory, larger ones in their (by now idle) sort-key row.
#ifndef EF_MS_DCAP
#define EF_MS_DCAP 4096
#endif
constexpr uint32_t kMsDcap = EF_MS_DCAP;

template <int BT, typename PT, bool SORT>  // PT: the position type (uint16_t while S < 2^16)
__global__ void __launch_bounds__(BT) k_merge_scatter(VArgs A) {
  extern __shared__ uint32_t ms_sh[];
  constexpr uint32_t NWARP = BT / 32;
  __shared__ uint32_t wsum[NWARP], slot_sh[NWARP][32];
  const Geo& G = A.g;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const unsigned full = 0xffffffffu;
  uint32_t* slot = slot_sh[wid];  // kept ranks of the warp's round, by ordinal
  uint32_t* rm = ms_sh;           // [W + 2] removed ranks; ranks past the parent's count read as removed
  uint32_t* cumk = rm + A.W + 2;  // [W + 1] kept ranks before each mask word
  // !SORT: [S] output position of every fresh key (ascending).  SORT: [2^12] bucket counters,
  // [kMsDcap] first key words by job (then, aliased, the positions), [kMsDcap] job indices in
  // key order
  uint32_t* bins = cumk + A.W + 1;
  uint32_t* top_sm = bins + (1u << kDirBits);
  PT* pb_sm = reinterpret_cast<PT*>(SORT ? top_sm : bins);
  uint16_t* perm_sm = reinterpret_cast<uint16_t*>(top_sm + kMsDcap);
  for (uint32_t lc = blockIdx.x; lc < A.n; lc += gridDim.x) {
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;  // CTA-uniform
    const VPlan& P = A.plan[c];
    const uint32_t pn = (uint32_t)P.pn, d = A.dcount[lc], nw = (pn + 31) >> 5;
    PT* pb = pb_sm;
    uint32_t* top = top_sm;
    uint16_t* perm = perm_sm;
    if (SORT && d > kMsDcap) {  // CTA-uniform: the candidate's sort-key row (8 S bytes)
      top = reinterpret_cast<uint32_t*>(A.skey + (uint64_t)lc * A.S);
      pb = reinterpret_cast<PT*>(top);
      perm = reinterpret_cast<uint16_t*>(top + A.S);
    }
    const uint4* fk = reinterpret_cast<const uint4*>(A.fresh + 2ull * lc * A.S);  // fresh keys, job order
    const uint32_t* grm = A.rmask + (uint64_t)lc * A.W;
    for (uint32_t x = threadIdx.x; x < nw + 2; x += BT) {
      uint32_t v = x < nw ? grm[x] : 0xffffffffu;
      if (x + 1 == nw && (pn & 31u)) v |= ~((1u << (pn & 31u)) - 1u);
      rm[x] = v;
    }
    __syncthreads();
    // kept ranks before each word: a block scan over contiguous runs of words
    const uint32_t per = (nw + BT - 1) / BT, x0 = min(nw, threadIdx.x * per), x1 = min(nw, x0 + per);
    uint32_t s = 0;
    for (uint32_t x = x0; x < x1; ++x) s += __popc(~rm[x]);
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(full, inc, o);
      if ((int)lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    uint32_t run = inc - s, na = 0;
#pragma unroll
    for (uint32_t w = 0; w < NWARP; ++w) {
      const uint32_t v = wsum[w];
      run += w < wid ? v : 0u;
      na += v;
    }
    for (uint32_t x = x0; x < x1; ++x) {
      cumk[x] = run;
      run += __popc(~rm[x]);
    }
    if (threadIdx.x == 0) cumk[nw] = na;
    __syncthreads();
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint4* pa = reinterpret_cast<const uint4*>(R.skeys(G));
    const uint32_t* D = A.pdir + (uint64_t)P.parent * kDirN;
    const uint4* bk = reinterpret_cast<const uint4*>(A.fresh_sorted + 2ull * lc * A.S);
    if (SORT) {  // the fresh keys in key order: perm[k] = job index of the k-th smallest
      uint32_t lg = 5;  // pow2(d) buckets, 32 .. 2^12, on the top bits (~1 key each)
      while ((1u << lg) < d && lg < kDirBits) ++lg;
      const uint32_t nbk = 1u << lg;
      for (uint32_t b = threadIdx.x; b < nbk; b += BT) bins[b] = 0;
      __syncthreads();
      for (uint32_t j = threadIdx.x; j < d; j += BT) {
        const uint2 x = reinterpret_cast<const uint2*>(fk + j)[0];
        const uint32_t tw = __byte_perm(x.x, 0, 0x0123);  // first 4 key bytes, big endian
        top[j] = tw;
        atomicAdd(&bins[tw >> (32 - lg)], 1u);
      }
      __syncthreads();
      block_excl_scan_inplace<BT>(bins, nbk, wsum);
      __syncthreads();
      for (uint32_t j = threadIdx.x; j < d; j += BT) perm[atomicAdd(&bins[top[j] >> (32 - lg)], 1u)] = (uint16_t)j;
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < nbk; b += BT) {  // bins[b]: the end of bucket b
        const uint32_t e = bins[b], s0 = b ? bins[b - 1] : 0u;
        for (uint32_t x = s0 + 1; x < e; ++x) {  // by the first 4 bytes, the full key on a tie
          const uint16_t v = perm[x];
          const uint32_t tv = top[v];
          uint32_t y = x;
          while (y > s0) {
            const uint16_t u = perm[y - 1];
            const uint32_t tu = top[u];
            bool less = tv < tu;
            if (tv == tu) {
              uint64_t v0, v1, u0, u1;
              be_key(fk[v], v0, v1);
              be_key(fk[u], u0, u1);
              less = be_less(v0, v1, u0, u1);
            }
            if (!less) break;
            perm[y] = u;
            --y;
          }
          perm[y] = v;
        }
      }
      __syncthreads();  // (top is dead from here: pb reuses it)
    }
    // 1) every fresh key's position: j + the kept parent keys <= it (the parent's key first on a tie)
    // two keys per thread and pass, their searches interleaved (independent load chains)
    auto fresh_key = [&](uint32_t k) -> uint4 { return SORT ? fk[perm[k]] : bk[k]; };  // the k-th smallest
    for (uint32_t j0 = threadIdx.x; j0 < d; j0 += 2 * BT) {
      const uint32_t j1 = j0 + BT;
      const bool h1 = j1 < d;
      uint64_t b0, b1, e0 = ~0ull, e1 = ~0ull;
      be_key(fresh_key(j0), b0, b1);
      if (h1) be_key(fresh_key(j1), e0, e1);
      const uint32_t tb = (uint32_t)(b0 >> (64 - kDirBits)), te = (uint32_t)(e0 >> (64 - kDirBits));
      uint32_t lo = __ldg(D + tb), hi = __ldg(D + tb + 1);  // the parent ranks sharing its top bits
      uint32_t lo1 = h1 ? __ldg(D + te) : 0u, hi1 = h1 ? __ldg(D + te + 1) : 0u;
      while (lo < hi || lo1 < hi1) {
        const bool s0 = lo < hi, s1 = lo1 < hi1;
        const uint32_t m0 = (lo + hi) >> 1, m1 = (lo1 + hi1) >> 1;
        const uint4 x0 = __ldg(pa + (s0 ? m0 : 0u)), x1 = __ldg(pa + (s1 ? m1 : 0u));
        uint64_t a0, a1, f0, f1;
        be_key(x0, a0, a1);
        be_key(x1, f0, f1);
        if (s0) {
          if (be_less(b0, b1, a0, a1)) hi = m0;
          else lo = m0 + 1;
        }
        if (s1) {
          if (be_less(e0, e1, f0, f1)) hi1 = m1;
          else lo1 = m1 + 1;
        }
      }
      pb[j0] = (PT)(j0 + cumk[lo >> 5] + __popc(~rm[lo >> 5] & ((1u << (lo & 31u)) - 1u)));
      if (h1) pb[j1] = (PT)(j1 + cumk[lo1 >> 5] + __popc(~rm[lo1 >> 5] & ((1u << (lo1 & 31u)) - 1u)));
    }
    __syncthreads();
    auto select_kept = [&](uint32_t i) -> uint32_t {  // rank of the i-th kept parent key (i < na)
      uint32_t l = 0, h = nw;                          // last word with cumk <= i
      while (h - l > 1) {
        const uint32_t mid = (l + h) >> 1;
        if (cumk[mid] <= i) l = mid;
        else h = mid;
      }
      return 32u * l + nth_bit(~rm[l], i - cumk[l]);
    };
    // 2) the stream, 32 positions per warp round over a contiguous span per warp
    const uint32_t tot = na + d;
    uint4* out = reinterpret_cast<uint4*>(A.kstream + 2ull * lc * A.S);
    const uint32_t span = (tot + NWARP * 32 - 1) / (NWARP * 32) * 32;
    uint32_t p0 = wid * span;
    const uint32_t pend = min(tot, p0 + span);
    if (p0 < pend) {  // warp-uniform
      uint32_t nb = 0, hb = d;  // fresh keys before p0
      while (nb < hb) {
        const uint32_t mid = (nb + hb) >> 1;
        if ((uint32_t)pb[mid] < p0) nb = mid + 1;
        else hb = mid;
      }
      uint32_t ka = p0 - nb;                         // kept parent keys before p0
      uint32_t rc = ka < na ? select_kept(ka) : pn;  // the next kept rank
      const uint32_t ltm = (1u << lane) - 1u;
      for (; p0 < pend; p0 += 32) {
        const uint32_t v = nb + lane < d ? (uint32_t)pb[nb + lane] : 0xffffffffu;
        const uint32_t bmask = __reduce_or_sync(full, v - p0 < 32u ? 1u << (v - p0) : 0u);
        const uint32_t cnt = min(32u, pend - p0), nf = __popc(bmask), nA = cnt - nf;
        uint32_t have = 0;  // kept ranks published in slot[] (ordinals < nA)
        if (nA) {  // the kept ranks among rc .. rc + 63 publish themselves by ordinal
          const uint32_t wi = rc >> 5, sh = rc & 31u;
          const uint32_t k_lo = ~__funnelshift_r(rm[wi], rm[wi + 1], sh);
          const uint32_t k_hi = ~__funnelshift_r(rm[wi + 1], rm[wi + 2], sh);
          const uint32_t c_lo = __popc(k_lo);
          const uint32_t o_lo = __popc(k_lo & ltm), o_hi = c_lo + __popc(k_hi & ltm);
          if (((k_lo >> lane) & 1u) && o_lo < nA) slot[o_lo] = rc + lane;
          if (((k_hi >> lane) & 1u) && o_hi < nA) slot[o_hi] = rc + 32u + lane;
          have = min(nA, c_lo + __popc(k_hi));
          __syncwarp();
        }
        const uint32_t before = __popc(bmask & ltm);
        if (lane < cnt) {
          uint4 key;
          if ((bmask >> lane) & 1u) {
            key = fresh_key(nb + before);
          } else {
            const uint32_t t = lane - before;
            key = __ldg(pa + (t < have ? slot[t] : select_kept(ka + t)));  // (< 32 kept ranks in 64: rare)
          }
          out[p0 + lane] = key;
        }
        if (nA) rc = (nA <= have ? slot[nA - 1] : select_kept(ka + nA - 1)) + 1u;
        __syncwarp();
        ka += nA;
        nb += nf;
      }
    }
    __syncthreads();  // rm, cumk and pb are the next candidate's
  }
}

// The digest's prefix for graphs with many outputs (DAG-5k / 20k: 1.2k / 4.8k outputs, a quarter
// of the digest's blocks): the input text and every output's key and port (graph.py:541-547,
// 18 bytes per output) as aligned little-endian words, a warp per candidate and a lane per
// word (at most two output records per word), so the digest thread streams it like the keys
// instead of chaining output -> source -> key loads and byte pushes.
// word q of the digest's prefix: the input text, then 18-byte output records
// rec(r, key0, key1, port_be) (graph.py:541-547), as little-endian words
template <class RecF>
__device__ __forceinline__ uint64_t prefix_word(uint32_t q, uint32_t li, const uint64_t* input_words, RecF rec) {
  const uint32_t x = 8u * q;
  if (x + 8u <= li) return __ldg(input_words + q);  // input text only
  uint32_t b = 0;  // bytes of this word taken so far
  uint64_t wv = 0;
  if (x < li) {  // the input text's tail (the words are zero padded)
    b = li - x;
    wv = __ldg(input_words + q) & ((1ull << (8 * b)) - 1ull);
  }
  // stream bytes [y, y + 8 - b) of the output records: record r from byte o, then r + 1
  const uint32_t y = x + b - li, r = y / 18u, o = y - 18u * r;
  uint64_t a0, a1, ap, n0 = 0, n1 = 0, np = 0;
  rec(r, a0, a1, ap);
  if (o + (8u - b) > 18u) rec(r + 1, n0, n1, np);
  // the two records as little-endian words: a0 | a1 | ap + n0 << 16 | n0 >> 48 + n1 << 16
  const uint64_t w2 = ap | (n0 << 16), w3 = (n0 >> 48) | (n1 << 16);
  const uint32_t jw = o >> 3, sh = 8u * (o & 7u);
  const uint64_t lo = jw == 0 ? a0 : jw == 1 ? a1 : w2;
  const uint64_t hi = jw == 0 ? a1 : jw == 1 ? w2 : w3;
  uint64_t v = sh ? (lo >> sh) | (hi << (64u - sh)) : lo;
  if (b) v &= (1ull << (8 * (8 - b))) - 1ull;
  return wv | (v << (8 * b));
}

// The first prefix block a candidate's digest must compress: its prefix equals the parent's up
// to output pfx_first, so the blocks before that byte are the parent's, whose BLAKE2b states
// k_pfx_chain has saved (the digest and k_prefix both start there).
__device__ __forceinline__ uint32_t pfx_block0(const VArgs& A, uint32_t lc, uint32_t li, uint32_t n_out) {
  if (!A.pfx_state) return 0u;
  const uint32_t fb = li + 18u * A.pfx_first[lc];
  return min(fb >> 7, (li + 18u * n_out) >> 7);
}

__global__ void __launch_bounds__(128) k_prefix(VArgs A) {
  const Geo& G = A.g;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t li = A.T.input_text_len;
  for (uint32_t lc = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; lc < A.n; lc += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;  // warp-uniform
    const VPlan& P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pkeys = R.keys(G);
    const uint32_t* pouts = R.outs(G);
    const uint32_t n_out = (uint32_t)R.h().n_out;
    const uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    const uint32_t* osrc = A.outsrc + (uint64_t)lc * A.Os;
    const uint32_t n_rm = (uint32_t)P.n_rm;
    const uint32_t rf0 = P.rm_from[0], rf1 = P.rm_from[1], rt0 = P.rm_to[0], rt1 = P.rm_to[1];
    // output record r: its key words and big-endian port (graph.py:541-547); zero past the last
    auto rec = [&](uint32_t r, uint64_t& k0, uint64_t& k1, uint64_t& pbe) {
      if (r >= n_out) {
        k0 = k1 = pbe = 0;
        return;
      }
      uint32_t ref = pouts[r];
      if (n_rm > 0 && ref == rf0) ref = rt0;  // vremap
      else if (n_rm > 1 && ref == rf1) ref = rt1;
      const uint64_t* kp;
      if (A.osrc) {
        const uint32_t sv = osrc[r], idx = sv & 0x7fffffu;
        kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
      } else {
        const uint32_t p = ref >> 8, fi = didx[p];
        kp = fi ? fresh + 2 * (fi - 1) : pkeys + 2 * p;
      }
      k0 = kp[0];
      k1 = kp[1];
      pbe = port_be(ref & 255u);
    };
    const uint32_t len = li + 18u * n_out;
    const uint32_t nwd = (len + 7) >> 3;
    uint64_t* out = A.pfx + (uint64_t)lc * A.pfx_stride;
    for (uint32_t q = 16u * pfx_block0(A, lc, li, n_out) + lane; q < nwd; q += 32)  // (the parent's blocks are skipped)
      out[q] = prefix_word(q, li, A.input_words, rec);
  }
}

// The parent's prefix chain: a warp per parent builds each 128-byte prefix block (16 lanes, a
// word each) and one lane compresses it, saving the state after every block.
__global__ void __launch_bounds__(32) k_pfx_chain(const unsigned long long* parent_addr, const Geo G, uint32_t n_parents,
                                                 const uint64_t* input_words, uint32_t li, uint32_t nst, uint64_t* states) {
  __shared__ uint64_t m[16];
  const uint32_t lane = threadIdx.x;
  for (uint32_t pi = blockIdx.x; pi < n_parents; pi += gridDim.x) {
    Rec R{reinterpret_cast<char*>(parent_addr[pi])};
    const uint64_t* pkeys = R.keys(G);
    const uint32_t* pouts = R.outs(G);
    const uint32_t n_out = (uint32_t)R.h().n_out;
    auto rec = [&](uint32_t r, uint64_t& k0, uint64_t& k1, uint64_t& pbe) {
      if (r >= n_out) {
        k0 = k1 = pbe = 0;
        return;
      }
      const uint32_t ref = pouts[r];
      k0 = pkeys[2 * (ref >> 8)];
      k1 = pkeys[2 * (ref >> 8) + 1];
      pbe = port_be(ref & 255u);
    };
    const uint32_t nbp = min((li + 18u * n_out) >> 7, nst - 1);
    uint64_t* st = states + (uint64_t)pi * nst * 8;
    uint64_t h[8];
    b2b_start(h, 8);
    if (lane < 8) st[lane] = h[lane];
    for (uint32_t b = 0; b < nbp; ++b) {
      if (lane < 16) m[lane] = prefix_word(16u * b + lane, li, input_words, rec);
      __syncwarp();
      if (lane == 0) {
        b2b_compress(h, m, 128ull * (b + 1), false);
#pragma unroll
        for (int i = 0; i < 8; ++i) st[8ull * (b + 1) + i] = h[i];
      }
      __syncwarp();
    }
  }
}

// The graph digest over a pre-merged key stream: the prefix (input declarations, output keys
// and ports) goes through the word sink; the keys follow as full words with a constant byte
// shift, loaded 16 words per block with independent 16-byte loads.
// PF: the key words of block b + 1 are loaded into registers while block b is compressed
// (large graphs: a few resident warps per SM cannot hide the stream's DRAM latency otherwise)
template <int BT, bool PF, int MINB>
__global__ void __launch_bounds__(BT, MINB) k_digest_pm(VArgs A) {
  __shared__ uint64_t blk[16 * BT];
  const Geo& G = A.g;
  const Tables& T = A.T;
  uint64_t* col = blk + threadIdx.x;
  for (uint32_t lc = blockIdx.x * BT + threadIdx.x; lc < A.n; lc += gridDim.x * BT) {
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;
    const VPlan& P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pkeys = R.keys(G);
    const uint32_t* pouts = R.outs(G);
    const int n_out = R.h().n_out;
    const uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    const uint64_t* ks = A.kstream + 2ull * lc * A.S;  // merged key stream
    const uint32_t li = T.input_text_len;
    const uint32_t n_child = (uint32_t)(P.n_keep + P.n_live);
    const uint32_t kwords = 2 * n_child;
    const uint64_t len = (uint64_t)li + 18ull * n_out + 16ull * n_child;
    const uint32_t nblk = (uint32_t)((len + 127) >> 7);
    int phase = 0;  // 0 input text, 1 outputs, 2 keys, 3 done
    uint32_t gi = 0, part = 0, kw = 0;
    uint64_t cw1 = 0;
    WordSink<BT> sk;
    sk.init(col);
    uint64_t h[8];
    b2b_start(h, 8);
    uint4 pf[9];
    uint32_t pf_kw = 0xffffffffu;
    // the prefix from k_prefix: pw_full whole words, then pw_rem bytes
    const uint64_t* pw = A.pfx ? A.pfx + (uint64_t)lc * A.pfx_stride : nullptr;
    const uint32_t pw_full = (uint32_t)(((uint64_t)li + 18ull * n_out) >> 3), pw_rem = (uint32_t)((li + 18ull * n_out) & 7);
    uint32_t pq = 0, b0 = 0;
    if (pw && A.pfx_state) {  // the blocks before the first changed output are the parent's: start from its state
      b0 = pfx_block0(A, lc, li, (uint32_t)n_out);
      const uint64_t* ps = A.pfx_state + ((uint64_t)P.parent * A.pfx_nst + b0) * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) h[i] = ps[i];
      pq = 16u * b0;
    }
    for (uint32_t b = b0; b < nblk; ++b) {
      sk.q = 0;
      if (pw && phase < 2) {  // whole prefix words (the sink is word-aligned until the last one)
        const uint32_t take = min(16u, pw_full - pq);
        uint64_t wv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) wv[i] = (uint32_t)i < take ? pw[pq + i] : 0ull;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if ((uint32_t)i < take) sk.push(wv[i], 8);
        pq += take;
        if (pq == pw_full && sk.q < 16) {
          if (pw_rem) sk.push(pw[pq], pw_rem);
          phase = 2;
        }
      }
      while (sk.q < 16 && phase < 2) {
        if (phase == 0) {
          if (gi * 8 < li) {
            sk.push(__ldg(A.input_words + gi), min(8u, li - gi * 8));
            ++gi;
          } else {
            phase = 1;
            gi = 0;
          }
        } else {
          if ((int)gi < n_out) {
            const uint32_t ref = vremap(P, pouts[gi]);
            if (part == 0) {
              const uint64_t* kp;
              if (A.osrc) {
                const uint32_t sv = A.outsrc[(uint64_t)lc * A.Os + gi], idx = sv & 0x7fffffu;
                kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
              } else {
                const uint32_t p = ref >> 8, fi = didx[p];
                kp = fi ? fresh + 2 * (fi - 1) : pkeys + 2 * p;
              }
              sk.push(kp[0], 8);
              cw1 = kp[1];
              part = 1;
            } else if (part == 1) {
              sk.push(cw1, 8);
              part = 2;
            } else {
              sk.push(port_be(ref & 255u), 2);
              part = 0;
              ++gi;
            }
          } else {
            phase = 2;
          }
        }
      }
      if (phase == 2 && sk.q < 16) {  // keys: full words at a constant shift
        const uint32_t room = 16 - sk.q;
        const uint32_t take = min(room, kwords - kw);
        uint64_t wv[16];
        if (pf_kw == kw) {  // the 16-byte pairs covering [kw, kw + 16) were loaded a block ahead
          const bool odd = kw & 1u;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint4 x = odd ? pf[(i + 1) >> 1] : pf[i >> 1];
            const bool hi = odd ? !(i & 1) : (i & 1);
            wv[i] = hi ? (((uint64_t)x.w << 32) | x.z) : (((uint64_t)x.y << 32) | x.x);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            if ((uint32_t)i < take) {
              const uint4 x = *reinterpret_cast<const uint4*>(ks + ((kw + i) & ~1u));
              // kw is even except after an odd take; load the aligned pair then pick
              const uint64_t lo = ((uint64_t)x.y << 32) | x.x, hi = ((uint64_t)x.w << 32) | x.z;
              if ((kw & 1u) == 0) {
                wv[i] = lo;
                wv[i + 1] = hi;
              } else {
                wv[i] = hi;
                wv[i + 1] = (uint32_t)(i + 1) < take ? ks[kw + i + 1] : 0;
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if ((uint32_t)i < take) sk.push(wv[i], 8);
        kw += take;
        if (kw == kwords) phase = 3;
        if (PF && kw < kwords) {  // the next block's pairs, in flight under this compression
          const uint32_t p0 = kw >> 1, np = (kwords + 1) >> 1;
          const uint4* k4 = reinterpret_cast<const uint4*>(ks);
#pragma unroll
          for (int k = 0; k < 9; ++k) pf[k] = p0 + k < np ? k4[p0 + k] : make_uint4(0, 0, 0, 0);
          pf_kw = kw;
        }
      }
      if (phase == 3 && sk.q < 16) {
        sk.flush();
        for (uint32_t q = sk.q; q < 16; ++q) col[q * BT] = 0;
      }
      b2b_compress_col<BT>(h, col, len < 128ull * (b + 1) ? len : 128ull * (b + 1), b + 1 == nblk);
    }
    A.res[c].hash = B2b::bswap64(h[0]);
    if (A.stats) atomicAdd(A.stats + 1, (unsigned long long)(nblk - b0));
  }
}

// Rows > 256, fused: the graph digest of k_digest_pm with the key stream produced on the fly
// instead of read from a merged row (no k_merge_big, no stream written and re-read: 2 x 16 B
// per key of HBM traffic saved).  The thread merges, in the digest's order, the parent's
// sorted keys minus the removed ranks (A: kept ranks walked through the removed mask, the keys
// read from the parent record, shared by the parent's candidates through L2) with the
// candidate's sorted fresh keys (B, from the key sort), parent first on equal keys as in
// k_merge / k_merge_big.  The next A keys and the next B key are in flight while a key is
// placed, so the compression's loads are L2 hits with their latency overlapped.
template <int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB) k_digest_mg(VArgs A) {
  __shared__ uint64_t blk[16 * BT];
  const Geo& G = A.g;
  const Tables& T = A.T;
  uint64_t* col = blk + threadIdx.x;
  for (uint32_t lc = blockIdx.x * BT + threadIdx.x; lc < A.n; lc += gridDim.x * BT) {
    const uint32_t c = A.c0 + lc;
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;
    const VPlan& P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    const uint64_t* pkeys = R.keys(G);
    const uint32_t* pouts = R.outs(G);
    const int n_out = R.h().n_out;
    const uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    const uint32_t li = T.input_text_len;
    const uint32_t n_child = (uint32_t)(P.n_keep + P.n_live);
    const uint64_t len = (uint64_t)li + 18ull * n_out + 16ull * n_child;
    const uint32_t nblk = (uint32_t)((len + 127) >> 7);
    // the two sorted streams
    const uint32_t pn = (uint32_t)P.pn, d = A.dcount[lc];
    const uint32_t* rm = A.rmask + (uint64_t)lc * A.W;
    const uint4* a4 = reinterpret_cast<const uint4*>(R.skeys(G));
    const uint4* b4 = reinterpret_cast<const uint4*>(A.fresh_sorted + 2ull * lc * A.S);
    uint32_t wd = 0, bits = pn ? ~__ldg(rm) & (pn >= 32 ? 0xffffffffu : ((1u << pn) - 1u)) : 0u;
    auto next_rank = [&]() -> uint32_t {  // the next kept parent rank (pn: none left)
      while (!bits) {
        if (++wd >= (pn + 31) >> 5) return pn;
        bits = ~__ldg(rm + wd);
        if (wd == (pn >> 5)) bits &= (1u << (pn & 31u)) - 1u;
      }
      const uint32_t x = 32u * wd + (uint32_t)(__ffs(bits) - 1);
      bits &= bits - 1u;
      return x;
    };
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    uint32_t ra0 = next_rank(), ra1 = ra0 < pn ? next_rank() : pn;
    uint4 ac = ra0 < pn ? __ldg(a4 + ra0) : z4, an = ra1 < pn ? __ldg(a4 + ra1) : z4;
    bool ha = ra0 < pn;
    uint32_t ra2 = ra1 < pn ? next_rank() : pn;
    uint4 bc = d ? b4[0] : z4, bn = d > 1 ? b4[1] : z4;
    uint32_t j = 0;
    auto be = [](const uint4& x, uint64_t& k0, uint64_t& k1) {
      k0 = B2b::bswap64(((uint64_t)x.y << 32) | x.x);
      k1 = B2b::bswap64(((uint64_t)x.w << 32) | x.z);
    };
    // next key of the merged stream (raw words w0, w1)
    auto next_key = [&](uint64_t& w0, uint64_t& w1) {
      uint64_t a0, a1, b0, b1;
      be(ac, a0, a1);
      be(bc, b0, b1);
      const bool take_a = ha && (j >= d || !be_less(b0, b1, a0, a1));
      const uint4 x = take_a ? ac : bc;
      w0 = ((uint64_t)x.y << 32) | x.x;
      w1 = ((uint64_t)x.w << 32) | x.z;
      if (take_a) {
        ac = an;
        ha = ra1 < pn;
        ra1 = ra2;
        an = ra2 < pn ? __ldg(a4 + ra2) : z4;
        ra2 = ra2 < pn ? next_rank() : pn;
      } else {
        bc = bn;
        ++j;
        bn = j + 1 < d ? b4[j + 1] : z4;
      }
    };
    int phase = 0;  // 0 input text, 1 outputs, 2 keys, 3 done
    uint32_t gi = 0, part = 0, kdone = 0;
    uint64_t cw1 = 0;
    WordSink<BT> sk;
    sk.init(col);
    uint64_t h[8];
    b2b_start(h, 8);
    for (uint32_t b = 0; b < nblk; ++b) {
      sk.q = 0;
      while (sk.q < 16 && phase < 2) {
        if (phase == 0) {
          if (gi * 8 < li) {
            sk.push(__ldg(A.input_words + gi), min(8u, li - gi * 8));
            ++gi;
          } else {
            phase = 1;
            gi = 0;
          }
        } else {
          if ((int)gi < n_out) {
            const uint32_t ref = vremap(P, pouts[gi]);
            if (part == 0) {
              const uint64_t* kp;
              if (A.osrc) {
                const uint32_t sv = A.outsrc[(uint64_t)lc * A.Os + gi], idx = sv & 0x7fffffu;
                kp = (sv & kFresh) ? fresh + 2 * idx : pkeys + 2 * idx;
              } else {
                const uint32_t p = ref >> 8, fi = didx[p];
                kp = fi ? fresh + 2 * (fi - 1) : pkeys + 2 * p;
              }
              sk.push(kp[0], 8);
              cw1 = kp[1];
              part = 1;
            } else if (part == 1) {
              sk.push(cw1, 8);
              part = 2;
            } else {
              sk.push(port_be(ref & 255u), 2);
              part = 0;
              ++gi;
            }
          } else {
            phase = 2;
          }
        }
      }
      // keys: whole keys (two words) while at least two words are free in the block; a key
      // that straddles the block boundary leaves its second word for the next block
      // (an 8-byte push writes exactly one word, whatever the byte shift)
      while (phase == 2 && sk.q < 16) {
        if (part == 3) {  // the second word of a straddling key
          sk.push(cw1, 8);
          part = 0;
          if (++kdone == n_child) phase = 3;
          continue;
        }
        if (kdone == n_child) {
          phase = 3;
          break;
        }
        uint64_t w0, w1;
        next_key(w0, w1);
        sk.push(w0, 8);
        if (sk.q < 16) {
          sk.push(w1, 8);
          if (++kdone == n_child) phase = 3;
        } else {
          cw1 = w1;
          part = 3;
        }
      }
      if (phase == 3 && sk.q < 16) {
        sk.flush();
        for (uint32_t q = sk.q; q < 16; ++q) col[q * BT] = 0;
      }
      b2b_compress_col_pf<BT>(h, col, len < 128ull * (b + 1) ? len : 128ull * (b + 1), b + 1 == nblk);
    }
    A.res[c].hash = B2b::bswap64(h[0]);
    if (A.stats) atomicAdd(A.stats + 1, (unsigned long long)nblk);
  }
}

// full mode: one job per node in topological order (job index = topological slot), every
// producer key fresh.  Block per record: slots in parallel, ref offsets by a block scan.
template <int BT>
__global__ void __launch_bounds__(BT) k_full_jobs(VArgs A) {
  __shared__ uint32_t sh_scan[BT / 32 + 1];
  const Geo& G = A.g;
  const Tables& T = A.T;
  for (uint32_t lc = blockIdx.x; lc < A.n; lc += gridDim.x) {
    const uint32_t c = A.c0 + lc;
    Rec R{reinterpret_cast<char*>(A.parent_addr[c])};
    const int n = R.h().n;
    const uint32_t* topo = R.topo(G);
    const uint32_t* sig = R.sig(G);
    const uint32_t* aux = R.aux(G);
    const uint32_t* nin = R.nin(G);
    const uint32_t* inoff = R.inoff(G);
    const uint32_t* refs = R.refs(G);
    uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    uint32_t* jv = A.jv + (uint64_t)lc * A.S;
    Job* jobs = A.jobs + (uint64_t)lc * A.S;
    uint32_t* rs = A.refsrc + (uint64_t)lc * A.Rs;
    for (int s = threadIdx.x; s < n; s += BT) {
      const uint32_t v = topo[s];
      didx[v] = (uint32_t)s + 1;
      jv[s] = v;
    }
    __syncthreads();
    uint32_t run = 0;
    for (int s0 = 0; s0 < n; s0 += BT) {
      const int s = s0 + threadIdx.x;
      uint32_t v = 0, sg = 0, nr = 0;
      bool input = false;
      if (s < n) {
        v = topo[s];
        sg = sig[v];
        input = T.sig_desc[sg].kind == EF_K_INPUT;
        nr = input ? 0u : nin[v];
      }
      uint32_t tot;
      const uint32_t r = run + block_excl_scan<BT>(nr, &tot, sh_scan);
      if (s < n) {
        if (input) {
          jobs[s] = Job{sg, aux[v], 0u, kInputJob};
        } else {
          const uint32_t r0 = inoff[v];
          for (uint32_t k = 0; k < nr; ++k) {
            const uint32_t ref = refs[r0 + k];
            rs[r + k] = kFresh | ((ref & 255u) << 23) | (didx[ref >> 8] - 1);
          }
          jobs[s] = Job{sg, aux[v], r, nr};
        }
      }
      run += tot;
    }
    if (threadIdx.x == 0) {
      A.dcount[lc] = (uint32_t)n;
      A.seg_begin[lc] = (int32_t)((uint64_t)lc * A.S);
      A.seg_end[lc] = (int32_t)((uint64_t)lc * A.S + n);
    }
    __syncthreads();
  }
}

// full mode: write the node keys, the sorted order, the sorted keys and the ranks into the
// record (block per record, coalesced)
__global__ void k_full_store(VArgs A) {
  const Geo& G = A.g;
  for (uint32_t lc = blockIdx.x; lc < A.n; lc += gridDim.x) {
    const uint32_t c = A.c0 + lc;
    Rec R{reinterpret_cast<char*>(A.parent_addr[c])};
    const int n = R.h().n;
    const uint32_t* didx = A.didx + (uint64_t)lc * A.S;
    const uint32_t* jv = A.jv + (uint64_t)lc * A.S;
    const uint64_t* fresh = A.fresh + 2ull * lc * A.S;
    const uint64_t* fs = A.fresh_sorted + 2ull * lc * A.S;
    const uint32_t* sv = A.sval_sorted + (uint64_t)lc * A.S;
    uint64_t* keys = R.keys(G);
    uint64_t* skeys = R.skeys(G);
    uint32_t* sperm = R.sperm(G);
    uint32_t* srank = R.srank(G);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t j = didx[i] - 1;
      keys[2 * i] = fresh[2 * j];
      keys[2 * i + 1] = fresh[2 * j + 1];
      const uint32_t v = jv[sv[i]];
      sperm[i] = v;
      srank[v] = (uint32_t)i;
      skeys[2 * i] = fs[2 * i];
      skeys[2 * i + 1] = fs[2 * i + 1];
    }
  }
}

// step-wide maxima of record sizes (sizes the full-mode scratch)
__global__ void k_rec_max(const unsigned long long* rec, uint32_t n, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const ef_rec_header& H = *reinterpret_cast<const ef_rec_header*>(rec[i]);
    atomicMax(out, (uint32_t)H.n);
    atomicMax(out + 1, (uint32_t)H.n_refs);
  }
}

// ------------------------------------------------------------------------------------------
// the inner search on a virtual candidate: child nodes in id order are the parent positions
// minus the dropped ones (the rewritten node with its new signature), then the new nodes
// (their ids are max + 1, max + 2: rules.py:129-131)
// ------------------------------------------------------------------------------------------

struct VirtView {
  const uint32_t* nsk;  // the parent's movable-node bits (k_price_nsk), or null: the dense sweep
  const uint32_t* psig;
  const uint32_t* p_ro;  // the parent's per-node price rows (k_match)
  const uint32_t* p_rn;
  int32_t drop0, drop1, mod, n_keep;
  uint32_t mod_sig, s_new0, s_new1;
  int n;
  __device__ __forceinline__ int ppos(int i) const {
    int pp = i;
    if (drop0 >= 0 && pp >= drop0) ++pp;
    if (drop1 >= 0 && pp >= drop1) ++pp;
    return pp;
  }
  __device__ __forceinline__ uint32_t sig(int i) const {
    if (i < n_keep) {
      const int pp = ppos(i);
      return pp == mod ? mod_sig : psig[pp];
    }
    return i == n_keep ? s_new0 : s_new1;
  }
  __device__ __forceinline__ uint2 info(int i, const Tables& T) const {
    if (i < n_keep) {
      const int pp = ppos(i);
      if (pp != mod) return make_uint2(p_ro[pp], p_rn[pp]);
      return T.sig_info[mod_sig];
    }
    return T.sig_info[i == n_keep ? s_new0 : s_new1];
  }
};

__device__ __forceinline__ const uint32_t* view_nsk(const VirtView& V) { return V.nsk; }

// The d = 1 sweep over the parent positions whose node can move (>= 2 rows, not an input, not
// skipped by the kind's exact shortcut: k_price_nsk), in order, with the candidate's dropped
// positions cleared and its rewritten node always visited (sweep_node re-checks every node, so
// a superset is exact).  The other nodes of the dense sweep do nothing but count, so the result
// is the dense sweep's bit for bit; the new nodes (ids n_keep, n_keep + 1) follow densely.
template <class F>
__device__ __forceinline__ void sparse_sweep(const VirtView& V, unsigned mask, bool running, const uint32_t* nsk,
                                             const Tables& T, F&& sweep_node, int& n_dense0) {
  const int npp = V.n_keep + (V.drop0 >= 0 ? 1 : 0) + (V.drop1 >= 0 ? 1 : 0);
  const int nwm = (int)__reduce_max_sync(mask, (unsigned)((npp + 31) >> 5));
  for (int w = 0; w < nwm; ++w) {
    uint32_t x = 0;
    if (running && 32 * w < npp) {
      x = nsk[w];
      if (V.drop0 >= 0 && (V.drop0 >> 5) == w) x &= ~(1u << (V.drop0 & 31));
      if (V.drop1 >= 0 && (V.drop1 >> 5) == w) x &= ~(1u << (V.drop1 & 31));
      if (V.mod >= 0 && (V.mod >> 5) == w) x |= 1u << (V.mod & 31);
    }
    for (uint32_t u = __reduce_or_sync(mask, x); u; u &= u - 1u) {  // warp-uniform, ascending
      const int b = __ffs(u) - 1;
      if ((x >> b) & 1u) {
        const int pp = 32 * w + b;
        const int i = pp - (V.drop0 >= 0 && pp > V.drop0 ? 1 : 0) - (V.drop1 >= 0 && pp > V.drop1 ? 1 : 0);
        sweep_node(i, pp == V.mod ? T.sig_info[V.mod_sig] : make_uint2(V.p_ro[pp], V.p_rn[pp]));
      }
    }
  }
  n_dense0 = V.n_keep;
}

// per parent: bit pp set when the d = 1 sweep can move node pp (price_d1's own test)
template <int KIND>
__global__ void k_price_nsk(PriceArgs PA, const unsigned long long* parent_addr, const uint32_t* pscratch,
                            uint64_t pstride, uint32_t n_parents, uint32_t W, uint32_t* nsk) {
  const Geo& G = PA.g;
  const uint32_t skip = d1_skip_bits<KIND>(PA.pp);
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t pi = blockIdx.x; pi < n_parents; pi += gridDim.x) {
    Rec R{reinterpret_cast<char*>(parent_addr[pi])};
    const uint32_t n = (uint32_t)R.h().n;
    const uint32_t* p_rn = pscratch + (uint64_t)pi * pstride + 7ull * G.cap_nodes + 1 + 2ull * G.cap_refs + G.cap_nodes;
    for (uint32_t w = wid; w < W; w += nwarps) {
      const uint32_t pp = 32u * w + lane;
      bool mv = false;
      if (pp < n) {
        const uint32_t y = p_rn[pp], nr = y & kInfoRows;
        mv = !(nr < 2u || (y & kInfoInput) || (skip && (y & skip) == skip));
      }
      const uint32_t word = __ballot_sync(0xffffffffu, mv);
      if (lane == 0) nsk[(uint64_t)pi * W + w] = word;
    }
  }
}

struct VPriceArgs {
  const uint32_t* nsk;  // [parent][nsk_W] k_price_nsk, or null
  uint32_t nsk_W;
  PriceArgs pa;
  const uint32_t* pscratch;
  uint64_t pstride;
  const VPlan* plan;
  const unsigned long long* parent_addr;
  uint8_t* alg8;  // [total][S]: assignment per child node of every priced candidate
  uint8_t* algt;  // rows > 256: the sweep's rows interleaved per warp (lane-minor), one per thread
  uint32_t S;
  ef_cand_result* out;  // speculative pricing: results by candidate here, not in pa.res (null: pa.res)
};

// one thread per survivor of the step's dedup (the compacted list); KIND < 0: any cost kind / radius
template <int KIND, bool SM_ROW>
__global__ void __launch_bounds__(EF_PRICE_THREADS) k_price_v(VPriceArgs A, const uint32_t* plist, const uint32_t* plist_n) {
  extern __shared__ uint8_t sm_alg[];  // SM_ROW: the sweep's row, one column per thread (S x 64 bytes)
  const Geo& G = A.pa.g;
  const uint32_t total = *plist_n;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t span = (total + 31) / 32 * 32;  // whole warps iterate together
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < span; k += stride) {
    const unsigned mask = __ballot_sync(0xffffffffu, k < total);
    if (k >= total) continue;
    const uint32_t c = plist[k];
    ef_cand_result& res = A.out ? A.out[c] : A.pa.res[c];
    const VPlan& P = A.plan[c];
    Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
    VirtView V;
    V.nsk = A.nsk ? A.nsk + (uint64_t)P.parent * A.nsk_W : nullptr;
    V.psig = R.sig(G);
    V.p_ro = A.pscratch + (uint64_t)P.parent * A.pstride + 7ull * G.cap_nodes + 1 + 2ull * G.cap_refs;
    V.p_rn = V.p_ro + G.cap_nodes;
    V.drop0 = P.drop0;
    V.drop1 = P.drop1;
    V.mod = P.mod;
    V.n_keep = P.n_keep;
    V.mod_sig = P.mod_sig;
    V.s_new0 = P.live[0] ? P.new_sig[0] : P.new_sig[1];
    V.s_new1 = P.new_sig[1];
    V.n = P.n_keep + P.n_live;
    uint8_t* alg = A.alg8 + (uint64_t)c * A.S;
    const uint32_t skip = d1_skip_bits<KIND>(A.pa.pp);
    if (KIND >= 0 && SM_ROW) {
      for (int i = 0; i < V.n; ++i) sm_alg[i * EF_PRICE_THREADS + threadIdx.x] = 0;
      price_d1<KIND>(A.pa, V, AlgRow{sm_alg + threadIdx.x, EF_PRICE_THREADS}, res, mask, skip);
      for (int i = 0; i < V.n; ++i) alg[i] = sm_alg[i * EF_PRICE_THREADS + threadIdx.x];
    } else if (KIND >= 0 && A.algt) {  // the row interleaved across the warp: accesses coalesce
      const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
      uint8_t* col = A.algt + (uint64_t)(gt >> 5) * 32u * A.S + (gt & 31u);
      for (int i = 0; i < V.n; ++i) col[i * 32] = 0;
      price_d1<KIND>(A.pa, V, AlgRow{col, 32}, res, mask, skip);
      for (int i = 0; i < V.n; ++i) alg[i] = col[i * 32];
    } else if (KIND >= 0) {  // the step cleared the rows (alg8)
      price_d1<KIND>(A.pa, V, AlgRow{alg, 1}, res, mask, skip);
    } else {
      price_graph(A.pa, V, alg, res);
    }
  }
}

// k_price_v with PL lanes per candidate (price_d1_lanes): a group of PL lanes prices one
// candidate of the list; the sweep's row of each group lives in shared memory when `smrow`
// (S bytes per group), else in the candidate's global alg8 row.
template <int KIND, int PL>
__global__ void __launch_bounds__(EF_PRICE_THREADS) k_price_lanes(VPriceArgs A, const uint32_t* plist,
                                                                  const uint32_t* plist_n, int smrow) {
  extern __shared__ uint8_t sm_rows[];
  const Geo& G = A.pa.g;
  const uint32_t total = *plist_n;
  const uint32_t lane = threadIdx.x & 31u, sl = lane % PL, gbase = lane - sl;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr uint32_t GPW = 32 / PL;
  uint8_t* srow = sm_rows + (uint64_t)(threadIdx.x / PL) * A.S;
  const uint32_t skip = d1_skip_bits<KIND>(A.pa.pp);
  for (uint32_t base = gw * GPW; base < total; base += nwarps * GPW) {  // warp-uniform
    const uint32_t kk = base + lane / PL;
    const bool valid = kk < total;
    const uint32_t c = valid ? plist[kk] : 0u;
    VirtView V{};
    V.n = 0;
    uint8_t* alg = A.alg8 + (uint64_t)c * A.S;
    ef_cand_result* res = nullptr;
    if (valid) {
      res = A.out ? A.out + c : A.pa.res + c;
      const VPlan& P = A.plan[c];
      Rec R{reinterpret_cast<char*>(A.parent_addr[P.parent])};
      V.psig = R.sig(G);
      V.p_ro = A.pscratch + (uint64_t)P.parent * A.pstride + 7ull * G.cap_nodes + 1 + 2ull * G.cap_refs;
      V.p_rn = V.p_ro + G.cap_nodes;
      V.drop0 = P.drop0;
      V.drop1 = P.drop1;
      V.mod = P.mod;
      V.n_keep = P.n_keep;
      V.mod_sig = P.mod_sig;
      V.s_new0 = P.live[0] ? P.new_sig[0] : P.new_sig[1];
      V.s_new1 = P.new_sig[1];
      V.n = P.n_keep + P.n_live;
    }
    uint8_t* row = smrow ? srow : alg;
    for (int i = (int)sl; i < V.n; i += PL) row[i] = 0;  // row 0 everywhere (price_d1 writes changes only)
    __syncwarp();
    price_d1_lanes<KIND, PL>(A.pa, V, AlgRow{row, 1}, res, valid, sl, gbase, skip);
    __syncwarp();
    if (smrow)
      for (int i = (int)sl; i < V.n; i += PL) alg[i] = row[i];
    __syncwarp();
  }
}

// Speculative pricing (large graphs): the candidates to price before deduplication is known,
// i.e. every complete candidate within the node cap (a superset of the survivors)
__global__ void k_spec_list(const ef_cand_result* res, uint32_t total, int32_t node_cap, uint32_t* list,
                            uint32_t* list_n, ef_cand_result* spec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t span = (total + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < span; c += gridDim.x * blockDim.x) {
    bool in = false;
    if (c < total) {
      spec[c].flags = 0;  // price_d1 ors PRICED / MISSING in
      in = !(res[c].flags & EF_F_INCOMPLETE) && res[c].n_compute <= node_cap;
    }
    const unsigned m = __ballot_sync(__activemask(), in);
    if (m) {
      uint32_t base = 0;
      const int leader = __ffs(m) - 1;
      if ((int)lane == leader) base = atomicAdd(list_n, (uint32_t)__popc(m));
      base = __shfl_sync(__activemask(), base, leader);
      if (in) list[base + __popc(m & ((1u << lane) - 1u))] = c;
    }
  }
}

// after the dedup: the speculative prices of the survivors (the candidates the dedup's list
// holds: FIRST -- PFIRST per parent -- not VISITED, not CAPPED) into the step's results;
// the others stay unpriced, exactly as if only the survivors had been priced
__global__ void k_spec_commit(ef_cand_result* res, const ef_cand_result* spec, uint32_t total, int per_parent) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    ef_cand_result& r = res[c];
    const uint32_t f = r.flags;
    const uint32_t first = per_parent ? EF_F_PFIRST : EF_F_FIRST;
    if ((f & EF_F_INCOMPLETE) || (f & (first | EF_F_VISITED | EF_F_CAPPED)) != first) continue;
    const ef_cand_result& x = spec[c];
    r.cost = x.cost;
    r.time_ms = x.time_ms;
    r.energy = x.energy;
    r.evals = x.evals;
    r.sweeps = x.sweeps;
    r.flags = f | (x.flags & (EF_F_PRICED | EF_F_MISSING));
  }
}

// copy the priced assignment of kept candidates into their materialised records
// (rows = 1: the step's rows hold row indices (price_d1): the algorithm ids are read from the
// signature's cost rows; 0: algorithm ids (price_graph))
__global__ void k_keep_alg(const uint8_t* alg8, uint32_t S, const uint32_t* cand, const unsigned long long* dst,
                           uint32_t n, Geo G, Tables T, int rows) {
  for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
    Rec C{reinterpret_cast<char*>(dst[k])};
    const int nn = C.h().n;
    const uint8_t* src = alg8 + (uint64_t)cand[k] * S;
    const uint32_t* sig = C.sig(G);
    uint8_t* out = C.alg(G);
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
      uint8_t a = src[i];
      if (rows) {
        const uint2 info = T.sig_info[sig[i]];
        a = (info.y & kInfoInput) ? 0 : (uint8_t)T.row_alg[info.x + a];
      }
      out[i] = a;
    }
  }
}

// ------------------------------------------------------------------------------------------
// hash-owner sharding: every candidate's (hash, global order) goes to rank hash % world,
// which decides first occurrence (smallest global order over all ranks) and membership in
// its shard of the visited set; the verdicts come back in send order.
// ------------------------------------------------------------------------------------------

struct RouteArgs {
  const ef_cand_result* res;
  uint32_t total, world;
  uint64_t order_base;
  uint32_t* count;   // [world]
  uint32_t* cursor;  // [world] exclusive offsets (host-computed), advanced by the scatter
  uint64_t* send;    // [n_send][2]
  uint32_t* perm;    // send position -> candidate
};

__device__ __forceinline__ uint32_t owner_of(uint64_t h, uint32_t world) { return (uint32_t)(h % world); }

// per-block owner histograms in shared memory, one global atomic per (block, owner)
__global__ void k_route_count(RouteArgs R) {
  extern __shared__ uint32_t hist[];
  for (uint32_t w = threadIdx.x; w < R.world; w += blockDim.x) hist[w] = 0;
  __syncthreads();
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < R.total; c += gridDim.x * blockDim.x) {
    const ef_cand_result& r = R.res[c];
    if (r.flags & EF_F_INCOMPLETE) continue;
    atomicAdd(&hist[owner_of(r.hash, R.world)], 1u);
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < R.world; w += blockDim.x)
    if (hist[w]) atomicAdd(&R.count[w], hist[w]);
}

// each block reserves its range per owner once, then its threads fill it
__global__ void k_route_scatter(RouteArgs R) {
  extern __shared__ uint32_t hist[];  // [world] counts, then [world] block bases
  uint32_t* base = hist + R.world;
  const uint32_t per = (R.total + gridDim.x - 1) / gridDim.x;  // contiguous candidates per block
  const uint32_t lo = blockIdx.x * per, hi = min(R.total, lo + per);
  for (uint32_t w = threadIdx.x; w < R.world; w += blockDim.x) hist[w] = 0;
  __syncthreads();
  for (uint32_t c = lo + threadIdx.x; c < hi; c += blockDim.x)
    if (!(R.res[c].flags & EF_F_INCOMPLETE)) atomicAdd(&hist[owner_of(R.res[c].hash, R.world)], 1u);
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < R.world; w += blockDim.x) {
    base[w] = hist[w] ? atomicAdd(&R.cursor[w], hist[w]) : 0u;
    hist[w] = 0;
  }
  __syncthreads();
  for (uint32_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    const ef_cand_result& r = R.res[c];
    if (r.flags & EF_F_INCOMPLETE) continue;
    const uint32_t o = owner_of(r.hash, R.world);
    const uint32_t pos = base[o] + atomicAdd(&hist[o], 1u);
    R.send[2 * (uint64_t)pos] = r.hash;
    R.send[2 * (uint64_t)pos + 1] = R.order_base + c;
    R.perm[pos] = c;
  }
}

struct OwnerArgs {
  const uint64_t* recv;  // [n][2] (hash, global order)
  uint32_t n;
  uint32_t* verdict;     // [n] EF_F_FIRST | EF_F_VISITED
  unsigned long long* key;
  unsigned long long* ord;
  uint32_t mask;
  unsigned long long* vis_key;
  uint32_t vis_mask;
  unsigned long long* vis_count;
  uint32_t* err;  // bit 8: visited shard full
};

__global__ void k_owner_claim(OwnerArgs O) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    uint32_t s = (uint32_t)mix64(h) & O.mask;
    for (uint32_t probe = 0; probe <= O.mask; ++probe, s = (s + 1) & O.mask) {
      const unsigned long long prev = atomicCAS(&O.key[s], 0ULL, key);
      if (prev == 0ULL || prev == key) {
        atomicMin(&O.ord[s], (unsigned long long)O.recv[2 * (uint64_t)i + 1]);
        break;
      }
    }
  }
}

__global__ void k_owner_resolve(OwnerArgs O) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    unsigned long long first = ~0ULL;
    uint32_t s = (uint32_t)mix64(h) & O.mask;
    for (uint32_t probe = 0; probe <= O.mask; ++probe, s = (s + 1) & O.mask) {
      if (O.key[s] == key) {
        first = O.ord[s];
        break;
      }
    }
    uint32_t v = first == O.recv[2 * (uint64_t)i + 1] ? EF_F_FIRST : 0u;
    if (vis_contains(O.vis_key, O.vis_mask, key, h)) v |= EF_F_VISITED;
    O.verdict[i] = v;
  }
}

__global__ void k_owner_insert(OwnerArgs O) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    if (O.verdict[i] != EF_F_FIRST) continue;
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    if (!vis_insert(O.vis_key, O.vis_mask, O.vis_count, key, h)) atomicOr(O.err, 8u);
  }
}

// fixed-capacity buckets: pair k of owner o at o * cap + k; one warp-aggregated atomic per
// owner present in the warp.  perm[o * cap + k] = candidate (the bucket's order does not
// matter: the owner decides first occurrence by the global order carried in the pair)
__global__ void k_route_pad(RouteArgs R, uint32_t cap) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t span = (R.total + 31) / 32 * 32;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < span; c += gridDim.x * blockDim.x) {
    const bool live = c < R.total && !(R.res[c].flags & EF_F_INCOMPLETE);
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (!live) continue;
    const uint64_t h = R.res[c].hash;
    const uint32_t o = owner_of(h, R.world);
    const unsigned peers = __match_any_sync(act, o);
    const uint32_t leader = (uint32_t)(__ffs(peers) - 1);
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&R.count[o], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const uint32_t k = base + __popc(peers & ((1u << lane) - 1u));  // < cap: cap >= candidates
    const uint64_t pos = (uint64_t)o * cap + k;
    R.send[2 * pos] = h;
    R.send[2 * pos + 1] = R.order_base + c;
    R.perm[pos] = c;
  }
}

// padded receive buffers: slot i is valid iff i % cap < counts[i / cap]; invalid verdicts are 0
__global__ void k_owner_claim_pad(OwnerArgs O, const uint32_t* counts, uint32_t cap) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    if (i % cap >= counts[i / cap]) continue;
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    uint32_t s = (uint32_t)mix64(h) & O.mask;
    for (uint32_t probe = 0; probe <= O.mask; ++probe, s = (s + 1) & O.mask) {
      const unsigned long long prev = atomicCAS(&O.key[s], 0ULL, key);
      if (prev == 0ULL || prev == key) {
        atomicMin(&O.ord[s], (unsigned long long)O.recv[2 * (uint64_t)i + 1]);
        break;
      }
    }
  }
}

__global__ void k_owner_resolve_pad(OwnerArgs O, const uint32_t* counts, uint32_t cap) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    if (i % cap >= counts[i / cap]) {
      O.verdict[i] = 0;
      continue;
    }
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    unsigned long long first = ~0ULL;
    uint32_t s = (uint32_t)mix64(h) & O.mask;
    for (uint32_t probe = 0; probe <= O.mask; ++probe, s = (s + 1) & O.mask) {
      if (O.key[s] == key) {
        first = O.ord[s];
        break;
      }
    }
    uint32_t v = first == O.recv[2 * (uint64_t)i + 1] ? EF_F_FIRST : 0u;
    if (vis_contains(O.vis_key, O.vis_mask, key, h)) v |= EF_F_VISITED;
    O.verdict[i] = v;
  }
}

__global__ void k_owner_insert_pad(OwnerArgs O, const uint32_t* counts, uint32_t cap) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < O.n; i += gridDim.x * blockDim.x) {
    if (i % cap >= counts[i / cap] || O.verdict[i] != EF_F_FIRST) continue;
    const uint64_t h = O.recv[2 * (uint64_t)i];
    const unsigned long long key = h ? h : 0x8000000000000000ULL;
    if (!vis_insert(O.vis_key, O.vis_mask, O.vis_count, key, h)) atomicOr(O.err, 8u);
  }
}

// verdicts in the padded send layout -> candidate flags and node cap
__global__ void k_apply_verdicts_pad(ef_cand_result* res, const uint32_t* perm, const uint32_t* counts,
                                     const uint32_t* verdict, uint32_t world, uint32_t cap, int node_cap) {
  const uint64_t n = (uint64_t)world * cap;
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i % cap >= counts[i / cap]) continue;
    const uint32_t c = perm[i];
    uint32_t f = res[c].flags | (verdict[i] & (EF_F_FIRST | EF_F_VISITED));
    if (res[c].n_compute > node_cap) f |= EF_F_CAPPED;
    res[c].flags = f;
  }
}

// verdicts (send order) -> candidate flags and node cap
__global__ void k_apply_verdicts(ef_cand_result* res, const uint32_t* perm, const uint32_t* verdict, uint32_t n,
                                 int node_cap) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t c = perm[i];
    uint32_t f = res[c].flags | (verdict[i] & (EF_F_FIRST | EF_F_VISITED));
    if (res[c].n_compute > node_cap) f |= EF_F_CAPPED;
    res[c].flags = f;
  }
}

// survivors in candidate order (neighbouring lanes price siblings of one parent)
__global__ void k_compact_survivors(const ef_cand_result* res, uint32_t total, uint32_t* plist, uint32_t* plist_n) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t span = (total + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < span; c += gridDim.x * blockDim.x) {
    const bool survivor =
        c < total && (res[c].flags & (EF_F_INCOMPLETE | EF_F_FIRST | EF_F_VISITED | EF_F_CAPPED)) == EF_F_FIRST;
    const unsigned m = __ballot_sync(0xffffffffu, survivor);
    if (m) {
      uint32_t base = 0;
      const int leader = __ffs(m) - 1;
      if ((int)lane == leader) base = atomicAdd(plist_n, (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (survivor) plist[base + __popc(m & ((1u << lane) - 1u))] = c;
    }
  }
}

// ------------------------------------------------------------------------------------------
// packed record upload: per record [n, n_refs, n_out, n_compute] then nid[n] sig[n] aux[n]
// nin[n] inoff[n+1] topo[n] refs[n_refs] outs[n_out] (uint32), scattered into the slots
// ------------------------------------------------------------------------------------------

__global__ void k_unpack(const uint8_t* blob, const unsigned long long* off, const unsigned long long* dst,
                         uint32_t n, Geo G) {
  for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(blob + off[r]);
    Rec R{reinterpret_cast<char*>(dst[r])};
    const uint32_t nn = p[0], nr = p[1], no = p[2];
    if (threadIdx.x < 16) reinterpret_cast<uint32_t*>(R.p)[threadIdx.x] = threadIdx.x < 4 ? p[threadIdx.x] : 0u;
    const uint32_t* q = p + 4;
    for (uint32_t i = threadIdx.x; i < nn; i += blockDim.x) {
      R.nid(G)[i] = (int32_t)q[i];
      R.sig(G)[i] = q[nn + i];
      R.aux(G)[i] = q[2 * nn + i];
      R.nin(G)[i] = q[3 * nn + i];
      R.inoff(G)[i] = q[4 * nn + i];
      R.topo(G)[i] = q[5 * nn + 1 + i];
      R.alg(G)[i] = 0;
    }
    if (threadIdx.x == 0) R.inoff(G)[nn] = q[5 * nn];
    const uint32_t* rq = q + 6 * nn + 1;
    for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) R.refs(G)[i] = rq[i];
    for (uint32_t i = threadIdx.x; i < no; i += blockDim.x) R.outs(G)[i] = rq[nr + i];
  }
}

// register-only BLAKE2b compressions: the ALU roofline of the hash kernels on this GPU
__global__ void __launch_bounds__(128) k_b2b_peak(uint64_t* out, int iters) {
  uint64_t h[8], m[16];
  for (int i = 0; i < 16; ++i) m[i] = (uint64_t)(threadIdx.x + 131 * blockIdx.x) * 0x9e3779b97f4a7c15ULL + i;
  for (int i = 0; i < 8; ++i) h[i] = b2b_iv(i);
  for (int r = 0; r < iters; ++r) {
    b2b_compress(h, m, 128, false);
    m[r & 15] ^= h[0];
  }
  uint64_t x = 0;
  for (int i = 0; i < 8; ++i) x ^= h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

// div_pre (the pricing's division by a normalisation reference) against the IEEE division:
// n random dividends per divisor -- uniform exponents in [-500, 500] and random significands,
// every 4th one with an all-ones / all-zeros low significand (the rounding boundaries) -- plus
// zeros; a mismatch is any bit difference
__global__ void k_div_check(const double* ys, uint32_t nys, uint64_t n, uint64_t seed,
                            unsigned long long* mismatches) {
  unsigned long long bad = 0;
  const uint64_t total = n * nys;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const double y = ys[t % nys];
    uint64_t z = (t + 1) * 0x9e3779b97f4a7c15ULL ^ seed;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    uint64_t mant = z & 0xfffffffffffffULL;
    const uint32_t sel = (uint32_t)(z >> 52) & 3u;
    if (sel == 1) mant |= 0xffffffULL;                  // low bits all ones
    if (sel == 2) mant &= ~0xffffffULL;                 // low bits all zeros
    const int64_t ex = (int64_t)((z >> 54) % 1001) - 500 + 1023;
    double x = __longlong_as_double((long long)(((uint64_t)ex << 52) | mant));
    if ((t & 1023) == 7) x = 0.0;
    if (z >> 63) x = -x;
    const double got = div_pre(x, y, rcp_or_zero(y)), want = x / y;
    bad += __double_as_longlong(got) != __double_as_longlong(want);
  }
  if (bad) atomicAdd(mismatches, bad);
}

}  // namespace ef
