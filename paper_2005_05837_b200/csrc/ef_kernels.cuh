// Kernels shared by the frontier step (ef_step.cuh) and the tables: rule matching, rewrite
// planning / record materialisation, dedup, pricing, weight-set derivation and digests.
//
//   k_match        one CTA per parent graph: use counts, consumer CSR and inverse topological
//                  order, then every rule at every node, emitted in the reference's site order
//                  (rules.py:147-331 matchers) with block-wide scans.
//   plan_rewrite   the rewrite of one site in parent coordinates (rules.py:164-331).
//   k_materialise  one CTA per KEPT candidate: copies the parent record applying the rewrite;
//                  child positions / offsets are closed-form in the <= 2 dropped nodes, so the
//                  copy is a single coalesced pass.
//   k_dedup_*      open-addressing tables: first occurrence inside the step (atomicMin on the
//                  candidate's sequence number) and membership in the visited set.
//   price_d1 /     the reference's first-improvement sweep (search.py:106-153) with CPython's
//   price_graph    Neumaier sum for the start totals; every floating-point operation in the
//                  reference's order, no FMA contraction (the library builds with --fmad=false).
//   k_derive       derived weight tensors (rules.py:231-232, 272-276, 326-327); their BLAKE2b
//                  digests (graph.py:510-517) are taken on host cores (ef_tables_commit).
#pragma once
#include <math_constants.h>
#include <stdint.h>

#include "ef_device.cuh"

namespace ef {

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------

template <int BT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, uint32_t* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < BT / 32 ? sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < BT / 32) sh[lane] = s;
    if (lane == BT / 32 - 1) sh[BT / 32] = s;
  }
  __syncthreads();
  uint32_t ex = x - v + (wid > 0 ? sh[wid - 1] : 0u);
  *total = sh[BT / 32];
  __syncthreads();
  return ex;
}

__device__ __forceinline__ uint32_t lookup_sig(const Tables& T, const ef_sig_desc& d) {
  uint64_t k = desc_key(d);
  uint32_t m = T.sig_ht_mask;
  if (m == 0) return kNone;
  uint32_t s = (uint32_t)k & m;
  for (uint32_t probe = 0; probe <= m; ++probe, s = (s + 1) & m) {
    unsigned long long kk = T.sig_ht_key[s];
    if (kk == 0ULL) return kNone;
    if (kk == k) {
      uint32_t id = T.sig_ht_val[s];
      if (desc_eq(T.sig_desc[id], d)) return id;
    }
  }
  return kNone;
}

__device__ __forceinline__ uint32_t lookup_derive(const Tables& T, int32_t op, uint32_t a, uint32_t b, int32_t s0) {
  uint64_t k = derive_key(op, a, b, s0);
  uint32_t m = T.dv_ht_mask;
  if (m == 0) return kNone;
  uint32_t s = (uint32_t)k & m;
  for (uint32_t probe = 0; probe <= m; ++probe, s = (s + 1) & m) {
    unsigned long long kk = T.dv_ht_key[s];
    if (kk == 0ULL) return kNone;
    if (kk == k) {
      uint32_t id = T.dv_ht_val[s];
      const int32_t* t = T.dv_tuple + 4 * id;
      if (t[0] == op && (uint32_t)t[1] == a && (uint32_t)t[2] == b && t[3] == s0) return id;
    }
  }
  return kNone;
}

__device__ __forceinline__ bool conv_compatible(const ef_sig_desc& a, const ef_sig_desc& b) {
  // rules.py:197 _CONV_MERGE_KEYS = kernel, stride, padding, has_activation
  return a.kh == b.kh && a.kw == b.kw && a.sh == b.sh && a.sw == b.sw && a.ph == b.ph && a.pw == b.pw &&
         a.act == b.act;
}

__device__ __forceinline__ ef_sig_desc conv_variant(const ef_sig_desc& c, int act, int oc) {
  ef_sig_desc d = c;
  d.act = act;
  d.oc = oc;
  d.out[1] = oc;
  return d;
}

__device__ __forceinline__ ef_sig_desc relu_of(const ef_sig_desc& conv) {
  ef_sig_desc d;
  int32_t* w = reinterpret_cast<int32_t*>(&d);
  for (int i = 0; i < (int)(sizeof(ef_sig_desc) / 4); ++i) w[i] = 0;
  d.kind = EF_K_RELU;
  d.rank = 4;
  for (int i = 0; i < 4; ++i) d.in[i] = d.out[i] = conv.out[i];
  return d;
}

__device__ __forceinline__ ef_sig_desc split2_of(const ef_sig_desc& merged, int s0, int s1) {
  ef_sig_desc d;
  int32_t* w = reinterpret_cast<int32_t*>(&d);
  for (int i = 0; i < (int)(sizeof(ef_sig_desc) / 4); ++i) w[i] = 0;
  d.kind = EF_K_SPLIT;
  d.rank = 4;
  for (int i = 0; i < 4; ++i) d.in[i] = d.out[i] = merged.out[i];
  d.out[1] = s0;
  d.axis = 1;
  d.nsizes = 2;
  d.s0 = s0;
  d.s1 = s1;
  return d;
}

// ------------------------------------------------------------------------------------------
// step arguments
// ------------------------------------------------------------------------------------------

struct StepArgs {
  Geo g;
  Tables T;
  const unsigned long long* parent_addr;
  uint32_t n_parents;
  uint32_t* pscratch;  // per parent: u0 u1 coff[+1] ccur [cap] clist[cap_refs] tslot s_v s_pk [cap] rslot[cap_refs]
  uint64_t pstride;    // words per parent
  int32_t rules[8];
  int32_t n_rules;
  unsigned long long* sites;  // per parent site_cap packed sites
  uint32_t site_cap;
  uint32_t* site_count;  // per parent
  uint32_t* cand_off;    // n_parents + 1
  uint32_t* total;       // [0] = number of candidates
  uint32_t cand_cap;
  ef_cand_result* res;
  ef_sig_desc* req_sig;
  uint32_t* n_req_sig;
  uint32_t req_sig_cap;
  int32_t* req_dv;
  uint32_t* n_req_dv;
  uint32_t req_dv_cap;
  uint32_t* err;  // bit0 site overflow, bit1 candidate overflow, bit2 record capacity, bit3 hash capacity
  // keep mode of k_materialise: write candidates sel[i] into the records at dst[i]
  const uint32_t* sel;
  uint32_t n_sel;
  const unsigned long long* dst;
};

__device__ __forceinline__ unsigned long long pack_site(uint32_t rule, uint32_t a, uint32_t b) {
  return ((unsigned long long)rule << 56) | ((unsigned long long)(a & 0xfffffffu) << 28) | (b & 0xfffffffu);
}

// ------------------------------------------------------------------------------------------
// k_match: one CTA per parent
// ------------------------------------------------------------------------------------------

template <int BT>
__global__ void __launch_bounds__(BT) k_match(StepArgs A) {
  __shared__ uint32_t sh_scan[BT / 32 + 1];
  const Geo& G = A.g;
  const Tables& T = A.T;
  for (uint32_t pi = blockIdx.x; pi < A.n_parents; pi += gridDim.x) {
    Rec R{reinterpret_cast<char*>(A.parent_addr[pi])};
    const int n = R.h().n, n_out = R.h().n_out;
    const uint32_t* sig = R.sig(G);
    const uint32_t* inoff = R.inoff(G);
    const uint32_t* nin = R.nin(G);
    const uint32_t* refs = R.refs(G);
    const uint32_t* outs = R.outs(G);
    uint32_t* u0 = A.pscratch + (uint64_t)pi * A.pstride;
    uint32_t* u1 = u0 + G.cap_nodes;
    uint32_t* coff = u1 + G.cap_nodes;
    uint32_t* ccur = coff + G.cap_nodes + 1;
    uint32_t* clist = ccur + G.cap_nodes;
    uint32_t* tslot = clist + G.cap_refs;  // inverse topological order (k_plan)
    {
      const uint32_t* topo = R.topo(G);
      for (int s = threadIdx.x; s < n; s += BT) tslot[topo[s]] = (uint32_t)s;
    }

    for (int i = threadIdx.x; i < n; i += BT) u0[i] = u1[i] = ccur[i] = 0;
    __syncthreads();
    {  // slot-space tables of the parent for k_reach / k_dirty_warp: node + packed (ref offset, arity)
       // per topological slot, and every ref as (producer slot << 8 | port)
      uint32_t* s_v = tslot + G.cap_nodes;
      uint32_t* s_pk = s_v + G.cap_nodes;
      uint32_t* rslot = s_pk + G.cap_nodes;
      const uint32_t* topo = R.topo(G);
      for (int s = threadIdx.x; s < n; s += BT) {
        const uint32_t v = topo[s];
        s_v[s] = v;
        s_pk[s] = inoff[v] | (nin[v] << 24);
      }
      const int n_refs = R.h().n_refs;
      for (int r = threadIdx.x; r < n_refs; r += BT) rslot[r] = (tslot[refs[r] >> 8] << 8) | (refs[r] & 255u);
      // per-node price rows {row_off, row_n | is_input << 31} (k_price_v reads one word pair per node)
      uint32_t* p_ro = rslot + G.cap_refs;
      uint32_t* p_rn = p_ro + G.cap_nodes;
      for (int v = threadIdx.x; v < n; v += BT) {
        const uint2 info = T.sig_info[sig[v]];
        p_ro[v] = info.x;
        p_rn[v] = info.y;
      }
    }
    for (int i = threadIdx.x; i < n; i += BT) {
      for (uint32_t r = inoff[i]; r < inoff[i] + nin[i]; ++r) {
        uint32_t p = refs[r] >> 8, port = refs[r] & 255u;
        atomicAdd(&ccur[p], 1u);
        if (port == 0) atomicAdd(&u0[p], 1u);
        else if (port == 1) atomicAdd(&u1[p], 1u);
      }
    }
    for (int o = threadIdx.x; o < n_out; o += BT) {
      uint32_t p = outs[o] >> 8, port = outs[o] & 255u;
      if (port == 0) atomicAdd(&u0[p], kOutMark);
      else if (port == 1) atomicAdd(&u1[p], kOutMark);
    }
    __syncthreads();
    // consumer CSR: exclusive scan of per-producer counts
    uint32_t run = 0;
    for (int c0 = 0; c0 < n; c0 += BT) {
      int i = c0 + threadIdx.x;
      uint32_t v = i < n ? ccur[i] : 0u, tot;
      uint32_t ex = block_excl_scan<BT>(v, &tot, sh_scan);
      if (i < n) coff[i] = run + ex;
      run += tot;
    }
    if (threadIdx.x == 0) coff[n] = run;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += BT) ccur[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += BT) {
      for (uint32_t r = inoff[i]; r < inoff[i] + nin[i]; ++r) {
        uint32_t p = refs[r] >> 8;
        clist[coff[p] + atomicAdd(&ccur[p], 1u)] = (uint32_t)i;
      }
    }
    __syncthreads();
    for (int p = threadIdx.x; p < n; p += BT) {  // consumer lists in position (= id) order
      uint32_t b = coff[p], e = coff[p + 1];
      for (uint32_t x = b + 1; x < e; ++x) {
        uint32_t v = clist[x];
        uint32_t y = x;
        while (y > b && clist[y - 1] > v) {
          clist[y] = clist[y - 1];
          --y;
        }
        clist[y] = v;
      }
    }
    __syncthreads();

    unsigned long long* out = A.sites + (uint64_t)pi * A.site_cap;
    uint32_t base = 0;
    bool overflow = false;
    for (int ri = 0; ri < A.n_rules; ++ri) {
      const int rule = A.rules[ri];
      for (int c0 = 0; c0 < n; c0 += BT) {
        const int i = c0 + threadIdx.x;
        uint32_t cnt = 0, a = 0, b = 0;
        if (i < n) {
          const ef_sig_desc& di = T.sig_desc[sig[i]];
          const int kind = di.kind;
          if (rule == EF_R_FUSE_CONV_RELU || rule == EF_R_FUSE_CONV_BN || rule == EF_R_SPLIT_MERGED) {
            // rules.py:147-161 / 303-318 / 245-261: producer conv, sole consumer of its edge
            const int want = rule == EF_R_FUSE_CONV_RELU ? EF_K_RELU : rule == EF_R_FUSE_CONV_BN ? EF_K_BATCHNORM : EF_K_SPLIT;
            if (kind == want && (rule != EF_R_SPLIT_MERGED || (di.axis == 1 && di.nsizes == 2))) {
              uint32_t src = refs[inoff[i]];
              uint32_t p = src >> 8, port = src & 255u;
              const ef_sig_desc& dp = T.sig_desc[sig[p]];
              uint32_t uses = port == 0 ? u0[p] : (port == 1 ? u1[p] : 2u);
              if (dp.kind == EF_K_CONV2D && (rule == EF_R_SPLIT_MERGED || dp.act == 0) && uses == 1u) {
                cnt = 1;
                a = p;
                b = (uint32_t)i;
              }
            }
          } else if (rule == EF_R_SPLIT_CONV_ACT) {  // rules.py:173-178
            if (kind == EF_K_CONV2D && di.act) {
              cnt = 1;
              a = (uint32_t)i;
            }
          } else if (rule == EF_R_FOLD_IDENTITY) {  // rules.py:288-290
            if (kind == EF_K_IDENTITY) {
              cnt = 1;
              a = (uint32_t)i;
            }
          } else if (rule == EF_R_MERGE_CONVS) {  // rules.py:200-215: partners after i on the same edge
            if (kind == EF_K_CONV2D) {
              uint32_t src = refs[inoff[i]];
              uint32_t p = src >> 8;
              for (uint32_t x = coff[p]; x < coff[p + 1]; ++x) {
                uint32_t c = clist[x];
                if (c <= (uint32_t)i) continue;
                const ef_sig_desc& dc = T.sig_desc[sig[c]];
                if (dc.kind == EF_K_CONV2D && refs[inoff[c]] == src && conv_compatible(di, dc)) ++cnt;
              }
              a = (uint32_t)i;
            }
          }
        }
        uint32_t tot;
        uint32_t ex = block_excl_scan<BT>(cnt, &tot, sh_scan);
        if (cnt) {
          uint32_t at = base + ex;
          if (rule == EF_R_MERGE_CONVS) {
            uint32_t src = refs[inoff[i]];
            uint32_t p = src >> 8;
            const ef_sig_desc& di = T.sig_desc[sig[i]];
            for (uint32_t x = coff[p]; x < coff[p + 1]; ++x) {
              uint32_t c = clist[x];
              if (c <= (uint32_t)i) continue;
              const ef_sig_desc& dc = T.sig_desc[sig[c]];
              if (dc.kind == EF_K_CONV2D && refs[inoff[c]] == src && conv_compatible(di, dc)) {
                if (at < A.site_cap) out[at] = pack_site(rule, (uint32_t)i, c);
                ++at;
              }
            }
          } else if (at < A.site_cap) {
            out[at] = pack_site(rule, a, b);
          }
        }
        base += tot;
      }
    }
    if (base > A.site_cap) overflow = true;
    if (threadIdx.x == 0) {
      atomicMax(&A.total[5], (uint32_t)n);  // step-wide maxima size the candidate scratch
      atomicMax(&A.total[6], R.h().n_refs);
      atomicMax(&A.total[8], (uint32_t)n_out);
      A.site_count[pi] = overflow ? A.site_cap : base;
      if (overflow) atomicOr(A.err, 1u);
    }
    __syncthreads();
  }
}

// exclusive scan of per-parent site counts -> candidate offsets (single CTA)
template <int BT>
__global__ void __launch_bounds__(BT) k_offsets(StepArgs A) {
  __shared__ uint32_t sh_scan[BT / 32 + 1];
  uint32_t run = 0;
  for (uint32_t c0 = 0; c0 < A.n_parents; c0 += BT) {
    uint32_t i = c0 + threadIdx.x;
    uint32_t v = i < A.n_parents ? A.site_count[i] : 0u, tot;
    uint32_t ex = block_excl_scan<BT>(v, &tot, sh_scan);
    if (i < A.n_parents) A.cand_off[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) {
    A.cand_off[A.n_parents] = run;
    A.total[4] = run;  // requested count; the pipeline sees 0 when it does not fit (the step reruns)
    A.total[0] = run > A.cand_cap ? 0u : run;
    if (run > A.cand_cap) atomicOr(A.err, 2u);
  }
}

// ------------------------------------------------------------------------------------------
// k_materialise: one CTA per kept candidate (keep mode: sel -> dst records)
// ------------------------------------------------------------------------------------------

struct Plan {
  int drop[2];  // ascending, -1 = none
  int mod;      // position rewritten in place
  uint32_t mod_sig, mod_aux;
  int n_new;  // new nodes before pruning (ids max+1, max+2)
  int live[2];
  uint32_t new_sig[2], new_aux[2], new_ref[2];  // new_ref in parent space: pos >= n means new node
  int n_rm;
  uint32_t rm_from[2], rm_to[2];
  int topo_node, topo_mode;  // 1 = emit node then new nodes, 2 = emit new nodes in its place
  int slot_of[3];            // topo slots of: drop[0], drop[1], topo_node
  int n_live;
  uint32_t touched[2];
  int incomplete;
  int drop_refs[2];  // ref ranges of the dropped nodes
  uint32_t drop_inoff[2];
};

__device__ void plan_rewrite(const StepArgs& A, Plan& P, Rec R, int n, uint32_t rule, uint32_t a, uint32_t b,
                             const uint32_t* u0, const uint32_t* u1) {
  const Geo& G = A.g;
  const Tables& T = A.T;
  const uint32_t* sig = R.sig(G);
  const uint32_t* aux = R.aux(G);
  const uint32_t* refs = R.refs(G);
  const uint32_t* inoff = R.inoff(G);
  P.drop[0] = P.drop[1] = -1;
  P.mod = -1;
  P.n_new = 0;
  P.live[0] = P.live[1] = 0;
  P.n_rm = 0;
  P.topo_node = -1;
  P.topo_mode = 0;
  P.touched[0] = P.touched[1] = kNone;
  P.incomplete = 0;
  auto need_sig = [&](const ef_sig_desc& d) -> uint32_t {
    uint32_t id = lookup_sig(T, d);
    if (id == kNone) {
      P.incomplete = 1;
      uint32_t k = atomicAdd(A.n_req_sig, 1u);
      if (k < A.req_sig_cap) A.req_sig[k] = d;
    }
    return id;
  };
  auto need_dv = [&](int32_t op, uint32_t x, uint32_t y, int32_t s0) -> uint32_t {
    uint32_t id = lookup_derive(T, op, x, y, s0);
    if (id == kNone) {
      P.incomplete = 1;
      uint32_t k = atomicAdd(A.n_req_dv, 1u);
      if (k < A.req_dv_cap) {
        A.req_dv[4 * k] = op;
        A.req_dv[4 * k + 1] = (int32_t)x;
        A.req_dv[4 * k + 2] = (int32_t)y;
        A.req_dv[4 * k + 3] = s0;
      }
    }
    return id;
  };
  const ef_sig_desc& da = T.sig_desc[sig[a]];
  switch (rule) {
    case EF_R_FUSE_CONV_RELU:  // rules.py:164-170
      P.drop[0] = (int)b;
      P.mod = (int)a;
      P.mod_sig = need_sig(conv_variant(da, 1, da.oc));
      P.mod_aux = aux[a];
      P.n_rm = 1;
      P.rm_from[0] = b << 8;
      P.rm_to[0] = a << 8;
      P.touched[0] = P.mod_sig;
      break;
    case EF_R_SPLIT_CONV_ACT: {  // rules.py:181-190
      P.mod = (int)a;
      P.mod_sig = need_sig(conv_variant(da, 0, da.oc));
      P.mod_aux = aux[a];
      P.n_new = 1;
      P.live[0] = 1;
      P.new_sig[0] = need_sig(relu_of(da));
      P.new_aux[0] = kEmptyWset;
      P.new_ref[0] = a << 8;
      P.n_rm = 1;
      P.rm_from[0] = a << 8;
      P.rm_to[0] = (uint32_t)n << 8;
      P.topo_node = (int)a;
      P.topo_mode = 1;
      P.touched[0] = P.mod_sig;
      P.touched[1] = P.new_sig[0];
      break;
    }
    case EF_R_MERGE_CONVS: {  // rules.py:225-242
      const ef_sig_desc& dbb = T.sig_desc[sig[b]];
      ef_sig_desc dm = conv_variant(da, da.act, da.oc + dbb.oc);
      P.drop[0] = (int)a;
      P.drop[1] = (int)b;
      P.n_new = 2;
      P.live[0] = P.live[1] = 1;
      P.new_sig[0] = need_sig(dm);
      P.new_aux[0] = need_dv(EF_D_MERGE, aux[a], aux[b], 0);
      P.new_ref[0] = refs[inoff[a]];
      P.new_sig[1] = need_sig(split2_of(dm, da.oc, dbb.oc));
      P.new_aux[1] = kEmptyWset;
      P.new_ref[1] = (uint32_t)n << 8;
      P.n_rm = 2;
      P.rm_from[0] = a << 8;
      P.rm_to[0] = ((uint32_t)(n + 1) << 8);
      P.rm_from[1] = b << 8;
      P.rm_to[1] = ((uint32_t)(n + 1) << 8) | 1u;
      P.topo_mode = 2;  // topo_node chosen once the slots of a and b are known
      P.touched[0] = P.new_sig[0];
      P.touched[1] = P.new_sig[1];
      break;
    }
    case EF_R_SPLIT_MERGED: {  // rules.py:264-281
      const ef_sig_desc& ds = T.sig_desc[sig[b]];
      P.drop[0] = (int)a;
      P.drop[1] = (int)b;
      P.n_new = 2;
      // _rebuild prunes a half whose split port feeds nothing
      P.live[0] = u0[b] != 0u;
      P.live[1] = u1[b] != 0u;
      if (P.live[0]) {
        P.new_sig[0] = need_sig(conv_variant(da, da.act, ds.s0));
        P.new_aux[0] = need_dv(EF_D_SLICE_LO, aux[a], 0, ds.s0);
        P.touched[0] = P.new_sig[0];
      }
      if (P.live[1]) {
        P.new_sig[1] = need_sig(conv_variant(da, da.act, ds.s1));
        P.new_aux[1] = need_dv(EF_D_SLICE_HI, aux[a], 0, ds.s0);
        P.touched[1] = P.new_sig[1];
      }
      P.new_ref[0] = P.new_ref[1] = refs[inoff[a]];
      P.n_rm = 2;
      P.rm_from[0] = b << 8;
      P.rm_to[0] = (uint32_t)n << 8;
      P.rm_from[1] = (b << 8) | 1u;
      P.rm_to[1] = (uint32_t)(n + 1) << 8;
      P.topo_node = (int)a;
      P.topo_mode = 2;
      break;
    }
    case EF_R_FOLD_IDENTITY:  // rules.py:293-296
      P.drop[0] = (int)a;
      P.n_rm = 1;
      P.rm_from[0] = a << 8;
      P.rm_to[0] = refs[inoff[a]];
      break;
    case EF_R_FUSE_CONV_BN:  // rules.py:321-331
      P.drop[0] = (int)b;
      P.mod = (int)a;
      P.mod_sig = sig[a];
      P.mod_aux = need_dv(EF_D_FOLD, aux[a], aux[b], 0);
      P.n_rm = 1;
      P.rm_from[0] = b << 8;
      P.rm_to[0] = a << 8;
      break;
  }
  if (P.drop[0] > P.drop[1] && P.drop[1] >= 0) {
    int t = P.drop[0];
    P.drop[0] = P.drop[1];
    P.drop[1] = t;
  }
  if (P.drop[0] < 0 && P.drop[1] >= 0) {
    P.drop[0] = P.drop[1];
    P.drop[1] = -1;
  }
  P.n_live = P.live[0] + P.live[1];
}

template <int BT>
__global__ void __launch_bounds__(BT) k_materialise(StepArgs A) {
  __shared__ Plan P;
  const Geo& G = A.g;
  for (uint32_t ci = blockIdx.x; ci < A.n_sel; ci += gridDim.x) {
    const uint32_t c = A.sel[ci];
    // parent of candidate c: last pi with cand_off[pi] <= c
    uint32_t lo = 0, hi = A.n_parents;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (A.cand_off[mid] <= c) lo = mid;
      else hi = mid;
    }
    const uint32_t pi = lo;
    const unsigned long long site = A.sites[(uint64_t)pi * A.site_cap + (c - A.cand_off[pi])];
    const uint32_t rule = (uint32_t)(site >> 56), sa = (uint32_t)(site >> 28) & 0xfffffffu, sb = (uint32_t)site & 0xfffffffu;
    Rec R{reinterpret_cast<char*>(A.parent_addr[pi])};
    Rec C{reinterpret_cast<char*>(A.dst[ci])};
    const int n = R.h().n, n_refs = R.h().n_refs, n_out = R.h().n_out;
    const uint32_t* u0 = A.pscratch + (uint64_t)pi * A.pstride;
    const uint32_t* u1 = u0 + G.cap_nodes;
    const uint32_t* pnin = R.nin(G);
    const uint32_t* pinoff = R.inoff(G);
    if (threadIdx.x == 0) {
      plan_rewrite(A, P, R, n, rule, sa, sb, u0, u1);
      P.slot_of[0] = P.slot_of[1] = P.slot_of[2] = -1;
      for (int k = 0; k < 2; ++k) {
        P.drop_refs[k] = P.drop[k] >= 0 ? (int)pnin[P.drop[k]] : 0;
        P.drop_inoff[k] = P.drop[k] >= 0 ? pinoff[P.drop[k]] : 0xffffffffu;
      }
    }
    __syncthreads();
    // topo slots of the special nodes
    {
      const uint32_t* ptopo = R.topo(G);
      for (int s = threadIdx.x; s < n; s += BT) {
        int v = (int)ptopo[s];
        if (v == P.drop[0]) P.slot_of[0] = s;
        if (v == P.drop[1]) P.slot_of[1] = s;
        if (P.topo_mode == 2 && rule == EF_R_MERGE_CONVS) {
          // merged conv + split go where the earlier of left/right was (both are dropped)
        } else if (v == P.topo_node) {
          P.slot_of[2] = s;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && rule == EF_R_MERGE_CONVS) {
      P.topo_node = P.slot_of[0] < P.slot_of[1] ? P.drop[0] : P.drop[1];
      P.slot_of[2] = min(P.slot_of[0], P.slot_of[1]);
    }
    __syncthreads();
    const int n_keep = n - (P.drop[0] >= 0) - (P.drop[1] >= 0);
    const int n_child = n_keep + P.n_live;
    const int drop_ref_tot = P.drop_refs[0] + P.drop_refs[1];
    const int n_refs_child = n_refs - drop_ref_tot + P.n_live;
    const bool fits = n_child <= (int)G.cap_nodes && n_refs_child <= (int)G.cap_refs;
    if (!fits) {
      if (threadIdx.x == 0) atomicOr(A.err, 4u);
      __syncthreads();
      continue;
    }
    const int d0 = P.drop[0], d1 = P.drop[1];
    // child position of a parent-space ref target
    auto cpos = [&](uint32_t ppos) -> uint32_t {
      if (ppos >= (uint32_t)n) {
        uint32_t k = ppos - (uint32_t)n;
        return (uint32_t)n_keep + (k == 1 ? (uint32_t)P.live[0] : 0u);
      }
      return ppos - (uint32_t)(d0 >= 0 && (uint32_t)d0 < ppos) - (uint32_t)(d1 >= 0 && (uint32_t)d1 < ppos);
    };
    auto remap = [&](uint32_t r) -> uint32_t {
      for (int k = 0; k < P.n_rm; ++k)
        if (r == P.rm_from[k]) return P.rm_to[k];
      return r;
    };
    auto map_ref = [&](uint32_t r) -> uint32_t { return (cpos(r >> 8) << 8) | (r & 255u); };
    // nodes
    {
      const int32_t* pnid = R.nid(G);
      const uint32_t* psig = R.sig(G);
      const uint32_t* paux = R.aux(G);
      int32_t* cnid = C.nid(G);
      uint32_t* csig = C.sig(G);
      uint32_t* caux = C.aux(G);
      uint32_t* cnin = C.nin(G);
      uint32_t* cinoff = C.inoff(G);
      const uint64_t* pkeys = R.keys(G);
      uint64_t* ckeys = C.keys(G);
      for (int i = threadIdx.x; i < n; i += BT) {
        if (i == d0 || i == d1) continue;
        uint32_t j = cpos((uint32_t)i);
        cnid[j] = pnid[i];
        ckeys[2 * j] = pkeys[2 * i];
        ckeys[2 * j + 1] = pkeys[2 * i + 1];
        csig[j] = i == P.mod ? P.mod_sig : psig[i];
        caux[j] = i == P.mod ? P.mod_aux : paux[i];
        cnin[j] = pnin[i];
        uint32_t off = pinoff[i];
        off -= (off > P.drop_inoff[0] ? (uint32_t)P.drop_refs[0] : 0u) + (off > P.drop_inoff[1] ? (uint32_t)P.drop_refs[1] : 0u);
        cinoff[j] = off;
      }
      if (threadIdx.x < 2) {
        const int k = threadIdx.x;
        if (k < P.n_new && P.live[k]) {
          uint32_t j = (uint32_t)n_keep + (k == 1 ? (uint32_t)P.live[0] : 0u);
          cnid[j] = R.nid(G)[n - 1] + 1 + k;
          csig[j] = P.new_sig[k];
          caux[j] = P.new_aux[k];
          cnin[j] = 1;
          cinoff[j] = (uint32_t)(n_refs - drop_ref_tot) + (j - (uint32_t)n_keep);
        }
      }
      if (threadIdx.x == 0) cinoff[n_child] = (uint32_t)n_refs_child;
    }
    __syncthreads();
    // refs of kept nodes (contiguous in the parent; dropped ranges removed)
    {
      const uint32_t* prefs = R.refs(G);
      uint32_t* crefs = C.refs(G);
      for (int r = threadIdx.x; r < n_refs; r += BT) {
        uint32_t ru = (uint32_t)r;
        bool in0 = P.drop[0] >= 0 && ru >= P.drop_inoff[0] && ru < P.drop_inoff[0] + (uint32_t)P.drop_refs[0];
        bool in1 = P.drop[1] >= 0 && ru >= P.drop_inoff[1] && ru < P.drop_inoff[1] + (uint32_t)P.drop_refs[1];
        if (in0 || in1) continue;
        uint32_t dst = ru - (ru > P.drop_inoff[0] ? (uint32_t)P.drop_refs[0] : 0u) - (ru > P.drop_inoff[1] ? (uint32_t)P.drop_refs[1] : 0u);
        uint32_t v = prefs[r];
        crefs[dst] = map_ref(remap(v));
      }
      if (threadIdx.x < 2) {
        const int k = threadIdx.x;
        if (k < P.n_new && P.live[k]) {
          uint32_t j = (uint32_t)n_keep + (k == 1 ? (uint32_t)P.live[0] : 0u);
          crefs[(uint32_t)(n_refs - drop_ref_tot) + (j - (uint32_t)n_keep)] = map_ref(P.new_ref[k]);
        }
      }
      const uint32_t* pouts = R.outs(G);
      uint32_t* couts = C.outs(G);
      for (int o = threadIdx.x; o < n_out; o += BT) couts[o] = map_ref(remap(pouts[o]));
    }
    // topological order: parent order with dropped slots removed and new nodes inserted
    {
      const uint32_t* ptopo = R.topo(G);
      uint32_t* ctopo = C.topo(G);
      // emission count of the <= 3 special slots
      int sp_slot[3], sp_emit[3];
      for (int k = 0; k < 3; ++k) {
        sp_slot[k] = P.slot_of[k];
        sp_emit[k] = 1;
      }
      // drops emit nothing unless they are the insertion point
      for (int k = 0; k < 2; ++k)
        if (sp_slot[k] >= 0) sp_emit[k] = 0;
      if (P.topo_mode == 1) sp_emit[2] = 1 + P.n_live;
      if (P.topo_mode == 2) sp_emit[2] = P.n_live;
      // a drop that is also the insertion slot must be counted once
      for (int k = 0; k < 2; ++k)
        if (sp_slot[k] >= 0 && sp_slot[k] == sp_slot[2]) sp_slot[k] = -1;
      for (int s = threadIdx.x; s < n; s += BT) {
        int shift = 0;
        bool special = false;
        for (int k = 0; k < 3; ++k) {
          if (sp_slot[k] < 0) continue;
          if (sp_slot[k] < s) shift += sp_emit[k] - 1;
          if (sp_slot[k] == s) special = true;
        }
        uint32_t at = (uint32_t)(s + shift);
        uint32_t v = ptopo[s];
        if (!special) {
          ctopo[at] = cpos(v);
        } else if (s == sp_slot[2]) {
          int e = 0;
          if (P.topo_mode == 1) ctopo[at + e++] = cpos(v);
          for (int k = 0; k < P.n_new; ++k)
            if (P.live[k]) ctopo[at + e++] = (uint32_t)n_keep + (k == 1 ? (uint32_t)P.live[0] : 0u);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ef_rec_header& H = C.h();
      H.n = n_child;
      H.n_refs = n_refs_child;
      H.n_out = n_out;
      H.n_compute = R.h().n_compute - (n - n_keep) + P.n_live;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// dedup: first occurrence in the step, then membership in the visited set
// ------------------------------------------------------------------------------------------

struct DedupArgs {
  ef_cand_result* res;
  const uint32_t* total;
  unsigned long long* step_key;
  uint32_t* step_seq;
  uint32_t step_mask;
  unsigned long long* vis_key;
  uint32_t vis_mask;
  unsigned long long* vis_count;
  int insert_visited;
  int node_cap;
  uint32_t* plist;    // survivors to price (appended in k_dedup_resolve), may be null
  uint32_t* plist_n;
  uint32_t* err;      // bit 8: visited set full
  int per_parent;     // also mark EF_F_PFIRST (second table at step_key/step_seq + step_mask + 1)
};

// step table: first occurrence of a key in candidate order (atomicMin on the index)
__device__ __forceinline__ void step_claim(unsigned long long* keys, uint32_t* seq, uint32_t mask,
                                           unsigned long long key, uint64_t h, uint32_t c) {
  uint32_t s = (uint32_t)mix64(h) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    unsigned long long prev = atomicCAS(&keys[s], 0ULL, key);
    if (prev == 0ULL || prev == key) {
      atomicMin(&seq[s], c);
      return;
    }
  }
}

__device__ __forceinline__ uint32_t step_first(const unsigned long long* keys, const uint32_t* seq, uint32_t mask,
                                               unsigned long long key, uint64_t h) {
  uint32_t s = (uint32_t)mix64(h) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    const unsigned long long k = keys[s];
    if (k == key) return seq[s];
    if (k == 0ULL) break;
  }
  return 0xffffffffu;
}

// Per-parent key of a candidate hash: a bijection of the hash for each parent (xor with a
// parent-dependent odd multiple), so the first occurrence of a hash within its own parent
// (rules.py:79-88 neighbors) is exact; distinct (hash, parent) pairs share a key only if two graph
// hashes differ by exactly that xor, as unlikely as the 64-bit hash collisions the reference's
// visited set already accepts.
__device__ __forceinline__ uint64_t parent_key(uint64_t h, uint32_t parent) {
  return h ^ ((uint64_t)(parent + 1) * 0x9E3779B97F4A7C15ULL);
}

__global__ void k_dedup_claim(DedupArgs A) {
  const uint32_t total = A.total[0];
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    if (A.res[c].flags & EF_F_INCOMPLETE) continue;
    unsigned long long h = A.res[c].hash;
    unsigned long long key = h ? h : 0x8000000000000000ULL;
    step_claim(A.step_key, A.step_seq, A.step_mask, key, h, c);
    if (A.per_parent) {
      const uint64_t hp = parent_key(h, A.res[c].parent);
      step_claim(A.step_key + A.step_mask + 1, A.step_seq + A.step_mask + 1, A.step_mask,
                 hp ? hp : 0x8000000000000000ULL, hp, c);
    }
  }
}

// Open-addressing visited set of 64-bit hashes (0 is stored as 1 << 63).  The host keeps it at
// most half full (vis_reserve in ef_api.cu grows it by rehashing), so probe runs are short; every
// probe loop is still bounded by the table size and reports a full table instead of spinning.
__device__ __forceinline__ bool vis_contains(const unsigned long long* keys, uint32_t mask, unsigned long long key,
                                             uint64_t h) {
  uint32_t s = (uint32_t)mix64(h) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    unsigned long long k = keys[s];
    if (k == key) return true;
    if (k == 0ULL) return false;
  }
  return false;
}

// insert; false when the table is full (the caller raises an error flag)
__device__ __forceinline__ bool vis_insert(unsigned long long* keys, uint32_t mask, unsigned long long* count,
                                           unsigned long long key, uint64_t h) {
  uint32_t s = (uint32_t)mix64(h) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    const unsigned long long prev = atomicCAS(&keys[s], 0ULL, key);
    if (prev == 0ULL) {
      atomicAdd(count, 1ULL);
      return true;
    }
    if (prev == key) return true;
  }
  return false;
}

__global__ void k_dedup_resolve(DedupArgs A) {
  const uint32_t total = A.total[0];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t span = (total + blockDim.x - 1) / blockDim.x * blockDim.x;  // whole warps iterate together
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < span; c += gridDim.x * blockDim.x) {
    bool survivor = false;
    if (c < total) {
      ef_cand_result& r = A.res[c];
      if (!(r.flags & EF_F_INCOMPLETE)) {
        unsigned long long h = r.hash;
        unsigned long long key = h ? h : 0x8000000000000000ULL;
        uint32_t f = r.flags;
        if (step_first(A.step_key, A.step_seq, A.step_mask, key, h) == c) f |= EF_F_FIRST;
        if (A.per_parent) {
          const uint64_t hp = parent_key(h, r.parent);
          if (step_first(A.step_key + A.step_mask + 1, A.step_seq + A.step_mask + 1, A.step_mask,
                         hp ? hp : 0x8000000000000000ULL, hp) == c)
            f |= EF_F_PFIRST;
        }
        bool seen = vis_contains(A.vis_key, A.vis_mask, key, h);
        if (seen) f |= EF_F_VISITED;
        if (r.n_compute > A.node_cap) f |= EF_F_CAPPED;
        r.flags = f;
        // priced: the first occurrence in the step, or (per_parent) in its parent
        const uint32_t first = A.per_parent ? EF_F_PFIRST : EF_F_FIRST;
        survivor = (f & (first | EF_F_VISITED | EF_F_CAPPED)) == first;
      }
    }
    if (A.plist) {  // warp-aggregated append keeps neighbouring candidates (same parent) together
      const unsigned m = __ballot_sync(__activemask(), survivor);
      if (m) {
        uint32_t base = 0;
        const int leader = __ffs(m) - 1;
        if ((int)lane == leader) base = atomicAdd(A.plist_n, (uint32_t)__popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (survivor) A.plist[base + __popc(m & ((1u << lane) - 1u))] = c;
      }
    }
  }
}

__global__ void k_visited_insert(DedupArgs A) {
  const uint32_t total = A.total[0];
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    const ef_cand_result& r = A.res[c];
    if ((r.flags & (EF_F_INCOMPLETE | EF_F_FIRST | EF_F_VISITED)) != EF_F_FIRST) continue;
    unsigned long long h = r.hash;
    unsigned long long key = h ? h : 0x8000000000000000ULL;
    if (!vis_insert(A.vis_key, A.vis_mask, A.vis_count, key, h)) atomicOr(A.err, 8u);
  }
}

__global__ void k_visited_put(unsigned long long* keys, uint32_t mask, unsigned long long* count, const uint64_t* hs,
                              uint32_t n, uint32_t* err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t h = hs[i];
    unsigned long long key = h ? h : 0x8000000000000000ULL;
    if (!vis_insert(keys, mask, count, key, h)) atomicOr(err, 8u);
  }
}

// grow the visited set: every stored key of the old table into the (empty) new one
__global__ void k_visited_rehash(const unsigned long long* old_keys, uint64_t old_n, unsigned long long* keys,
                                 uint32_t mask, unsigned long long* count, uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < old_n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = old_keys[i];
    if (!key) continue;
    const uint64_t h = key == 0x8000000000000000ULL ? 0ULL : key;
    if (!vis_insert(keys, mask, count, key, h)) atomicOr(err, 8u);
  }
}

// ------------------------------------------------------------------------------------------
// the alpha-prune of a step (search.py:258-267): a segmented-free exclusive prefix-min of the
// priced candidates' costs in (parent, rule, site) order, seeded with the best cost before the
// step.  prev_i = min(best, cost_j for priced j < i); BEST: cost_i < prev_i, ENQUEUE: cost_i <
// alpha * prev_i.  Three passes: tile minima, a scan of the tile minima, the in-tile scan.
// The running minimum updates only on a strict '<', like the reference's `best` (ties keep the
// earlier value; NaN never enters), so the combine op is associative in candidate order.
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ double min_keep_first(double a, double b) { return b < a ? b : a; }

template <int BT>
__device__ __forceinline__ double block_min(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min_keep_first(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < BT / 32 ? sh[lane] : CUDART_INF;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min_keep_first(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}

// exclusive prefix-min within the block (order = thread index), identity +inf
template <int BT>
__device__ __forceinline__ double block_exclusive_min(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = min_keep_first(y, x);
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    double w = lane < BT / 32 ? sh[lane] : CUDART_INF;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = min_keep_first(y, w);
    }
    sh[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  double ex = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) ex = CUDART_INF;
  if (wid > 0) ex = min_keep_first(sh[wid - 1], ex);
  __syncthreads();
  return ex;
}

// the candidates the reference evaluates when it expands the step's parents in order: priced and
// first in the step (per-parent pricing also prices later duplicates of other parents)
__device__ __forceinline__ bool prune_eligible(uint32_t f) {
  return (f & (EF_F_PRICED | EF_F_FIRST)) == (EF_F_PRICED | EF_F_FIRST);
}

__device__ __forceinline__ double priced_cost(const ef_cand_result& r) {
  return prune_eligible(r.flags) ? r.cost : CUDART_INF;
}

template <int BT>
__global__ void __launch_bounds__(BT) k_prune_tiles(const ef_cand_result* res, uint32_t total, double* tile_min) {
  __shared__ double sh[32];
  const uint32_t c = blockIdx.x * BT + threadIdx.x;
  const double v = block_min<BT>(c < total ? priced_cost(res[c]) : CUDART_INF, sh);
  if (threadIdx.x == 0) tile_min[blockIdx.x] = v;
}

// one block: tile_min[t] <- min(best, tile_min[0..t-1]) (the running best entering tile t)
template <int BT>
__global__ void __launch_bounds__(BT) k_prune_scan(double* tile_min, uint32_t n_tiles, double best) {
  __shared__ double sh[32];
  double carry = best;
  for (uint32_t t0 = 0; t0 < n_tiles; t0 += BT) {
    const uint32_t t = t0 + threadIdx.x;
    const double v = t < n_tiles ? tile_min[t] : CUDART_INF;
    const double ex = block_exclusive_min<BT>(v, sh);
    const double tot = block_min<BT>(v, sh);
    if (t < n_tiles) tile_min[t] = min_keep_first(carry, ex);
    carry = min_keep_first(carry, tot);
  }
}

template <int BT>
__global__ void __launch_bounds__(BT) k_prune_flags(ef_cand_result* res, uint32_t total, const double* tile_prev,
                                                    double alpha) {
  __shared__ double sh[32];
  const uint32_t c = blockIdx.x * BT + threadIdx.x;
  const bool in = c < total;
  const double v = in ? priced_cost(res[c]) : CUDART_INF;
  const double prev = min_keep_first(tile_prev[blockIdx.x], block_exclusive_min<BT>(v, sh));
  if (in && prune_eligible(res[c].flags)) {
    uint32_t f = res[c].flags & ~(uint32_t)(EF_F_BEST | EF_F_ENQUEUE);
    if (v < prev) f |= EF_F_BEST;
    if (v < alpha * prev) f |= EF_F_ENQUEUE;
    res[c].flags = f;
  }
}

// ------------------------------------------------------------------------------------------
// k_price: the inner search of search.py:106-153 (or the default assignment, 196-202)
// ------------------------------------------------------------------------------------------

struct PriceArgs {
  Geo g;
  Tables T;
  ef_price_params pp;
  const uint32_t* total;
  uint32_t n;
  const unsigned long long* rec;  // or null: cand_base
  char* cand_base;
  ef_cand_result* res;
  int step_mode;  // 1: only first & !visited & !capped & complete candidates
};

// ------------------------------------------------------------------------------------------
// x ** y as CPython computes it (C pow of glibc, correctly rounded in all but vanishingly rare
// cases).  CUDA's pow is accurate to 2 ulp, so a product cost (cost.py:246-248) could differ in
// its last bit and flip a sweep's strict '<'.  Here log and exp run in double-double (~100 bits):
// log by one Newton step on the hardware log, exp by range reduction, a Taylor series and ten
// squarings; the result rounds to the double nearest the exact power except when that lies
// within ~2^-40 ulp of a rounding boundary.  fma is used explicitly (exact products); the
// library builds with --fmad=false, so no other operation is contracted.
// ------------------------------------------------------------------------------------------

struct DD {
  double hi, lo;
};

__device__ __forceinline__ DD dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}

__device__ __forceinline__ DD dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}

__device__ __forceinline__ DD dd_add(DD x, DD y) {
  DD s = dd_two_sum(x.hi, y.hi), t = dd_two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}

__device__ __forceinline__ DD dd_mul(DD x, DD y) {
  const double p = x.hi * y.hi;
  double e = __fma_rn(x.hi, y.hi, -p);
  e += x.hi * y.lo + x.lo * y.hi;
  return dd_quick(p, e);
}

__device__ __forceinline__ DD dd_mul_d(DD x, double y) {
  const double p = x.hi * y;
  double e = __fma_rn(x.hi, y, -p);
  e += x.lo * y;
  return dd_quick(p, e);
}

__device__ __forceinline__ DD dd_div_d(DD x, double y) {
  const double q1 = x.hi / y;
  DD r = dd_add(x, dd_mul_d({q1, 0.0}, -y));
  const double q2 = r.hi / y;
  return dd_quick(q1, q2);
}

// exp of a double-double argument (|a| < 700)
__device__ DD dd_exp(DD a) {
  const DD ln2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
  const double k = rint(a.hi / ln2.hi);
  DD r = dd_add(a, dd_mul_d(ln2, -k));
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  // 1 + r + r^2/2! + ... + r^9/9! by Horner with exact integer divisions (|r| < 3.4e-4)
  DD p = {1.0, 0.0};
  for (int n = 9; n >= 1; --n) p = dd_add({1.0, 0.0}, dd_div_d(dd_mul(p, r), (double)n));
  for (int i = 0; i < 10; ++i) p = dd_mul(p, p);
  return {ldexp(p.hi, (int)k), ldexp(p.lo, (int)k)};
}

// log of a positive finite double: y0 = log(x), then y0 - 1 + x * exp(-y0)
__device__ DD dd_log(double x) {
  const double y0 = log(x);
  DD u = dd_mul_d(dd_exp({-y0, 0.0}), x);
  u = dd_add(u, {-1.0, 0.0});
  return dd_add({y0, 0.0}, u);
}

__device__ double pow_py(double x, double y) {
  if (y == 0.0 || x == 1.0) return 1.0;
  if (!(x > 0.0) || !isfinite(x) || !isfinite(y)) return pow(x, y);
  const DD z = dd_mul_d(dd_log(x), y);
  if (!(fabs(z.hi) < 700.0)) return pow(x, y);  // over/underflow: the hardware result
  const DD r = dd_exp(z);
  return r.hi + r.lo;
}

// Division by a normalisation reference (cost.py:284-296: t / t_ref, e / e_ref, p / p_ref),
// correctly rounded like the reference's float `/`, without a full division per evaluation:
// with r = RN(1 / y) taken once per thread, q0 = RN(x r) is within 2 ulp of x / y, one FMA
// residual correction q1 = RN(q0 + r RN(x - q0 y)) brings it within one ulp (faithful), and by
// Markstein's theorem a second correction is the correctly rounded quotient.  Exact for normal
// operands and quotients: |x|, |y| in [2^-500, 2^500] (checked; else -- and for NaN / inf --
// the IEEE division).  The residuals x - q y are exact (FMA).  tests/test_gpu_division.py
// compares it with the division on 2^27 operand pairs per reference.
struct Recip {
  double t, e, p;  // RN(1 / ref), or 0: divide
};

__device__ __forceinline__ double rcp_or_zero(double y) {
  const double a = fabs(y);
  return (a >= 0x1p-500 && a <= 0x1p500) ? 1.0 / y : 0.0;
}

__device__ __forceinline__ Recip recip_of(const ef_price_params& f) {
  return Recip{rcp_or_zero(f.t_ref), rcp_or_zero(f.e_ref), rcp_or_zero(f.p_ref)};
}

__device__ __forceinline__ double div_pre(double x, double y, double r) {
  const double a = fabs(x);
  if (r != 0.0 && a >= 0x1p-500 && a <= 0x1p500) {
    const double q0 = __dmul_rn(x, r);
    const double q1 = __fma_rn(__fma_rn(-q0, y, x), r, q0);
    return __fma_rn(__fma_rn(-q1, y, x), r, q1);
  }
  if (r != 0.0 && x == 0.0) return __dmul_rn(x, r);  // a signed zero, as x / y
  return x / y;
}

// cost.py:234-254 in the reference's operation order.  The reference always computes
// t = time/t_ref and e = energy/e_ref first; for the time / energy / power kinds those
// quotients are unused, so they are only formed where the result depends on them.
__device__ __forceinline__ double from_totals(const ef_price_params& f, const Recip& rc, double time_ms, double energy) {
  switch (f.kind) {
    case EF_C_TIME: return time_ms;
    case EF_C_ENERGY: return energy;
    case EF_C_POWER: return time_ms != 0.0 ? energy / time_ms : time_ms * 0.0;
    case EF_C_LINEAR: {
      const double t = div_pre(time_ms, f.t_ref, rc.t), e = div_pre(energy, f.e_ref, rc.e);
      return f.w * e + (1.0 - f.w) * t;
    }
    case EF_C_PRODUCT: {
      const double t = div_pre(time_ms, f.t_ref, rc.t), e = div_pre(energy, f.e_ref, rc.e);
      return pow_py(e, f.w) * pow_py(t, 1.0 - f.w);
    }
    default: {
      const double t = div_pre(time_ms, f.t_ref, rc.t), e = div_pre(energy, f.e_ref, rc.e);
      const double p = div_pre(time_ms != 0.0 ? energy / time_ms : time_ms * 0.0, f.p_ref, rc.p);
      return f.ct * t + f.ce * e + f.cp * p;
    }
  }
}

// CPython 3.12 builtin sum() over floats: Neumaier-compensated, start value int 0
struct NeumaierSum {
  double f, c;
  bool any;
  __device__ void init() {
    f = 0.0;
    c = 0.0;
    any = false;
  }
  __device__ void add(double x) {
    if (!any) {
      f = 0.0 + x;
      any = true;
      return;
    }
    double t = f + x;
    if (fabs(f) >= fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  // naive: CPython <= 3.11 sum(), plain left to right (the uncompensated running sum f)
  __device__ double result(int naive) const {
    double r = f;
    if (!naive && c != 0.0 && isfinite(c)) r += c;
    return r;
  }
};

constexpr int kMaxRadius = 16;

// the inner search on one graph given as a view: n nodes in id order, sig(i), alg row
template <class View>
__device__ void price_graph(const PriceArgs& A, const View& V, uint8_t* alg, ef_cand_result& res) {
  const Tables& T = A.T;
  const ef_price_params& F = A.pp;
  const int n = V.n;
  // start: lowest applicable algorithm (row 0) per compute node; Neumaier start totals
  NeumaierSum st, se;
  st.init();
  se.init();
  int ncomp = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t s = V.sig(i);
    if (T.sig_desc[s].kind == EF_K_INPUT) continue;
    ++ncomp;
    if (T.row_n[s] == 0) {
      res.flags |= EF_F_MISSING;
      return;
    }
    alg[i] = 0;
    st.add(T.row_t[T.row_off[s]]);
    se.add(T.row_e[T.row_off[s]]);
  }
  double t_tot = ncomp ? st.result(F.naive_sum) : 0.0;
  double e_tot = ncomp ? se.result(F.naive_sum) : 0.0;
  const Recip rc = recip_of(F);
  double cost = from_totals(F, rc, t_tot, e_tot);
  long long evals = 0;
  int sweeps = 0;
  if (A.pp.use_inner && ncomp > 0) {
    const int radius = min(min(F.d, ncomp), kMaxRadius);
    bool changed = true;
    while (changed) {
      changed = false;
      ++sweeps;
      // k = 1: every node, every alternative (ascending), first improvement
      for (int i = 0; i < n; ++i) {
        const uint32_t s = V.sig(i);
        if (T.sig_desc[s].kind == EF_K_INPUT) continue;
        const uint32_t nr = T.row_n[s];
        if (nr < 2) continue;
        const uint32_t ro = T.row_off[s];
        const uint32_t start = alg[i];
        for (uint32_t q = 0; q < nr; ++q) {
          if (q == start) continue;
          const uint32_t cur = alg[i];
          double dt = 0.0, de = 0.0;
          dt += T.row_t[ro + q] - T.row_t[ro + cur];
          de += T.row_e[ro + q] - T.row_e[ro + cur];
          const double cand = from_totals(F, rc, t_tot + dt, e_tot + de);
          ++evals;
          if (cand < cost) {
            alg[i] = (uint8_t)q;
            t_tot += dt;
            e_tot += de;
            cost = cand;
            changed = true;
          }
        }
      }
      // k >= 2: itertools.combinations(nids, k) x itertools.product(*alternatives)
      for (int k = 2; k <= radius; ++k) {
        int pos[kMaxRadius];
        int filled = 0;
        for (int i = 0; i < n && filled < k; ++i)
          if (T.sig_desc[V.sig(i)].kind != EF_K_INPUT) pos[filled++] = i;
        while (true) {
          uint32_t nalt[kMaxRadius], start[kMaxRadius], idx[kMaxRadius], psg[kMaxRadius];
          bool skip = false;
          for (int j = 0; j < k; ++j) {
            psg[j] = V.sig(pos[j]);
            nalt[j] = T.row_n[psg[j]] - 1;
            start[j] = alg[pos[j]];
            idx[j] = 0;
            if (nalt[j] == 0) skip = true;
          }
          if (!skip) {
            while (true) {
              double dt = 0.0, de = 0.0;
              uint32_t choice[kMaxRadius];
              for (int j = 0; j < k; ++j) {
                const uint32_t ro = T.row_off[psg[j]];
                const uint32_t q = idx[j] < start[j] ? idx[j] : idx[j] + 1;
                choice[j] = q;
                const uint32_t cur = alg[pos[j]];
                dt += T.row_t[ro + q] - T.row_t[ro + cur];
                de += T.row_e[ro + q] - T.row_e[ro + cur];
              }
              const double cand = from_totals(F, rc, t_tot + dt, e_tot + de);
              ++evals;
              if (cand < cost) {
                for (int j = 0; j < k; ++j) alg[pos[j]] = (uint8_t)choice[j];
                t_tot += dt;
                e_tot += de;
                cost = cand;
                changed = true;
              }
              int j = k - 1;  // next product index: last position varies fastest
              while (j >= 0 && ++idx[j] == nalt[j]) idx[j--] = 0;
              if (j < 0) break;
            }
          }
          // next combination of compute positions (lexicographic)
          int j = k - 1;
          bool advanced = false;
          while (j >= 0) {
            int q = pos[j] + 1;
            while (q < n && T.sig_desc[V.sig(q)].kind == EF_K_INPUT) ++q;
            int room = 0;
            for (int x = q; x < n && room < k - j; ++x)
              if (T.sig_desc[V.sig(x)].kind != EF_K_INPUT) ++room;
            if (q < n && room >= k - j) {
              pos[j] = q;
              int f2 = j + 1;
              for (int x = q + 1; x < n && f2 < k; ++x)
                if (T.sig_desc[V.sig(x)].kind != EF_K_INPUT) pos[f2++] = x;
              advanced = true;
              break;
            }
            --j;
          }
          if (!advanced) break;
        }
      }
    }
  }
  // row index -> algorithm id
  for (int i = 0; i < n; ++i) {
    const uint32_t s = V.sig(i);
    if (T.sig_desc[s].kind == EF_K_INPUT) continue;
    alg[i] = (uint8_t)T.row_alg[T.row_off[s] + alg[i]];
  }
  res.cost = cost;
  res.time_ms = t_tot;
  res.energy = e_tot;
  res.evals = A.pp.use_inner ? evals : 1;
  res.sweeps = sweeps;
  res.flags |= EF_F_PRICED;
}

template <int KIND>
__device__ __forceinline__ double cost_of(const ef_price_params& f, const Recip& rc, double time_ms, double energy) {
  if (KIND == EF_C_TIME) return time_ms;
  if (KIND == EF_C_ENERGY) return energy;
  if (KIND == EF_C_LINEAR) {
    const double t = div_pre(time_ms, f.t_ref, rc.t), e = div_pre(energy, f.e_ref, rc.e);
    return f.w * e + (1.0 - f.w) * t;
  }
  return from_totals(f, rc, time_ms, energy);
}

// The d = 1 sweep (search.py:106-153 with radius 1) specialised on the cost kind: the same
// floating-point operations in the same order as price_graph / the reference.  Written
// warp-synchronously: every loop runs a warp-uniform trip count (the lanes of `mask` price
// different candidates whose node counts differ by a few), with no early exits, so the warp
// never splits into groups that would then run the whole sweep one after another.
//
// Two exact shortcuts.  (1) The cost kinds time, energy and linear(w in [0, 1], positive refs)
// are non-decreasing in both totals, and `cost == cost_of(t_tot, e_tot)` holds throughout, so
// a node none of whose rows is below row 0 in the kind's totals (kInfoTMin / kInfoEMin, set
// per signature at commit) can never take an alternative: adding a non-negative difference
// never lowers a total (round-to-nearest is monotone).  Such a node stays at row 0 and only
// counts its nr - 1 evaluations per sweep, so the sweeps skip it (the `skip` argument of the
// kind).  (2) The row is zero on entry (row 0 everywhere; the caller clears it), the first
// sweep reads no row entry and a sweep writes a node's entry only when it changes.  The row
// holds ROW indices, not algorithm ids; the ids are read from the signature's rows where a
// record is written (k_keep_alg).
// the sparse-sweep mask of a view (VirtView on a parent: k_price_nsk), else null; the sparse
// sweep itself is VirtView's (ef_step.cuh), never reached for other views
template <class View>
__device__ __forceinline__ const uint32_t* view_nsk(const View&) { return nullptr; }
template <class View, class F>
__device__ __forceinline__ void sparse_sweep(const View&, unsigned, bool, const uint32_t*, const Tables&, F&&, int& n_dense0) {
  n_dense0 = 0;
}

template <int KIND, class View, class Alg>
__device__ void price_d1(const PriceArgs& A, const View& V, Alg alg, ef_cand_result& res, unsigned mask,
                         uint32_t skip) {
  const Tables& T = A.T;
  const ef_price_params& F = A.pp;
  const int n = V.n;
  const int nmax = __reduce_max_sync(mask, (unsigned)n);
  NeumaierSum st, se;
  st.init();
  se.init();
  int ncomp = 0;
  long long skip_evals = 0;  // evaluations per sweep of the skipped nodes
  bool missing = false;
  constexpr int G = 8;  // nodes whose rows are requested together (independent loads)
  for (int i0 = 0; i0 < nmax; i0 += G) {
    uint2 inf[G];
    double rt[G], re[G];
#pragma unroll
    for (int k = 0; k < G; ++k) inf[k] = i0 + k < n ? V.info(i0 + k, T) : make_uint2(0u, kInfoInput);
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const bool row = !(inf[k].y & kInfoInput) && (inf[k].y & kInfoRows);
      rt[k] = row ? T.row_t[inf[k].x] : 0.0;
      re[k] = row ? T.row_e[inf[k].x] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (missing || (inf[k].y & kInfoInput)) continue;
      ++ncomp;
      const uint32_t nr = inf[k].y & kInfoRows;
      if (nr == 0) {
        missing = true;
      } else {
        st.add(rt[k]);
        se.add(re[k]);
        if (skip && (inf[k].y & skip) == skip) skip_evals += nr - 1;
      }
    }
  }
  double t_tot = ncomp ? st.result(F.naive_sum) : 0.0;
  double e_tot = ncomp ? se.result(F.naive_sum) : 0.0;
  const Recip rc = recip_of(F);
  double cost = cost_of<KIND>(F, rc, t_tot, e_tot);
  long long evals = 0;
  int sweeps = 0;
  bool running = !missing && ncomp > 0;
  while (__any_sync(mask, running)) {
    bool changed = false;
    if (running) {
      ++sweeps;
      evals += skip_evals;
    }
    const bool first = sweeps == 1;
    // node i with info word pair inf: the first-improvement pass over its rows
    auto sweep_node = [&](const int i, const uint2 in) {
        const uint32_t nr = in.y & kInfoRows;
        if (nr < 2u || (in.y & kInfoInput) || (skip && (in.y & skip) == skip)) return;
        const uint32_t ro = in.x;
        const uint32_t start = first ? 0u : (uint32_t)alg[i];
        uint32_t cur = start;
        double ct = T.row_t[ro + cur], ce = T.row_e[ro + cur];
        for (uint32_t q = 0; q < nr; ++q) {  // branch-free body
          const double qt = T.row_t[ro + q], qe = T.row_e[ro + q];
          double dt = 0.0, de = 0.0;
          dt += qt - ct;
          de += qe - ce;
          const double nt = t_tot + dt, ne = e_tot + de;
          const double cand = cost_of<KIND>(F, rc, nt, ne);
          const bool act = q != start;
          evals += act ? 1 : 0;
          const bool take = act && cand < cost;
          cur = take ? q : cur;
          ct = take ? qt : ct;
          ce = take ? qe : ce;
          t_tot = take ? nt : t_tot;
          e_tot = take ? ne : e_tot;
          cost = take ? cand : cost;
          changed = changed || take;
        }
        if (cur != start) alg[i] = (uint8_t)cur;
    };
    const uint32_t* nsk = view_nsk(V);
    if (nsk) {  // sparse: only the parent positions whose node can move (k_price_nsk), in order
      int n_dense0;
      sparse_sweep(V, mask, running, nsk, T, sweep_node, n_dense0);
      for (int i0 = n_dense0; i0 < nmax; ++i0)  // then the new nodes (ids n_keep, n_keep + 1)
        if (running && i0 < n) sweep_node(i0, V.info(i0, T));
    } else {
      for (int i0 = 0; i0 < nmax; i0 += G) {
        uint2 inf[G];  // the rows of G nodes requested together
#pragma unroll
        for (int k = 0; k < G; ++k) inf[k] = running && i0 + k < n ? V.info(i0 + k, T) : make_uint2(0u, kInfoInput);
#pragma unroll
        for (int k = 0; k < G; ++k) sweep_node(i0 + k, inf[k]);
      }
    }
    running = running && changed;
  }
  if (missing) {
    res.flags |= EF_F_MISSING;
    return;
  }
  res.cost = cost;
  res.time_ms = t_tot;
  res.energy = e_tot;
  res.evals = evals;
  res.sweeps = sweeps;
  res.flags |= EF_F_PRICED;
}

// price_d1 with L lanes per candidate (lanes sl = 0..L-1 of a group starting at lane gbase).
// Every floating-point value of a candidate is computed by one lane with the operands the
// sequential sweep has at that point, so the results are price_d1's bit for bit:
//  * start totals: each window's L rows are loaded by the L lanes and summed in node order by
//    every lane of the group (the Neumaier sum is order-dependent: it stays sequential);
//  * sweeps: the L nodes of a window are evaluated at once, each against the current totals.
//    Nodes before the window's first node that takes an alternative saw the totals the
//    sequential sweep would have (no earlier node changed them), so they and that node are
//    committed -- its totals, cost and row entry become the group's -- and the window restarts
//    after it; the later nodes' evaluations are discarded.  Windows without a take commit all
//    L nodes.  Evaluation counts are per committed node (nr - 1 each, as in price_d1).
// Converged sweeps (usually every sweep after the first) run L nodes per step of the chain.
template <int KIND, int L, class View, class Alg>
__device__ void price_d1_lanes(const PriceArgs& A, const View& V, Alg alg, ef_cand_result* res, bool valid,
                               uint32_t sl, uint32_t gbase, uint32_t skip) {
  const Tables& T = A.T;
  const ef_price_params& F = A.pp;
  const Recip rc = recip_of(F);
  const unsigned full = 0xffffffffu;
  const int n = valid ? V.n : 0;
  const int nmax = __reduce_max_sync(full, (unsigned)n);
  NeumaierSum st, se;
  st.init();
  se.init();
  int ncomp = 0;
  long long skip_evals = 0;
  bool missing = false;
  for (int i0 = 0; i0 < nmax; i0 += L) {
    const int i = i0 + (int)sl;
    const uint2 inf = i < n ? V.info(i, T) : make_uint2(0u, kInfoInput);
    const bool row = !(inf.y & kInfoInput) && (inf.y & kInfoRows);
    const double rt = row ? T.row_t[inf.x] : 0.0, re = row ? T.row_e[inf.x] : 0.0;
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const uint32_t y = __shfl_sync(full, inf.y, gbase + k);
      const double xt = __shfl_sync(full, rt, gbase + k), xe = __shfl_sync(full, re, gbase + k);
      if (i0 + k >= n || missing || (y & kInfoInput)) continue;
      ++ncomp;
      const uint32_t nr = y & kInfoRows;
      if (nr == 0) {
        missing = true;
      } else {
        st.add(xt);
        se.add(xe);
        if (skip && (y & skip) == skip) skip_evals += nr - 1;
      }
    }
  }
  double t_tot = ncomp ? st.result(F.naive_sum) : 0.0;
  double e_tot = ncomp ? se.result(F.naive_sum) : 0.0;
  double cost = cost_of<KIND>(F, rc, t_tot, e_tot);
  long long evals = 0;
  int sweeps = 0;
  bool running = !missing && ncomp > 0;
  while (__any_sync(full, running)) {
    bool changed = false;
    if (running) {
      ++sweeps;
      evals += skip_evals;
    }
    const bool first = sweeps == 1;
    int i0 = 0;
    while (__any_sync(full, running && i0 < n)) {
      const bool act_w = running && i0 < n;  // group-uniform
      const int i = i0 + (int)sl;
      bool took = false;
      long long my_ev = 0;
      double lt = t_tot, le = e_tot, lc = cost;
      uint32_t cur = 0;
      if (act_w && i < n) {
        const uint2 inf = V.info(i, T);
        const uint32_t nr = inf.y & kInfoRows;
        if (!(nr < 2u || (inf.y & kInfoInput) || (skip && (inf.y & skip) == skip))) {
          const uint32_t ro = inf.x;
          const uint32_t start = first ? 0u : (uint32_t)alg[i];
          cur = start;
          double ct = T.row_t[ro + cur], ce = T.row_e[ro + cur];
          for (uint32_t q = 0; q < nr; ++q) {
            const double qt = T.row_t[ro + q], qe = T.row_e[ro + q];
            double dt = 0.0, de = 0.0;
            dt += qt - ct;
            de += qe - ce;
            const double nt = lt + dt, ne = le + de;
            const double cand = cost_of<KIND>(F, rc, nt, ne);
            const bool act = q != start;
            my_ev += act ? 1 : 0;
            const bool take = act && cand < lc;
            cur = take ? q : cur;
            ct = take ? qt : ct;
            ce = take ? qe : ce;
            lt = take ? nt : lt;
            le = take ? ne : le;
            lc = take ? cand : lc;
            took = took || take;
          }
        }
      }
      const unsigned tb = (__ballot_sync(full, took) >> gbase) & ((1u << L) - 1u);
      const int f = tb ? __ffs(tb) - 1 : L;  // the window's first node that took
      long long ev_sum = 0;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const long long x = __shfl_sync(full, my_ev, gbase + k);
        if (k <= f) ev_sum += x;
      }
      const int srcl = (int)gbase + (f < L ? f : 0);
      const double nt = __shfl_sync(full, lt, srcl), ne = __shfl_sync(full, le, srcl), nc = __shfl_sync(full, lc, srcl);
      if (act_w) {
        evals += ev_sum;
        if (f < L) {
          if ((int)sl == f) alg[i] = (uint8_t)cur;
          t_tot = nt;
          e_tot = ne;
          cost = nc;
          changed = true;
          i0 += f + 1;
        } else {
          i0 += L;
        }
      }
      __syncwarp();  // the committed row entry is visible to the lanes that read it next
    }
    running = running && changed;
  }
  if (!valid || sl != 0) return;
  if (missing) {
    res->flags |= EF_F_MISSING;
    return;
  }
  res->cost = cost;
  res->time_ms = t_tot;
  res->energy = e_tot;
  res->evals = evals;
  res->sweeps = sweeps;
  res->flags |= EF_F_PRICED;
}

// the per-signature bits of a cost kind's exact skip (price_d1), given the price parameters
template <int KIND>
__device__ __forceinline__ uint32_t d1_skip_bits(const ef_price_params& f) {
  if (KIND == EF_C_TIME) return kInfoTMin;
  if (KIND == EF_C_ENERGY) return kInfoEMin;
  if (KIND == EF_C_LINEAR && f.w >= 0.0 && f.w <= 1.0 && f.t_ref > 0.0 && f.e_ref > 0.0) return kInfoTMin | kInfoEMin;
  return 0u;
}

// a candidate's algorithm row: global bytes, or a shared-memory column (stride = block size)
struct AlgRow {
  uint8_t* p;
  int stride;
  __device__ __forceinline__ uint8_t& operator[](int i) const { return p[i * stride]; }
};

struct RecView {
  const uint32_t* s;
  int n;
  __device__ __forceinline__ uint32_t sig(int i) const { return s[i]; }
  __device__ __forceinline__ uint2 info(int i, const Tables& T) const { return T.sig_info[s[i]]; }
};

__global__ void k_price(PriceArgs A) {
  const Geo& G = A.g;
  const uint32_t total = A.total ? A.total[0] : A.n;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    ef_cand_result& res = A.res[c];
    if (A.step_mode) {
      if ((res.flags & (EF_F_INCOMPLETE | EF_F_FIRST | EF_F_VISITED | EF_F_CAPPED)) != EF_F_FIRST) continue;
    }
    Rec R{A.rec ? reinterpret_cast<char*>(A.rec[c]) : A.cand_base + (uint64_t)c * G.bytes};
    RecView V{R.sig(G), R.h().n};
    price_graph(A, V, R.alg(G), res);
  }
}

// ------------------------------------------------------------------------------------------
// record copy (keep candidates) and weight-set kernels
// ------------------------------------------------------------------------------------------

__global__ void k_copy_records(const unsigned long long* src, const unsigned long long* dst, uint32_t n, uint32_t bytes) {
  const uint32_t words = bytes / 16;
  for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(src[r]);
    uint4* d = reinterpret_cast<uint4*>(dst[r]);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) d[i] = s[i];
  }
}

// derived tensors (rules.py:231-232, 272-276, 326-327); every op one IEEE rounding, no FMA
struct DeriveJob {
  int32_t op;
  const double* wa;  // left / source conv weight
  const double* ba;  // its bias (null: zeros)
  const double* wb;  // MERGE: right weight; FOLD: bn scale
  const double* bb;  // MERGE: right bias (null: zeros); FOLD: bn shift
  uint64_t oc_a, oc_b, inner;  // out channels (a, b) and elements per out channel
  int32_t s0;
  double* w_out;
  double* b_out;
  uint64_t w_n, b_n;
};

__global__ void k_derive(const DeriveJob* jobs, uint32_t n) {
  for (uint32_t j = 0; j < n; ++j) {
    const DeriveJob J = jobs[j];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (uint64_t i = t0; i < J.w_n; i += stride) {
      double v;
      if (J.op == EF_D_MERGE) {
        const uint64_t na = J.oc_a * J.inner;
        v = i < na ? J.wa[i] : J.wb[i - na];
      } else if (J.op == EF_D_SLICE_LO) {
        v = J.wa[i];
      } else if (J.op == EF_D_SLICE_HI) {
        v = J.wa[(uint64_t)J.s0 * J.inner + i];
      } else {  // FOLD: weight * scale[:, None, None, None]
        v = __dmul_rn(J.wa[i], J.wb[i / J.inner]);
      }
      J.w_out[i] = v;
    }
    for (uint64_t i = t0; i < J.b_n; i += stride) {
      double v;
      if (J.op == EF_D_MERGE) {
        v = i < J.oc_a ? (J.ba ? J.ba[i] : 0.0) : (J.bb ? J.bb[i - J.oc_a] : 0.0);
      } else if (J.op == EF_D_SLICE_LO) {
        v = J.ba ? J.ba[i] : 0.0;
      } else if (J.op == EF_D_SLICE_HI) {
        v = J.ba ? J.ba[(uint64_t)J.s0 + i] : 0.0;
      } else {  // FOLD: bias * scale + shift
        v = __dadd_rn(__dmul_rn(J.ba ? J.ba[i] : 0.0, J.wb[i]), J.bb[i]);
      }
      J.b_out[i] = v;
    }
  }
}

}  // namespace ef
