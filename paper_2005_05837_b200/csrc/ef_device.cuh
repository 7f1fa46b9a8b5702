// Device-side data model shared by the kernels (ef_kernels.cuh) and the C ABI (ef_api.cu).
#pragma once
#include <stdint.h>

#include "../../include/ef200.h"
#include "ef_blake2b.cuh"

namespace ef {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kOutMark = 1u << 24;  // added to a use count when the edge is a graph output
constexpr uint32_t kEmptyWset = 0;       // weight-set id of "no weights"
// Tables::sig_info[s].y: the signature's row count and flags
constexpr uint32_t kInfoRows = 0xffffffu;    // number of cost rows
constexpr uint32_t kInfoInput = 1u << 31;    // input node (no rows, not priced)
constexpr uint32_t kInfoEMin = 1u << 30;     // no row has less energy than row 0
constexpr uint32_t kInfoTMin = 1u << 29;     // no row has less time than row 0

// record geometry (byte offsets inside one slot); mirrors ef_geometry
struct Geo {
  uint32_t cap_nodes, cap_refs, cap_outs, bytes;
  uint32_t o_nid, o_sig, o_aux, o_nin, o_inoff, o_topo, o_refs, o_outs, o_keys, o_alg, o_sperm, o_skeys, o_srank;
};

struct Rec {
  char* p;
  __host__ __device__ ef_rec_header& h() const { return *reinterpret_cast<ef_rec_header*>(p); }
  __host__ __device__ int32_t* nid(const Geo& g) const { return reinterpret_cast<int32_t*>(p + g.o_nid); }
  __host__ __device__ uint32_t* sig(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_sig); }
  __host__ __device__ uint32_t* aux(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_aux); }
  __host__ __device__ uint32_t* nin(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_nin); }
  __host__ __device__ uint32_t* inoff(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_inoff); }
  __host__ __device__ uint32_t* topo(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_topo); }
  __host__ __device__ uint32_t* refs(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_refs); }
  __host__ __device__ uint32_t* outs(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_outs); }
  __host__ __device__ uint64_t* keys(const Geo& g) const { return reinterpret_cast<uint64_t*>(p + g.o_keys); }
  __host__ __device__ uint8_t* alg(const Geo& g) const { return reinterpret_cast<uint8_t*>(p + g.o_alg); }
  __host__ __device__ uint32_t* sperm(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_sperm); }
  __host__ __device__ uint64_t* skeys(const Geo& g) const { return reinterpret_cast<uint64_t*>(p + g.o_skeys); }
  __host__ __device__ uint32_t* srank(const Geo& g) const { return reinterpret_cast<uint32_t*>(p + g.o_srank); }
};

// read-only tables, passed by value to kernels
struct Tables {
  const ef_sig_desc* sig_desc;
  const uint2* sig_info;  // per signature: {row_off, row_n | flags} (kInfo*; pricing)
  const uint32_t* sig_text_off;
  const uint32_t* sig_text_len;
  const uint8_t* sig_text;
  const uint32_t* row_off;
  const uint32_t* row_n;
  const int32_t* row_alg;
  const double* row_t;
  const double* row_e;
  const unsigned long long* sig_ht_key;
  const uint32_t* sig_ht_val;
  uint32_t sig_ht_mask;
  const uint64_t* ws_digest;  // 2 words per weight set (raw little-endian digest words)
  const int32_t* dv_tuple;    // 4 ints per weight set: op, a, b, s0 (op 0 = original)
  const unsigned long long* dv_ht_key;
  const uint32_t* dv_ht_val;
  uint32_t dv_ht_mask;
  const uint32_t* name_off;
  const uint32_t* name_len;
  const uint8_t* names;
  const uint8_t* input_text;
  uint32_t input_text_len;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// table key of a signature descriptor (never 0: 0 marks an empty slot)
__host__ __device__ inline uint64_t desc_key(const ef_sig_desc& d) {
  const int32_t* w = reinterpret_cast<const int32_t*>(&d);
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < (int)(sizeof(ef_sig_desc) / 4); ++i) h = mix64(h ^ (uint64_t)(uint32_t)w[i] ^ ((uint64_t)i << 40));
  return h | 1ULL;
}

__host__ __device__ inline uint64_t derive_key(int32_t op, uint32_t a, uint32_t b, int32_t s0) {
  uint64_t h = mix64(((uint64_t)(uint32_t)op << 32) ^ a ^ 0x51ed27ULL);
  h = mix64(h ^ ((uint64_t)b << 20) ^ (uint64_t)(uint32_t)s0);
  return h | 1ULL;
}

__host__ __device__ inline bool desc_eq(const ef_sig_desc& a, const ef_sig_desc& b) {
  const int32_t* x = reinterpret_cast<const int32_t*>(&a);
  const int32_t* y = reinterpret_cast<const int32_t*>(&b);
  for (int i = 0; i < (int)(sizeof(ef_sig_desc) / 4); ++i)
    if (x[i] != y[i]) return false;
  return true;
}

}  // namespace ef
