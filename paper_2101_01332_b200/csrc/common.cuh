// Shared types and helpers for libtsat (B200 / sm_100a).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;
typedef uint8_t u8;

#define TSAT_NONE 0xFFFFFFFFu

// node flag bits
#define NF_ALIVE 1u
#define NF_FILT 2u
#define NF_LOCK 0x80u  // transient: analysis merge lock of a root (rebuild)

// status / error codes shared with the Python boundary (_lib.py)
#include "../../include/tsat.h"

// device-side error record (first error wins)
struct DevError {
  int code;      // TsatStatus
  int detail;    // sub-code
  i64 a, b;      // context (node id, combo position, ...)
};

// TSAT_DEBUG_SYNCS: count memcpy / memset calls per source line (host debug)
extern bool g_dbg_sites;
void tsat_count_site(const char* what, const char* file, int line);
#define CUDA_OK(x)                                                                  \
  do {                                                                              \
    if (g_dbg_sites) tsat_count_site(#x, __FILE__, __LINE__);                       \
    cudaError_t _e = (x);                                                           \
    if (_e != cudaSuccess) {                                                        \
      throw TsatException(TSAT_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(_e) + \
                                            " at " __FILE__ ":" + std::to_string(__LINE__)); \
    }                                                                               \
  } while (0)

__device__ __forceinline__ void dev_set_error(DevError* e, int code, int detail, i64 a, i64 b) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->detail = detail;
    e->a = a;
    e->b = b;
  }
}

__host__ __device__ __forceinline__ u32 hash32(u32 x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ u64 hash_mix(u64 h, u64 v) {
  h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  return h;
}

// Union-find root lookup with path halving.  Halving only rewrites parent
// pointers of non-roots to an ancestor, so it is safe next to concurrent
// finds and next to the CAS root-linking in uf_union_min.
__device__ __forceinline__ u32 uf_find(u32* parent, u32 x) {
  while (true) {
    u32 p = parent[x];
    if (p == x) return x;
    u32 gp = parent[p];
    if (gp == p) return p;
    parent[x] = gp;
    x = gp;
  }
}

__device__ __forceinline__ u32 uf_find_ro(const u32* parent, u32 x) {
  u32 p;
  while ((p = parent[x]) != x) x = p;
  return x;
}

// lock-free min-root union; returns true when two roots were linked
__device__ __forceinline__ bool uf_union_min(u32* parent, u32 a, u32 b) {
  while (true) {
    a = uf_find_ro(parent, a);
    b = uf_find_ro(parent, b);
    if (a == b) return false;
    u32 lo = a < b ? a : b, hi = a < b ? b : a;
    if (atomicCAS(&parent[hi], hi, lo) == hi) return true;
  }
}
