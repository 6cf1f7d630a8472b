// Shared device helpers for libsfkv (sm_100a): the chained block hash, error plumbing, a
// three-phase device scan and growable scratch buffers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <string>
#include <utility>

#include "../../include/sfkv.h"

namespace sfkv {

constexpr int BT = SFKV_BLOCK_TOKENS;          // tokens per block
constexpr uint64_t KEY_EMPTY = 0ull;           // table key: never used
constexpr uint64_t KEY_TOMB = 1ull;            // table key: deleted
constexpr int64_t NO_OWNER = INT64_MAX;

// ---- the chained block hash (include/sfkv.h; identical to the oracle's restatement) ----------
__host__ __device__ constexpr uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

// NH keys (UMAC-style pair hash): key j of set s is a 32-bit slice of mix64(s * 16 + j + 1).
__host__ __device__ constexpr uint32_t nh_key(int set, int j) {
  return (uint32_t)(mix64((uint64_t)(set * 16 + j + 1)) >> (set ? 32 : 0));
}

// digest of block k with n valid tokens; t[i] for i >= n must already be zero.
//   acc_s = sum_{i<8} (t[2i] + K_s[2i]) * (t[2i+1] + K_s[2i+1])   (32-bit adds, 64-bit products)
//   digest = mix64(acc_0 ^ rotl(acc_1, 32) ^ (k * H + n))
// Two NH passes (each 2^-32-almost-universal on 32-bit words) under one 64-bit finaliser: a
// 64-bit non-cryptographic key at ~50 integer instructions per block. M never depends on it
// (it is token-compared); the dedup table verifies the block's tokens on every key hit.
__host__ __device__ __forceinline__ uint64_t block_digest_words(uint64_t k, uint32_t n,
                                                                const uint32_t* t) {
  uint64_t a0 = 0, a1 = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a0 += (uint64_t)(uint32_t)(t[2 * i] + nh_key(0, 2 * i)) *
          (uint64_t)(uint32_t)(t[2 * i + 1] + nh_key(0, 2 * i + 1));
    a1 += (uint64_t)(uint32_t)(t[2 * i] + nh_key(1, 2 * i)) *
          (uint64_t)(uint32_t)(t[2 * i + 1] + nh_key(1, 2 * i + 1));
  }
  return mix64(a0 ^ ((a1 << 32) | (a1 >> 32)) ^ (k * 0xD6E8FEB86659FD93ull + n));
}

// ---- L2 residency hints --------------------------------------------------------------------
// Streamed data (read or written once per batch) is marked evict_first so it does not push out
// what a later pass of the same batch re-reads (evict_last): chain sums, tables, records.
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_u64_hint(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_u32_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
// 16-B read-only load, no L1 allocation, with an L2 policy
__device__ __forceinline__ uint4 ld_nc16_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// The chain sum is taken mod 2^62 so a look-back status word can carry it next to a 2-bit flag.
constexpr uint64_t CHAIN_MASK = (1ull << 62) - 1;

__host__ __device__ __forceinline__ uint64_t chain_finalize(uint64_t s) {
  uint64_t c = mix64((s & CHAIN_MASK) ^ 0x5851F42D4C957F2Dull);
  return c < 2 ? c + 2 : c;
}

// ---- errors --------------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SFKV_CUDA(call)                                         \
  do {                                                          \
    cudaError_t e__ = (call);                                   \
    if (e__ != cudaSuccess) return ::sfkv::cuda_fail(e__, #call); \
  } while (0)

#define SFKV_LAUNCH_CHECK(what)                                 \
  do {                                                          \
    cudaError_t e__ = cudaGetLastError();                       \
    if (e__ != cudaSuccess) return ::sfkv::cuda_fail(e__, what); \
  } while (0)

// ---- growable device scratch --------------------------------------------------------------
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return 0;
    if (ptr) cudaFree(ptr);
    size_t nb = bytes ? bytes : 1 << 16;
    while (nb < need) nb *= 2;
    cudaError_t e = cudaMalloc(&ptr, nb);
    if (e != cudaSuccess) {
      ptr = nullptr;
      bytes = 0;
      return cuda_fail(e, "scratch cudaMalloc");
    }
    bytes = nb;
    return 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

// Carves typed, 256-B aligned sub-buffers out of one scratch allocation.
struct Carver {
  size_t off = 0;
  template <class T>
  size_t take(size_t n) {
    size_t o = (off + 255) & ~size_t(255);
    off = o + n * sizeof(T);
    return o;
  }
};

// ---- programmatic dependent launch -------------------------------------------------------
// Kernels of one pipeline on a stream are launched with programmatic stream serialization: the
// next kernel's CTAs may be scheduled while the previous grid drains; every kernel waits at its
// top (griddepcontrol.wait) until its predecessor has completed and its writes are visible, so
// the data dependencies are exactly those of plain stream order. Launch latency is hidden.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- device-wide exclusive scan (three phases, cub::BlockScan inside each CTA) --------------
// out[i] = sum_{j<i} f(j) for i in [0, n], out[n] = total. f is a device functor (int64 result).
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class F>
__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(F f, int64_t n, int64_t* tile_sums) {
  using BS = cub::BlockReduce<int64_t, SCAN_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  pdl_enter();
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < n) s += f(idx);
  }
  s = BS(tmp).Sum(s);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) scan_tiles_kernel(int64_t* tile_sums, int64_t ntiles);

template <class F>
__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(F f, int64_t n, const int64_t* tile_off,
                                                          int64_t* out) {
  using BS = cub::BlockScan<int64_t, SCAN_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  pdl_enter();
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t v[SCAN_ITEMS];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;  // blocked arrangement
    v[i] = idx < n ? f(idx) : 0;
  }
  int64_t agg;
  BS(tmp).ExclusiveSum(v, v, agg);
  int64_t t0 = tile_off[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    if (idx < n) out[idx] = t0 + v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = t0 + agg;
}

// Small scans (<= 4 tiles): one CTA walks the tiles in order with a running carry — one launch
// instead of three (the free-bitmap scan of a commit, the tracker's per-workflow counts). At 8
// tiles the serial walk already cost more than the three-kernel scan.
#ifndef SFKV_SCAN_SINGLE
#define SFKV_SCAN_SINGLE 4
#endif
constexpr int64_t SCAN_SINGLE_MAX_TILES = SFKV_SCAN_SINGLE;
template <class F>
__global__ void __launch_bounds__(SCAN_THREADS) scan_single_kernel(F f, int64_t n, int64_t* out) {
  using BS = cub::BlockScan<int64_t, SCAN_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  pdl_enter();
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += SCAN_TILE) {
    int64_t v[SCAN_ITEMS];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
      const int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;  // blocked arrangement
      v[i] = idx < n ? f(idx) : 0;
    }
    int64_t agg;
    BS(tmp).ExclusiveSum(v, v, agg);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
      const int64_t idx = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
      if (idx < n) out[idx] = carry + v[i];
    }
    carry += agg;
    __syncthreads();  // tmp reused
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// Scratch needed by exclusive_scan for n items (tile sums).
inline size_t scan_scratch_elems(int64_t n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }

// The reduce phase reads items in a strided arrangement and the apply phase in a blocked one;
// both cover exactly the same index range per tile, so the tile sums agree.
template <class F>
int exclusive_scan(F f, int64_t n, int64_t* out, int64_t* tile_scratch, cudaStream_t st) {
  int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (ntiles == 0) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), st);
    SFKV_LAUNCH_CHECK("scan (empty)");
    return 0;
  }
  if (ntiles <= SCAN_SINGLE_MAX_TILES) {
    SFKV_CUDA(launch_pdl(scan_single_kernel<F>, dim3(1), dim3(SCAN_THREADS), st, f, n, out));
    return 0;
  }
  SFKV_CUDA(launch_pdl(scan_reduce_kernel<F>, dim3((unsigned)ntiles), dim3(SCAN_THREADS), st, f, n, tile_scratch));
  SFKV_CUDA(launch_pdl(scan_tiles_kernel, dim3(1), dim3(1024), st, tile_scratch, ntiles));
  SFKV_CUDA(launch_pdl(scan_apply_kernel<F>, dim3((unsigned)ntiles), dim3(SCAN_THREADS), st, f, n,
                       (const int64_t*)tile_scratch, out));
  return 0;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline int check_device(int dev) {
  // cached per device: cudaGetDeviceProperties costs milliseconds, entry points call this often
  static int ok[64] = {0};
  if (dev >= 0 && dev < 64 && ok[dev]) return 0;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(SFKV_ENODEV, "no CUDA device visible");
  if (dev < 0 || dev >= n) return fail(SFKV_ENODEV, "device ordinal out of range");
  int major = 0, minor = 0;
  SFKV_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  SFKV_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10) return fail(SFKV_ENODEV, "libsfkv is built for sm_100a (B200); device is sm_" +
                                                std::to_string(major * 10 + minor));
  if (dev < 64) ok[dev] = 1;
  return 0;
}

// ---- small device helpers ---------------------------------------------------------------
// Largest r in [0, n) with off[r] <= x (off non-decreasing, off[0] = 0 <= x).
__device__ __forceinline__ int64_t upper_index(const int64_t* __restrict__ off, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;  // invariant: off[lo] <= x, answer in [lo, hi)
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void atomic_add_i64(long long* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

struct ReqBlocks {  // blocks of request i of a CSR batch
  const int64_t* tok_off;
  __device__ int64_t operator()(int64_t i) const { return (tok_off[i + 1] - tok_off[i] + 15) / 16; }
};

inline int grid_for(int64_t work, int threads, int max_blocks) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

}  // namespace sfkv
