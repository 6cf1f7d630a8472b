// K5/K8: KV payload movement — commit scatter with copy-on-share, gather, cross-pool handoff.
//
// The reference moves no KV bytes (its "cache" is a token list, simulated_backend.hpp:115); these
// kernels move the Llama-3-8B-shaped payload the build keeps per block:
//   block  [n_slabs = 64][16 slots][slab_row_bytes = 2048]  = 2 MiB, contiguous
//   staging (prefill output / gather output) [slab][token][slab_row_bytes]
// Every unit of work is (block, slab): up to 16 rows x 2 KiB that are contiguous on both sides
// (32 KiB for a full block), copied by one warp with 16-B vector loads/stores, eight loads in flight
// per lane before the stores (L1::no_allocate loads, streaming stores). Units are spread over a
// persistent grid (8 CTAs x 8 warps per SM) in grid-stride order. HBM-bound: algorithmic bytes are
// 2 x bytes moved (read + write); no tensor cores.
#include "pool.cuh"

namespace sfkv {



__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// One warp copies `bytes` (multiple of 16, both sides 16-B aligned).
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                          int64_t bytes, int lane) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  const int64_t n = bytes >> 4;
  constexpr int U = 8;
  int64_t i = lane;
  for (; i + (U - 1) * 32 < n; i += U * 32) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(s + i + u * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) st_stream(d + i + u * 32, v[u]);
  }
  for (; i < n; i += 32) st_stream(d + i, ld_stream(s + i));
}

struct PayloadKernelArgs {
  PayloadJob j;
  uint8_t* kv;
  int64_t block_bytes;
  int32_t n_slabs;
  int64_t row;
  const uint8_t* staging;
  const int64_t* staging_off;
  const uint8_t* src_kv;   // handoff source payload (another pool, or a peer rank's over NVLink)
  const int32_t* src_blk;  // handoff source block of every batch item
  int64_t src_block_bytes;
  int64_t src_n_blocks;
  int* error_out;          // the destination pool's sticky error
};

__global__ void __launch_bounds__(256) payload_kernel(PayloadKernelArgs P) {
  pdl_enter();
  const PayloadJob& j = P.j;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (*j.error) return;
  const int64_t total = j.rank[j.n_items] * P.n_slabs;
  for (int64_t u = warp; u < total; u += nwarps) {
    const int64_t a = u / P.n_slabs;
    const int s = (int)(u - a * P.n_slabs);
    const int64_t item = j.alloc_list[a];
    const int64_t r = upper_index(j.blk_off, j.n, item);
    const int64_t k = item - j.blk_off[r];
    const int64_t len = j.tok_off[r + 1] - j.tok_off[r];
    const int64_t rem = len - k * BT;
    const int nval = (int)(rem < BT ? rem : BT);
    const int64_t M = j.M[r];
    int64_t j0 = M - k * BT;
    j0 = j0 < 0 ? 0 : (j0 > nval ? nval : j0);
    uint8_t* dst = P.kv + (int64_t)j.bid[item] * P.block_bytes + (int64_t)s * BT * P.row;
    if (j0 > 0) {  // copy-on-share: cached rows of the old pin's boundary block
      const int32_t old = j.cow_src[a];
      const uint8_t* src = P.kv + (int64_t)old * P.block_bytes + (int64_t)s * BT * P.row;
      warp_copy(dst, src, j0 * P.row, lane);
    }
    if (nval > j0) {
      const uint8_t* src;
      if (P.src_kv) {  // handoff: same rows of the source block of this item
        const int32_t sb = P.src_blk[item];
        if ((uint64_t)sb >= (uint64_t)P.src_n_blocks) {  // device-side guard on the peer's region
          if (lane == 0) *P.error_out = SFKV_EINVAL;
          continue;
        }
        src = P.src_kv + (int64_t)sb * P.src_block_bytes + ((int64_t)s * BT + j0) * P.row;
      } else {  // staging rows [M, P): row index (k*16 + j0 - M)
        src = P.staging + P.staging_off[r] + ((int64_t)s * (len - M) + k * BT + j0 - M) * P.row;
      }
      warp_copy(dst + j0 * P.row, src, (nval - j0) * P.row, lane);
    }
  }
}

static int sm_count_p() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int launch_payload(sfkv_pool* p, const PayloadJob& j, const void* kv_src, const int64_t* kv_src_off,
                   const PayloadSource* src, cudaStream_t st) {
  PayloadKernelArgs P;
  P.j = j;
  P.kv = p->kv;
  P.block_bytes = p->block_bytes;
  P.n_slabs = p->cfg.n_slabs;
  P.row = p->cfg.slab_row_bytes;
  P.staging = static_cast<const uint8_t*>(kv_src);
  P.staging_off = kv_src_off;
  P.src_kv = src ? src->kv : nullptr;
  P.src_blk = src ? src->blk : nullptr;
  P.src_block_bytes = src ? src->block_bytes : 0;
  P.src_n_blocks = src ? src->n_blocks : 0;
  P.error_out = &p->ctr->error;
  SFKV_CUDA(launch_pdl(payload_kernel, dim3(sm_count_p() * 8), dim3(256), st, P));
  return 0;
}

// ---- gather: pins -> contiguous staging [slab][token][row] --------------------------------
struct GatherArgs {
  int64_t n;
  const int32_t* wf;
  const int64_t* blk_off;  // scan of pin block counts
  uint8_t* dst;
  const int64_t* dst_off;
  const int64_t* pin_len;
  const int32_t* pin_blk;
  int32_t max_pin_blocks;
  const uint8_t* kv;
  int64_t block_bytes;
  int32_t n_slabs;
  int64_t row;
};

__global__ void __launch_bounds__(256) gather_kernel(GatherArgs G) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = G.blk_off[G.n] * G.n_slabs;
  for (int64_t u = warp; u < total; u += nwarps) {
    const int64_t item = u / G.n_slabs;
    const int s = (int)(u - item * G.n_slabs);
    const int64_t r = upper_index(G.blk_off, G.n, item);
    const int64_t k = item - G.blk_off[r];
    const int32_t w = G.wf[r];
    const int64_t L = G.pin_len[w];
    const int64_t rem = L - k * BT;
    const int nval = (int)(rem < BT ? rem : BT);
    const int32_t id = G.pin_blk[(int64_t)w * G.max_pin_blocks + k];
    const uint8_t* src = G.kv + (int64_t)id * G.block_bytes + (int64_t)s * BT * G.row;
    uint8_t* dst = G.dst + G.dst_off[r] + ((int64_t)s * L + k * BT) * G.row;
    warp_copy(dst, src, nval * G.row, lane);
  }
}

struct PinBlockCount {  // device-side slot guard: an out-of-range slot gathers nothing
  const int32_t* wf;
  const int64_t* pin_len;
  const int32_t* pin_nblk;
  int32_t max_wf;
  int* error;
  __device__ int64_t operator()(int64_t i) const {
    const int32_t w = wf[i];
    if ((uint32_t)w >= (uint32_t)max_wf) {
      *error = SFKV_EINVAL;
      return 0;
    }
    return pin_len[w] < 0 ? 0 : pin_nblk[w];
  }
};

int gather_dev(sfkv_pool* p, int64_t n, const int32_t* wf, void* dst, const int64_t* dst_off) {
  if (!p->kv) return fail(SFKV_EINVAL, "gather: pool has no KV payload (n_slabs == 0)");
  if (n <= 0) return 0;
  cudaStream_t st = p->stream;
  Carver cv;
  const size_t o_off = cv.take<int64_t>(n + 1), o_tmp = cv.take<int64_t>(scan_scratch_elems(n));
  if (int rc = p->small.ensure(cv.off)) return rc;
  char* base = p->small.as<char>();
  int64_t* blk_off = reinterpret_cast<int64_t*>(base + o_off);
  if (int rc = exclusive_scan(PinBlockCount{wf, p->pin_len, p->pin_nblk, p->cfg.max_workflows, &p->ctr->error}, n, blk_off,
                              reinterpret_cast<int64_t*>(base + o_tmp), st))
    return rc;
  GatherArgs G;
  G.n = n;
  G.wf = wf;
  G.blk_off = blk_off;
  G.dst = static_cast<uint8_t*>(dst);
  G.dst_off = dst_off;
  G.pin_len = p->pin_len;
  G.pin_blk = p->pin_blk;
  G.max_pin_blocks = p->cfg.max_pin_blocks;
  G.kv = p->kv;
  G.block_bytes = p->block_bytes;
  G.n_slabs = p->cfg.n_slabs;
  G.row = p->cfg.slab_row_bytes;
  gather_kernel<<<sm_count_p() * 8, 256, 0, st>>>(G);
  SFKV_LAUNCH_CHECK("gather_kernel");
  return 0;
}

}  // namespace sfkv
