// extern "C" entry points of libsfkv.so (include/sfkv.h). Validation, host<->device staging for
// the host-pointer variants, and per-device contexts for the pool-less memory-manager / mapper
// calls. Everything below the ABI runs the sm_100a kernels in match.cu, commit.cu, copy.cu and
// mm_map.cu; there is no CPU compute path.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pool.cuh"

namespace sfkv {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? SFKV_ENOMEM : SFKV_ECUDA;
}

__global__ void __launch_bounds__(1024) scan_tiles_kernel(int64_t* tile_sums, int64_t ntiles) {
  pdl_enter();
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += 1024) {
    const int64_t i = base + threadIdx.x;
    int64_t v = i < ntiles ? tile_sums[i] : 0, agg;
    BS(tmp).ExclusiveSum(v, v, agg);
    if (i < ntiles) tile_sums[i] = v + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
}

__global__ void pool_init_kernel(sfkv_pool P) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < P.table_slots; i += stride) {
    P.slots[i].key = KEY_EMPTY;
    P.slots[i].val = -1;
    P.slots[i].pad = 0;
    P.towner[i] = NO_OWNER;
  }
  for (int64_t w = t0; w < P.n_words; w += stride) {
    const int64_t lo = w * 32, hi = lo + 32;
    P.free_bits[w] = hi <= P.cfg.n_blocks ? 0xffffffffu
                                          : (P.cfg.n_blocks > lo ? ((1u << (P.cfg.n_blocks - lo)) - 1u) : 0u);
  }
  for (int64_t w = t0; w < P.cfg.max_workflows; w += stride) {
    P.pin_len[w] = -1;
    P.pin_nblk[w] = 0;
  }
  for (int64_t b = t0; b < P.cfg.n_blocks; b += stride) {
    P.blk_ref[b] = 0;
    P.blk_in_table[b] = 0;
    P.blk_n[b] = 0;
    P.blk_slot[b] = -1;
    P.blk_parent[b] = -1;
  }
}

template <class T>
static int dalloc(T** p, size_t n) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_fail(e, "pool cudaMalloc");
  }
  return 0;
}

static void pool_free(sfkv_pool* p) {
  if (!p) return;
  cudaFree(p->pin_len);
  cudaFree(p->pin_nblk);
  cudaFree(p->pin_blk);
  cudaFree(p->pin_tok);
  cudaFree(p->blk_key);
  cudaFree(p->blk_parent);
  cudaFree(p->blk_tok);
  cudaFree(p->blk_n);
  cudaFree(p->blk_in_table);
  cudaFree(p->blk_ref);
  cudaFree(p->blk_slot);
  cudaFree(p->free_bits);
  cudaFree(p->slots);
  cudaFree(p->towner);
  cudaFree(p->kv);
  cudaFree(p->ctr);
  if (p->ctr_host) cudaFreeHost(p->ctr_host);
  if (p->host_stage) cudaFreeHost(p->host_stage);
  p->scratch.release();
  p->small.release();
  p->io.release();
  p->prep_status.release();
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  if (p->aux) cudaStreamDestroy(p->aux);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  delete p;
}

// sfkv_pool_reserve: pins copied into the grown [W2][MB2] block tables and [W2][32 G2][stride]
// token copies; new slots start without a pin.
__global__ void pin_regrow_kernel(const int64_t* len0, const int32_t* nblk0, const int32_t* blk0,
                                  const uint32_t* tok0, int64_t W0, int64_t MB0, int64_t G0,
                                  int64_t* len1, int32_t* nblk1, int32_t* blk1, uint32_t* tok1,
                                  int64_t W1, int64_t MB1, int64_t G1) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t w = t0; w < W1; w += stride) {
    len1[w] = w < W0 ? len0[w] : -1;
    nblk1[w] = w < W0 ? nblk0[w] : 0;
  }
  // one thread per (workflow, block) of the old layout: table entry + its 16 token words
  for (int64_t i = t0; i < W0 * MB0; i += stride) {
    const int64_t w = i / MB0, k = i - w * MB0;
    if (len0[w] < 0 || k >= nblk0[w]) continue;
    blk1[w * MB1 + k] = blk0[i];
    const uint4* s = reinterpret_cast<const uint4*>(tok0 + pin_tok_index(w, k, 0, G0));
    uint4* d = reinterpret_cast<uint4*>(tok1 + pin_tok_index(w, k, 0, G1));
#pragma unroll
    for (int q = 0; q < BT / 4; ++q) d[q] = s[q];
  }
}

// New block ids [B0, B1): unreferenced, free, outside the table.
__global__ void blocks_grow_kernel(sfkv_pool P, int64_t B0) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = B0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < P.cfg.n_blocks; b += stride) {
    P.blk_ref[b] = 0;
    P.blk_in_table[b] = 0;
    P.blk_n[b] = 0;
    P.blk_slot[b] = -1;
    P.blk_key[b] = 0;
    P.blk_parent[b] = -1;
    atomicOr(&P.free_bits[b >> 5], 1u << (b & 31));
  }
}

template <class T>
static int dgrow(T** p, size_t old_n, size_t new_n, cudaStream_t st) {
  T* q = nullptr;
  if (int rc = dalloc(&q, new_n)) return rc;
  if (old_n) {
    cudaError_t e = cudaMemcpyAsync(q, *p, old_n * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      cudaFree(q);
      return cuda_fail(e, "pool_reserve copy");
    }
  }
  cudaStreamSynchronize(st);
  cudaFree(*p);
  *p = q;
  return 0;
}

static int read_counters(sfkv_pool* p) {
  SFKV_CUDA(cudaMemcpyAsync(p->ctr_host, p->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

// The pool's sticky device-side error, reported once: read, cleared, and turned into a status.
static int check_sticky(sfkv_pool* p) {
  if (int rc = read_counters(p)) return rc;
  const int e = p->ctr_host->error;
  if (!e) return 0;
  SFKV_CUDA(cudaMemsetAsync(&p->ctr->error, 0, sizeof(int), p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  p->ctr_host->error = 0;
  if (e == SFKV_EPOOL) return fail(e, "physical block pool or block table exhausted");
  if (e == SFKV_ESTALE) return fail(e, "payload staging assumed a different cached prefix M");
  if (e == SFKV_EINVAL) return fail(e, "device-side argument check: workflow slot out of range");
  return fail(e, "device-side error");
}

// _dev entry points: pointer alignment the kernels rely on (uint4 / TMA token loads, 8-B offsets)
static bool misaligned(const void* ptr, uintptr_t a) { return ptr && (reinterpret_cast<uintptr_t>(ptr) & (a - 1)); }
static int check_dev_args(const char* fn, const int32_t* wf, const int64_t* tok_off, const uint32_t* tok) {
  if (misaligned(tok, 16)) return fail(SFKV_EINVAL, std::string(fn) + ": tok must be 16-byte aligned");
  if (misaligned(tok_off, 8)) return fail(SFKV_EINVAL, std::string(fn) + ": tok_off must be 8-byte aligned");
  if (misaligned(wf, 4)) return fail(SFKV_EINVAL, std::string(fn) + ": wf must be 4-byte aligned");
  return 0;
}

// Host-pointer staging: copies into p->io and returns device pointers.
struct IoLayout {
  Carver cv;
  std::vector<std::pair<size_t, const void*>> in;  // (offset, host src) with sizes below
  std::vector<size_t> in_bytes;
};

}  // namespace sfkv

using namespace sfkv;

extern "C" {

const char* sfkv_last_error(void) { return g_err.c_str(); }
int sfkv_abi_version(void) { return SFKV_ABI_VERSION; }

uint64_t sfkv_block_digest(uint64_t k, uint32_t n, const uint32_t* t) {
  uint32_t z[BT];
  for (int j = 0; j < BT; ++j) z[j] = (uint32_t)j < n ? t[j] : 0u;
  return block_digest_words(k, n, z);
}
uint64_t sfkv_chain_finalize(uint64_t s) { return chain_finalize(s); }

int sfkv_pool_create(const sfkv_pool_config* cfg, sfkv_pool** out) {
  if (!cfg || !out) return fail(SFKV_EINVAL, "pool_create: null argument");
  if (cfg->max_workflows <= 0 || cfg->n_blocks <= 0 || cfg->capacity_tokens <= 0 ||
      cfg->max_pin_blocks <= 0 || cfg->max_pin_blocks > (1 << 26) || cfg->table_log2 < 4 || cfg->table_log2 > 40 || cfg->n_slabs < 0 ||
      (cfg->n_slabs > 0 && (cfg->slab_row_bytes <= 0 || cfg->slab_row_bytes % 16 != 0)) ||
      cfg->n_blocks >= INT32_MAX)
    return fail(SFKV_EINVAL, "pool_create: invalid configuration");
  if ((int64_t(1) << cfg->table_log2) <= cfg->n_blocks)
    return fail(SFKV_EINVAL, "pool_create: table must have more slots than blocks");
  if (int rc = check_device(cfg->device)) return rc;
  DeviceGuard g(cfg->device);
  auto* p = new sfkv_pool;
  p->cfg = *cfg;
  p->block_bytes = (int64_t)cfg->n_slabs * BT * cfg->slab_row_bytes;
  p->n_words = (cfg->n_blocks + 31) / 32;
  p->table_slots = int64_t(1) << cfg->table_log2;
  const size_t W = cfg->max_workflows, B = cfg->n_blocks, MB = cfg->max_pin_blocks;
  int rc = 0;
  if ((rc = dalloc(&p->pin_len, W)) || (rc = dalloc(&p->pin_nblk, W)) ||
      (rc = dalloc(&p->pin_blk, W * MB)) || (rc = dalloc(&p->pin_tok, W * (size_t)pin_groups(*cfg) * 32 * PIN_STRIDE)) ||
      (rc = dalloc(&p->blk_key, B)) || (rc = dalloc(&p->blk_parent, B)) || (rc = dalloc(&p->blk_tok, B * BT)) ||
      (rc = dalloc(&p->blk_n, B)) || (rc = dalloc(&p->blk_in_table, B)) ||
      (rc = dalloc(&p->blk_ref, B)) || (rc = dalloc(&p->blk_slot, B)) ||
      (rc = dalloc(&p->free_bits, (size_t)p->n_words)) ||
      (rc = dalloc(&p->slots, (size_t)p->table_slots)) ||
      (rc = dalloc(&p->towner, (size_t)p->table_slots)) || (rc = dalloc(&p->ctr, 1))) {
    pool_free(p);
    return rc;
  }
  if (p->block_bytes > 0 && (rc = dalloc(&p->kv, B * (size_t)p->block_bytes))) {
    pool_free(p);
    return rc;
  }
  cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p->ctr_host), sizeof(DevCounters));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    pool_free(p);
    return cuda_fail(e, "pool_create");
  }
  p->own_stream = true;
  cudaMemsetAsync(p->ctr, 0, sizeof(DevCounters), p->stream);
  cudaMemsetAsync(p->blk_tok, 0, B * BT * sizeof(uint32_t), p->stream);
  if (p->kv) cudaMemsetAsync(p->kv, 0, B * (size_t)p->block_bytes, p->stream);
  pool_init_kernel<<<1184, 256, 0, p->stream>>>(*p);
  e = cudaStreamSynchronize(p->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    pool_free(p);
    return cuda_fail(e, "pool_create init");
  }
  *out = p;
  return 0;
}

int sfkv_pool_reserve(sfkv_pool* p, int32_t max_workflows, int32_t max_pin_blocks, int64_t n_blocks) {
  if (!p) return fail(SFKV_EINVAL, "null pool");
  if (max_pin_blocks > (1 << 26) || n_blocks >= INT32_MAX)
    return fail(SFKV_EINVAL, "pool_reserve: size out of range");
  DeviceGuard g(p->cfg.device);
  cudaStream_t st = p->stream;
  SFKV_CUDA(cudaStreamSynchronize(st));
  if (p->aux) SFKV_CUDA(cudaStreamSynchronize(p->aux));
  const int64_t W0 = p->cfg.max_workflows, MB0 = p->cfg.max_pin_blocks, B0 = p->cfg.n_blocks;
  const int64_t W1 = std::max<int64_t>(W0, max_workflows), MB1 = std::max<int64_t>(MB0, max_pin_blocks),
                B1 = std::max<int64_t>(B0, n_blocks);
  if (W1 > W0 || MB1 > MB0) {
    sfkv_pool_config c1 = p->cfg;
    c1.max_workflows = (int32_t)W1;
    c1.max_pin_blocks = (int32_t)MB1;
    const int64_t G0 = pin_groups(p->cfg), G1 = pin_groups(c1);
    int64_t* len1 = nullptr;
    int32_t *nblk1 = nullptr, *blk1 = nullptr;
    uint32_t* tok1 = nullptr;
    int rc = 0;
    if ((rc = dalloc(&len1, W1)) || (rc = dalloc(&nblk1, W1)) || (rc = dalloc(&blk1, W1 * MB1)) ||
        (rc = dalloc(&tok1, W1 * G1 * 32 * PIN_STRIDE))) {
      cudaFree(len1); cudaFree(nblk1); cudaFree(blk1); cudaFree(tok1);
      return rc;
    }
    pin_regrow_kernel<<<1184, 256, 0, st>>>(p->pin_len, p->pin_nblk, p->pin_blk, p->pin_tok, W0, MB0, G0,
                                            len1, nblk1, blk1, tok1, W1, MB1, G1);
    SFKV_LAUNCH_CHECK("pin_regrow_kernel");
    SFKV_CUDA(cudaStreamSynchronize(st));
    cudaFree(p->pin_len); cudaFree(p->pin_nblk); cudaFree(p->pin_blk); cudaFree(p->pin_tok);
    p->pin_len = len1; p->pin_nblk = nblk1; p->pin_blk = blk1; p->pin_tok = tok1;
    p->cfg.max_workflows = (int32_t)W1;
    p->cfg.max_pin_blocks = (int32_t)MB1;
  }
  if (B1 > B0) {
    if (p->kv && p->exported)
      return fail(SFKV_EINVAL, "pool_reserve: the KV region was exported (CUDA IPC); it cannot move");
    const int64_t nw1 = (B1 + 31) / 32;
    int rc = 0;
    if ((rc = dgrow(&p->blk_key, B0, B1, st)) || (rc = dgrow(&p->blk_parent, B0, B1, st)) ||
        (rc = dgrow(&p->blk_tok, B0 * BT, B1 * BT, st)) ||
        (rc = dgrow(&p->blk_n, B0, B1, st)) || (rc = dgrow(&p->blk_in_table, B0, B1, st)) ||
        (rc = dgrow(&p->blk_ref, B0, B1, st)) || (rc = dgrow(&p->blk_slot, B0, B1, st)) ||
        (rc = dgrow(&p->free_bits, p->n_words, nw1, st)))
      return rc;
    SFKV_CUDA(cudaMemsetAsync(p->blk_tok + B0 * BT, 0, (B1 - B0) * BT * sizeof(uint32_t), st));
    if (nw1 > p->n_words)
      SFKV_CUDA(cudaMemsetAsync(p->free_bits + p->n_words, 0, (nw1 - p->n_words) * sizeof(uint32_t), st));
    if (p->kv) {
      if ((rc = dgrow(&p->kv, B0 * p->block_bytes, B1 * p->block_bytes, st))) return rc;
      SFKV_CUDA(cudaMemsetAsync(p->kv + B0 * p->block_bytes, 0, (B1 - B0) * p->block_bytes, st));
    }
    p->cfg.n_blocks = B1;
    p->n_words = nw1;
    blocks_grow_kernel<<<1184, 256, 0, st>>>(*p, B0);
    SFKV_LAUNCH_CHECK("blocks_grow_kernel");
    int log2 = p->cfg.table_log2;
    while ((int64_t(1) << log2) < 2 * B1) ++log2;
    if (log2 != p->cfg.table_log2) {  // keep the load factor <= 1/2: a larger table, re-indexed
      Slot* slots1 = nullptr;
      int64_t* towner1 = nullptr;
      if ((rc = dalloc(&slots1, size_t(1) << log2)) || (rc = dalloc(&towner1, size_t(1) << log2))) {
        cudaFree(slots1);
        return rc;
      }
      SFKV_CUDA(cudaStreamSynchronize(st));
      cudaFree(p->slots);
      cudaFree(p->towner);
      p->slots = slots1;
      p->towner = towner1;
      p->table_slots = int64_t(1) << log2;
      p->cfg.table_log2 = log2;
      if ((rc = rebuild_table_now(p))) return rc;
    }
  }
  SFKV_CUDA(cudaStreamSynchronize(st));
  SFKV_CUDA(cudaGetLastError());
  return 0;
}

int sfkv_pool_config_get(sfkv_pool* p, sfkv_pool_config* out) {
  if (!p || !out) return fail(SFKV_EINVAL, "null argument");
  *out = p->cfg;
  return 0;
}

int sfkv_pool_destroy(sfkv_pool* p) {
  if (!p) return 0;
  DeviceGuard g(p->cfg.device);
  cudaStreamSynchronize(p->stream);
  pool_free(p);
  return 0;
}

int sfkv_pool_set_stream(sfkv_pool* p, void* stream) {
  if (!p) return fail(SFKV_EINVAL, "null pool");
  DeviceGuard g(p->cfg.device);
  cudaStreamSynchronize(p->stream);
  if (p->own_stream) cudaStreamDestroy(p->stream);
  p->stream = static_cast<cudaStream_t>(stream);
  p->own_stream = false;
  return 0;
}

int sfkv_pool_sync(sfkv_pool* p) {
  if (!p) return fail(SFKV_EINVAL, "null pool");
  DeviceGuard g(p->cfg.device);
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return check_sticky(p);  // device-side errors of the _dev calls since the last report
}

int sfkv_pool_kv(sfkv_pool* p, void** kv, int64_t* block_bytes) {
  if (!p || !kv || !block_bytes) return fail(SFKV_EINVAL, "null argument");
  *kv = p->kv;
  *block_bytes = p->block_bytes;
  return 0;
}

// ---------------------------------------------------------------- lookup ------------------
static int match_common(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                        const uint32_t* tok, int64_t* out_M, uint64_t* out_hash, int32_t* out_block,
                        int64_t* out_hit, int64_t n_items_bound, int64_t n_tok_bound) {
  cudaStream_t st = p->stream;
  const int64_t n_items = n_items_bound;  // upper bound; kernels read the exact count on device
  Carver c0;
  const size_t o_blk = c0.take<int64_t>(n + 1);
  if (int rc = p->small.ensure(c0.off)) return rc;
  int64_t* blk_off = reinterpret_cast<int64_t*>(p->small.as<char>() + o_blk);  // written by prep
  Carver cv;
  const size_t o_tile = cv.take<int64_t>(match_tile_state_elems(n_items, n));
  if (int rc = p->scratch.ensure(cv.off)) return rc;
  MatchArgs a{};
  a.n = n;
  a.wf = wf;
  a.tok_off = tok_off;
  a.tok = tok;
  a.blk_off = blk_off;
  a.n_items = n_items;
  a.n_tok_bound = n_tok_bound;
  a.out_M = out_M;
  a.out_hash = out_hash;
  a.out_block = out_block;
  a.out_hit = out_hit;
  return launch_match(p, a, reinterpret_cast<int64_t*>(p->scratch.as<char>() + o_tile), st);
}

static int64_t host_items(int64_t n, const int64_t* tok_off) {
  int64_t s = 0;
  for (int64_t r = 0; r < n; ++r) s += (tok_off[r + 1] - tok_off[r] + BT - 1) / BT;
  return s;
}

static int validate_batch_host(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off) {
  if (n < 0 || !tok_off) return fail(SFKV_EINVAL, "invalid batch");
  if (tok_off[0] != 0) return fail(SFKV_EINVAL, "tok_off[0] must be 0");
  for (int64_t r = 0; r < n; ++r) {
    if (tok_off[r + 1] < tok_off[r]) return fail(SFKV_EINVAL, "tok_off must be non-decreasing");
    if (wf && (wf[r] < 0 || wf[r] >= p->cfg.max_workflows))
      return fail(SFKV_EINVAL, "workflow slot out of range");
  }
  return 0;
}

// Copies (wf, tok_off, tok) to the device io buffer; returns device pointers.
static int stage_batch(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                       const uint32_t* tok, size_t extra_bytes, int32_t** d_wf, int64_t** d_off,
                       uint32_t** d_tok, char** d_extra) {
  const int64_t T = tok_off[n];
  Carver cv;
  const size_t o_wf = cv.take<int32_t>(n), o_off = cv.take<int64_t>(n + 1),
               o_tok = cv.take<uint32_t>(T + 4), o_ex = cv.take<char>(extra_bytes);
  if (int rc = p->io.ensure(cv.off)) return rc;
  char* b = p->io.as<char>();
  cudaStream_t st = p->stream;
  if (wf) SFKV_CUDA(cudaMemcpyAsync(b + o_wf, wf, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_off, tok_off, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (T > 0) SFKV_CUDA(cudaMemcpyAsync(b + o_tok, tok, T * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  *d_wf = reinterpret_cast<int32_t*>(b + o_wf);
  *d_off = reinterpret_cast<int64_t*>(b + o_off);
  *d_tok = reinterpret_cast<uint32_t*>(b + o_tok);
  if (d_extra) *d_extra = b + o_ex;
  return 0;
}

int sfkv_match_batch(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                     const uint32_t* tok, int64_t* out_M, uint64_t* out_hash) {
  if (!p || !out_M) return fail(SFKV_EINVAL, "match_batch: null argument");
  if (n == 0) return 0;
  if (!wf) return fail(SFKV_EINVAL, "match_batch: null wf");
  if (int rc = validate_batch_host(p, n, wf, tok_off)) return rc;
  DeviceGuard g(p->cfg.device);
  const int64_t items = host_items(n, tok_off);
  int32_t* dwf;
  int64_t* doff;
  uint32_t* dtok;
  char* ex;
  const size_t out_bytes = n * sizeof(int64_t) + 256 + (out_hash ? items * sizeof(uint64_t) : 0);
  if (int rc = stage_batch(p, n, wf, tok_off, tok, out_bytes, &dwf, &doff, &dtok, &ex)) return rc;
  int64_t* dM = reinterpret_cast<int64_t*>(ex);
  uint64_t* dh = out_hash ? reinterpret_cast<uint64_t*>(ex + ((n * sizeof(int64_t) + 255) & ~size_t(255))) : nullptr;
  if (int rc = match_common(p, n, dwf, doff, dtok, dM, dh, nullptr, nullptr, items, tok_off[n])) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_M, dM, n * sizeof(int64_t), cudaMemcpyDeviceToHost, p->stream));
  if (out_hash && items)
    SFKV_CUDA(cudaMemcpyAsync(out_hash, dh, items * sizeof(uint64_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

int sfkv_match_batch_dev(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                         const uint32_t* tok, int64_t n_tokens, int64_t* out_M, uint64_t* out_hash) {
  if (!p || !wf || !tok_off || !tok || !out_M || n_tokens < 0)
    return fail(SFKV_EINVAL, "match_batch_dev: bad argument");
  if (n <= 0) return n == 0 ? 0 : fail(SFKV_EINVAL, "negative batch");
  if (int rc = check_dev_args("match_batch_dev", wf, tok_off, tok)) return rc;
  if (misaligned(out_M, 8) || misaligned(out_hash, 8)) return fail(SFKV_EINVAL, "match_batch_dev: unaligned output");
  DeviceGuard g(p->cfg.device);
  return match_common(p, n, wf, tok_off, tok, out_M, out_hash, nullptr, nullptr, n + n_tokens / BT, n_tokens);
}

int sfkv_lookup_batch(sfkv_pool* p, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                      int32_t* out_block, int64_t* out_hit) {
  if (!p || !out_block || !out_hit) return fail(SFKV_EINVAL, "lookup_batch: null argument");
  if (n == 0) return 0;
  if (int rc = validate_batch_host(p, n, nullptr, tok_off)) return rc;
  DeviceGuard g(p->cfg.device);
  const int64_t items = host_items(n, tok_off);
  int32_t* dwf;
  int64_t* doff;
  uint32_t* dtok;
  char* ex;
  const size_t o2 = (n * sizeof(int64_t) + 255) & ~size_t(255);
  if (int rc = stage_batch(p, n, nullptr, tok_off, tok, o2 + items * sizeof(int32_t) + 16, &dwf, &doff, &dtok, &ex))
    return rc;
  int64_t* dhit = reinterpret_cast<int64_t*>(ex);
  int32_t* dblk = reinterpret_cast<int32_t*>(ex + o2);
  if (int rc = match_common(p, n, nullptr, doff, dtok, nullptr, nullptr, dblk, dhit, items, tok_off[n])) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_hit, dhit, n * sizeof(int64_t), cudaMemcpyDeviceToHost, p->stream));
  if (items)
    SFKV_CUDA(cudaMemcpyAsync(out_block, dblk, items * sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

int sfkv_lookup_batch_dev(sfkv_pool* p, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                          int64_t n_tokens, int32_t* out_block, int64_t* out_hit) {
  if (!p || !tok_off || !tok || !out_block || !out_hit || n_tokens < 0)
    return fail(SFKV_EINVAL, "lookup_batch_dev: bad argument");
  if (n <= 0) return n == 0 ? 0 : fail(SFKV_EINVAL, "negative batch");
  if (int rc = check_dev_args("lookup_batch_dev", nullptr, tok_off, tok)) return rc;
  if (misaligned(out_block, 4) || misaligned(out_hit, 8)) return fail(SFKV_EINVAL, "lookup_batch_dev: unaligned output");
  DeviceGuard g(p->cfg.device);
  return match_common(p, n, nullptr, tok_off, tok, nullptr, nullptr, out_block, out_hit, n + n_tokens / BT,
                      n_tokens);
}

// ---------------------------------------------------------------- retain ------------------
int sfkv_commit_batch(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                      const uint32_t* tok, const void* kv_src, const int64_t* kv_src_off,
                      const int64_t* m_expected, int32_t* out_status) {
  if (!p || !out_status) return fail(SFKV_EINVAL, "commit_batch: null argument");
  if (n == 0) return 0;
  if (!wf) return fail(SFKV_EINVAL, "commit_batch: null wf");
  if (int rc = validate_batch_host(p, n, wf, tok_off)) return rc;
  {
    std::vector<int32_t> s(wf, wf + n);
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end())
      return fail(SFKV_EINVAL, "commit_batch: workflow slots must be distinct within a batch");
  }
  if (kv_src && (!kv_src_off || !p->kv)) return fail(SFKV_EINVAL, "commit_batch: kv_src needs kv_src_off and a payload pool");
  DeviceGuard g(p->cfg.device);
  // Host staging copy: KV staging rows are [slab][P - M][row] per request; their total size is
  // only known from M. Host payload commits therefore take the device-resident path: the caller's
  // kv_src must be device memory (e.g. a torch tensor) even in this host-pointer variant.
  int32_t* dwf;
  int64_t* doff;
  uint32_t* dtok;
  char* ex;
  const size_t o_me = (n * sizeof(int32_t) + 255) & ~size_t(255);
  const size_t o_ko = o_me + ((n * sizeof(int64_t) + 255) & ~size_t(255));
  const size_t ex_bytes = o_ko + n * sizeof(int64_t) + 16;
  if (int rc = stage_batch(p, n, wf, tok_off, tok, ex_bytes, &dwf, &doff, &dtok, &ex)) return rc;
  int32_t* dst = reinterpret_cast<int32_t*>(ex);
  int64_t* dme = nullptr;
  int64_t* dko = nullptr;
  if (m_expected) {
    dme = reinterpret_cast<int64_t*>(ex + o_me);
    SFKV_CUDA(cudaMemcpyAsync(dme, m_expected, n * sizeof(int64_t), cudaMemcpyHostToDevice, p->stream));
  }
  if (kv_src) {
    dko = reinterpret_cast<int64_t*>(ex + o_ko);
    SFKV_CUDA(cudaMemcpyAsync(dko, kv_src_off, n * sizeof(int64_t), cudaMemcpyHostToDevice, p->stream));
  }
  if (int rc = commit_dev(p, n, dwf, doff, dtok, host_items(n, tok_off), tok_off[n], kv_src, dko, dme, dst,
                          nullptr))
    return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_status, dst, n * sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
  return check_sticky(p);
}

int sfkv_commit_batch_dev(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                          const uint32_t* tok, int64_t n_tokens, const void* kv_src,
                          const int64_t* kv_src_off, const int64_t* m_expected, int32_t* out_status) {
  if (!p || !wf || !tok_off || !tok || !out_status) return fail(SFKV_EINVAL, "commit_batch_dev: null argument");
  if (n <= 0) return n == 0 ? 0 : fail(SFKV_EINVAL, "negative batch");
  if (kv_src && (!kv_src_off || !p->kv)) return fail(SFKV_EINVAL, "commit_batch_dev: kv_src needs kv_src_off and a payload pool");
  if (int rc = check_dev_args("commit_batch_dev", wf, tok_off, tok)) return rc;
  if (misaligned(kv_src_off, 8) || misaligned(m_expected, 8) || misaligned(out_status, 4))
    return fail(SFKV_EINVAL, "commit_batch_dev: unaligned argument");
  DeviceGuard g(p->cfg.device);
  if (n_tokens < 0) return fail(SFKV_EINVAL, "commit_batch_dev: negative n_tokens");
  return commit_dev(p, n, wf, tok_off, tok, n + n_tokens / BT, n_tokens, kv_src, kv_src_off, m_expected,
                    out_status, nullptr);
}

// ---------------------------------------------------------------- evict -------------------
int sfkv_flush(sfkv_pool* p, int32_t wf, int64_t* freed) {
  if (!p || !freed) return fail(SFKV_EINVAL, "flush: null argument");
  if (wf != SFKV_FLUSH_ALL && (wf < 0 || wf >= p->cfg.max_workflows))
    return fail(SFKV_EINVAL, "flush: workflow slot out of range");
  DeviceGuard g(p->cfg.device);
  p->flush_calls++;
  if (wf == SFKV_FLUSH_ALL) {
    if (int rc = read_counters(p)) return rc;
    *freed = p->ctr_host->occupancy;
    if (int rc = flush_dev(p, 0, nullptr, nullptr, true)) return rc;
    SFKV_CUDA(cudaStreamSynchronize(p->stream));
    return 0;
  }
  if (int rc = p->io.ensure(512)) return rc;
  int32_t* dwf = p->io.as<int32_t>();
  int64_t* dfreed = reinterpret_cast<int64_t*>(p->io.as<char>() + 256);
  SFKV_CUDA(cudaMemcpyAsync(dwf, &wf, sizeof(int32_t), cudaMemcpyHostToDevice, p->stream));
  if (int rc = flush_dev(p, 1, dwf, dfreed, false)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(freed, dfreed, sizeof(int64_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

int sfkv_flush_batch(sfkv_pool* p, int64_t n, const int32_t* wf, int64_t* out_freed) {
  if (!p || (n > 0 && (!wf || !out_freed))) return fail(SFKV_EINVAL, "flush_batch: null argument");
  if (n == 0) return 0;
  for (int64_t r = 0; r < n; ++r)
    if (wf[r] < 0 || wf[r] >= p->cfg.max_workflows) return fail(SFKV_EINVAL, "flush_batch: slot out of range");
  {
    std::vector<int32_t> s(wf, wf + n);
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end())
      return fail(SFKV_EINVAL, "flush_batch: workflow slots must be distinct within a batch");
  }
  DeviceGuard g(p->cfg.device);
  p->flush_calls += (uint64_t)n;
  const size_t o = (n * sizeof(int32_t) + 255) & ~size_t(255);
  if (int rc = p->io.ensure(o + n * sizeof(int64_t))) return rc;
  int32_t* dwf = p->io.as<int32_t>();
  int64_t* dfreed = reinterpret_cast<int64_t*>(p->io.as<char>() + o);
  SFKV_CUDA(cudaMemcpyAsync(dwf, wf, n * sizeof(int32_t), cudaMemcpyHostToDevice, p->stream));
  if (int rc = flush_dev(p, n, dwf, dfreed, false)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_freed, dfreed, n * sizeof(int64_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

// ---------------------------------------------------------------- inspection --------------
static int read_pin_len(sfkv_pool* p, int32_t wf, int64_t* len) {
  SFKV_CUDA(cudaMemcpyAsync(len, p->pin_len + wf, sizeof(int64_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

int sfkv_preserve(sfkv_pool* p, int32_t wf, int32_t* has_pin) {
  if (!p || !has_pin || wf < 0 || wf >= p->cfg.max_workflows) return fail(SFKV_EINVAL, "preserve: bad argument");
  DeviceGuard g(p->cfg.device);
  p->preserve_calls++;
  int64_t len = -1;
  if (int rc = read_pin_len(p, wf, &len)) return rc;
  *has_pin = len >= 0 ? 1 : 0;
  return 0;
}

int sfkv_pinned_token_count(sfkv_pool* p, int32_t wf, int64_t* n_tokens) {
  if (!p || !n_tokens || wf < 0 || wf >= p->cfg.max_workflows) return fail(SFKV_EINVAL, "pinned_token_count: bad argument");
  DeviceGuard g(p->cfg.device);
  int64_t len = -1;
  if (int rc = read_pin_len(p, wf, &len)) return rc;
  *n_tokens = len < 0 ? 0 : len;
  return 0;
}

int sfkv_cache_utilization(sfkv_pool* p, double* util) {
  if (!p || !util) return fail(SFKV_EINVAL, "cache_utilization: null argument");
  DeviceGuard g(p->cfg.device);
  if (int rc = read_counters(p)) return rc;
  *util = static_cast<double>(p->ctr_host->occupancy) / static_cast<double>(p->cfg.capacity_tokens);
  return 0;
}

int sfkv_stats(sfkv_pool* p, sfkv_pool_stats* o) {
  if (!p || !o) return fail(SFKV_EINVAL, "stats: null argument");
  DeviceGuard g(p->cfg.device);
  if (int rc = read_counters(p)) return rc;
  o->occupancy_tokens = p->ctr_host->occupancy;
  o->capacity_tokens = p->cfg.capacity_tokens;
  o->capacity_rejections = p->ctr_host->rejections;
  o->flush_calls = p->flush_calls;
  o->preserve_calls = p->preserve_calls;
  o->blocks_in_use = p->ctr_host->blocks_in_use;
  o->table_live = p->ctr_host->table_live;
  o->table_tombstones = p->ctr_host->table_tomb;
  return 0;
}

int sfkv_pin_blocks(sfkv_pool* p, int32_t wf, int32_t* ids, uint64_t* hashes, int32_t cap,
                    int32_t* n_blocks) {
  if (!p || !n_blocks || wf < 0 || wf >= p->cfg.max_workflows) return fail(SFKV_EINVAL, "pin_blocks: bad argument");
  DeviceGuard g(p->cfg.device);
  int64_t len = -1;
  int32_t nb = 0;
  if (int rc = read_pin_len(p, wf, &len)) return rc;
  SFKV_CUDA(cudaMemcpy(&nb, p->pin_nblk + wf, sizeof(int32_t), cudaMemcpyDeviceToHost));
  nb = len < 0 ? 0 : nb;
  *n_blocks = nb;
  const int32_t m = nb < cap ? nb : cap;
  const int64_t pb = (int64_t)wf * p->cfg.max_pin_blocks;
  std::vector<int32_t> idv(m > 0 ? m : 1);
  if (m) SFKV_CUDA(cudaMemcpy(idv.data(), p->pin_blk + pb, m * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (ids && m) std::copy(idv.begin(), idv.begin() + m, ids);
  for (int32_t k = 0; hashes && k < m; ++k)  // a block's key is its chained hash
    SFKV_CUDA(cudaMemcpy(hashes + k, p->blk_key + idv[k], sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return 0;
}

int sfkv_block_refcounts(sfkv_pool* p, uint32_t* out) {
  if (!p || !out) return fail(SFKV_EINVAL, "block_refcounts: null argument");
  DeviceGuard g(p->cfg.device);
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  SFKV_CUDA(cudaMemcpy(out, p->blk_ref, p->cfg.n_blocks * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return 0;
}

// ---------------------------------------------------------------- gather / handoff --------
int sfkv_gather_dev(sfkv_pool* p, int64_t n, const int32_t* wf, void* dst, const int64_t* dst_off) {
  if (!p || (n > 0 && (!wf || !dst || !dst_off))) return fail(SFKV_EINVAL, "gather_dev: null argument");
  DeviceGuard g(p->cfg.device);
  return gather_dev(p, n, wf, dst, dst_off);
}

__global__ void pin_tokens_kernel(const int32_t* pin_blk, const uint32_t* blk_tok, int32_t nb,
                                  uint32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)nb * BT;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = blk_tok[(int64_t)pin_blk[i / BT] * BT + (i % BT)];
}

int sfkv_pin_tokens(sfkv_pool* p, int32_t wf, uint32_t* out, int64_t cap, int64_t* n_tokens) {
  if (!p || !n_tokens || wf < 0 || wf >= p->cfg.max_workflows || (cap > 0 && !out))
    return fail(SFKV_EINVAL, "pin_tokens: bad argument");
  DeviceGuard g(p->cfg.device);
  int64_t L = -1;
  int32_t nb = 0;
  if (int rc = read_pin_len(p, wf, &L)) return rc;
  *n_tokens = L < 0 ? 0 : L;
  if (L <= 0 || cap <= 0) return 0;
  SFKV_CUDA(cudaMemcpy(&nb, p->pin_nblk + wf, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (int rc = p->io.ensure((size_t)nb * BT * sizeof(uint32_t))) return rc;
  uint32_t* d = p->io.as<uint32_t>();
  pin_tokens_kernel<<<grid_for((int64_t)nb * BT, 256, 1024), 256, 0, p->stream>>>(
      p->pin_blk + (int64_t)wf * p->cfg.max_pin_blocks, p->blk_tok, nb, d);
  SFKV_LAUNCH_CHECK("pin_tokens_kernel");
  const int64_t m = L < cap ? L : cap;
  SFKV_CUDA(cudaMemcpyAsync(out, d, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, p->stream));
  SFKV_CUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

int sfkv_handoff(sfkv_pool* src, int32_t wf_src, sfkv_pool* dst, int32_t wf_dst, int32_t* status) {
  if (!src || !dst || !status || wf_src < 0 || wf_src >= src->cfg.max_workflows || wf_dst < 0 ||
      wf_dst >= dst->cfg.max_workflows)
    return fail(SFKV_EINVAL, "handoff: bad argument");
  if (src->cfg.n_slabs != dst->cfg.n_slabs || src->cfg.slab_row_bytes != dst->cfg.slab_row_bytes)
    return fail(SFKV_EINVAL, "handoff: pools have different KV shapes");
  int64_t L = -1;
  int32_t nb = 0;
  {
    DeviceGuard g(src->cfg.device);
    if (int rc = read_pin_len(src, wf_src, &L)) return rc;
    if (L < 0) return fail(SFKV_EINVAL, "handoff: source workflow has no pin");
    SFKV_CUDA(cudaMemcpy(&nb, src->pin_nblk + wf_src, sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  DeviceGuard g(dst->cfg.device);
  if (src->cfg.device != dst->cfg.device) {
    cudaError_t e = cudaDeviceEnablePeerAccess(src->cfg.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "enable peer access");
    cudaGetLastError();
  }
  // tokens of the source pin -> dst io buffer (peer reads when the pools are on different GPUs)
  const size_t o_off = ((size_t)(nb * BT + 4) * sizeof(uint32_t) + 255) & ~size_t(255);
  if (int rc = dst->io.ensure(o_off + 2 * sizeof(int64_t) + 256 + 16)) return rc;
  uint32_t* dtok = dst->io.as<uint32_t>();
  int64_t* doff = reinterpret_cast<int64_t*>(dst->io.as<char>() + o_off);
  int32_t* dwf = reinterpret_cast<int32_t*>(dst->io.as<char>() + o_off + 64);
  int32_t* dst_status = reinterpret_cast<int32_t*>(dst->io.as<char>() + o_off + 128);
  // run the token gather on the destination device, reading the source pool through its pointer
  if (nb > 0) {
    pin_tokens_kernel<<<grid_for((int64_t)nb * BT, 256, 1024), 256, 0, dst->stream>>>(
        src->pin_blk + (int64_t)wf_src * src->cfg.max_pin_blocks, src->blk_tok, nb, dtok);
    SFKV_LAUNCH_CHECK("pin_tokens_kernel");
  }
  const int64_t off[2] = {0, L};
  SFKV_CUDA(cudaMemcpyAsync(doff, off, sizeof(off), cudaMemcpyHostToDevice, dst->stream));
  SFKV_CUDA(cudaMemcpyAsync(dwf, &wf_dst, sizeof(int32_t), cudaMemcpyHostToDevice, dst->stream));
  // the source pool's stream must not be mutating the pin meanwhile
  {
    DeviceGuard gs(src->cfg.device);
    SFKV_CUDA(cudaStreamSynchronize(src->stream));
  }
  PayloadSource ps;
  ps.kv = src->kv;
  ps.blk = src->pin_blk + (int64_t)wf_src * src->cfg.max_pin_blocks;  // item k = block k
  ps.block_bytes = src->block_bytes;
  ps.n_blocks = src->cfg.n_blocks;
  if (int rc = commit_dev(dst, 1, dwf, doff, dtok, nb, (int64_t)nb * BT, nullptr, nullptr, nullptr, dst_status,
                          dst->kv ? &ps : nullptr))
    return rc;
  SFKV_CUDA(cudaMemcpyAsync(status, dst_status, sizeof(int32_t), cudaMemcpyDeviceToHost, dst->stream));
  return check_sticky(dst);
}


// ---------------------------------------------------------------- cross-process handoff ---
int sfkv_pool_export(sfkv_pool* p, sfkv_ipc_handle* out) {
  if (!p || !out) return fail(SFKV_EINVAL, "pool_export: null argument");
  if (!p->kv) return fail(SFKV_EINVAL, "pool_export: pool has no KV payload (n_slabs == 0)");
  DeviceGuard g(p->cfg.device);
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(out->handle), "ipc handle size");
  cudaIpcMemHandle_t h;
  SFKV_CUDA(cudaIpcGetMemHandle(&h, p->kv));
  p->exported = true;
  memset(out, 0, sizeof(*out));
  memcpy(out->handle, &h, sizeof(h));
  out->kv_bytes = p->cfg.n_blocks * p->block_bytes;
  out->block_bytes = p->block_bytes;
  out->n_slabs = p->cfg.n_slabs;
  out->slab_row_bytes = p->cfg.slab_row_bytes;
  return 0;
}

int sfkv_peer_open(const sfkv_ipc_handle* h, int32_t device, sfkv_peer** out) {
  if (!h || !out) return fail(SFKV_EINVAL, "peer_open: null argument");
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  cudaIpcMemHandle_t ih;
  memcpy(&ih, h->handle, sizeof(ih));
  void* ptr = nullptr;
  SFKV_CUDA(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
  auto* peer = new sfkv_peer;
  peer->device = device;
  peer->kv = static_cast<uint8_t*>(ptr);
  peer->kv_bytes = h->kv_bytes;
  peer->block_bytes = h->block_bytes;
  peer->n_slabs = h->n_slabs;
  peer->slab_row_bytes = h->slab_row_bytes;
  *out = peer;
  return 0;
}

int sfkv_peer_close(sfkv_peer* peer) {
  if (!peer) return fail(SFKV_EINVAL, "peer_close: null peer");
  DeviceGuard g(peer->device);
  cudaError_t e = cudaIpcCloseMemHandle(peer->kv);
  delete peer;
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return 0;
}

int sfkv_pin_export(sfkv_pool* p, int32_t wf, uint32_t* tok, int32_t* block_ids, int64_t cap,
                    int64_t* n_tokens) {
  if (!p || !n_tokens || wf < 0 || wf >= p->cfg.max_workflows || (cap > 0 && (!tok || !block_ids)))
    return fail(SFKV_EINVAL, "pin_export: bad argument");
  if (int rc = sfkv_pin_tokens(p, wf, tok, cap, n_tokens)) return rc;
  const int64_t L = *n_tokens;
  if (L <= 0 || cap < L) return 0;
  DeviceGuard g(p->cfg.device);
  const int64_t nb = (L + BT - 1) / BT;
  SFKV_CUDA(cudaMemcpy(block_ids, p->pin_blk + (int64_t)wf * p->cfg.max_pin_blocks,
                       nb * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return 0;
}

static int handoff_shape_ok(const sfkv_pool* dst, const sfkv_peer* src) {
  if (!dst->kv) return fail(SFKV_EINVAL, "handoff_recv: destination pool has no KV payload");
  if (src->n_slabs != dst->cfg.n_slabs || src->slab_row_bytes != dst->cfg.slab_row_bytes)
    return fail(SFKV_EINVAL, "handoff_recv: pools have different KV shapes");
  return 0;
}

int sfkv_handoff_recv_batch(sfkv_pool* dst, const sfkv_peer* src, int64_t n, const int32_t* wf,
                            const int64_t* tok_off, const uint32_t* tok, const int32_t* src_blocks,
                            int32_t* out_status) {
  if (!dst || !src || !out_status || (n > 0 && (!wf || !tok_off || !src_blocks)))
    return fail(SFKV_EINVAL, "handoff_recv_batch: null argument");
  if (n == 0) return 0;
  if (int rc = handoff_shape_ok(dst, src)) return rc;
  if (int rc = validate_batch_host(dst, n, wf, tok_off)) return rc;
  DeviceGuard g(dst->cfg.device);
  const int64_t items = host_items(n, tok_off);
  {
    const int64_t src_n = src->block_bytes ? src->kv_bytes / src->block_bytes : 0;
    for (int64_t i = 0; i < items; ++i)
      if (src_blocks[i] < 0 || src_blocks[i] >= src_n)
        return fail(SFKV_EINVAL, "handoff_recv_batch: source block outside the peer's KV region");
  }
  int32_t* dwf;
  int64_t* doff;
  uint32_t* dtok;
  char* ex;
  const size_t o_blk = (n * sizeof(int32_t) + 255) & ~size_t(255);
  if (int rc = stage_batch(dst, n, wf, tok_off, tok, o_blk + items * sizeof(int32_t) + 16, &dwf, &doff,
                           &dtok, &ex))
    return rc;
  int32_t* dstatus = reinterpret_cast<int32_t*>(ex);
  int32_t* dblk = reinterpret_cast<int32_t*>(ex + o_blk);
  if (items > 0)
    SFKV_CUDA(cudaMemcpyAsync(dblk, src_blocks, items * sizeof(int32_t), cudaMemcpyHostToDevice, dst->stream));
  PayloadSource ps;
  ps.kv = src->kv;
  ps.blk = dblk;
  ps.block_bytes = src->block_bytes;
  ps.n_blocks = src->block_bytes ? src->kv_bytes / src->block_bytes : 0;
  if (int rc = commit_dev(dst, n, dwf, doff, dtok, items, tok_off[n], nullptr, nullptr, nullptr, dstatus, &ps))
    return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_status, dstatus, n * sizeof(int32_t), cudaMemcpyDeviceToHost, dst->stream));
  return check_sticky(dst);
}

int sfkv_handoff_recv_batch_dev(sfkv_pool* dst, const sfkv_peer* src, int64_t n, const int32_t* wf,
                                const int64_t* tok_off, const uint32_t* tok, int64_t n_tokens,
                                const int32_t* src_blocks, int32_t* out_status) {
  if (!dst || !src || !out_status || (n > 0 && (!wf || !tok_off || !tok || !src_blocks)))
    return fail(SFKV_EINVAL, "handoff_recv_batch_dev: null argument");
  if (n <= 0) return n == 0 ? 0 : fail(SFKV_EINVAL, "negative batch");
  if (n_tokens < 0) return fail(SFKV_EINVAL, "handoff_recv_batch_dev: negative n_tokens");
  if (int rc = handoff_shape_ok(dst, src)) return rc;
  DeviceGuard g(dst->cfg.device);
  PayloadSource ps;
  ps.kv = src->kv;
  ps.blk = src_blocks;
  ps.block_bytes = src->block_bytes;
  ps.n_blocks = src->block_bytes ? src->kv_bytes / src->block_bytes : 0;
  return commit_dev(dst, n, wf, tok_off, tok, n + n_tokens / BT, n_tokens, nullptr, nullptr, nullptr, out_status,
                    &ps);
}

}  // extern "C"

