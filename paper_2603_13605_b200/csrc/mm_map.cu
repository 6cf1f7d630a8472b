// K6 pressure argmin (memory manager) and K7 stage-mapper scoring.
//
// K6 replaces pressure_actions (memory.cpp:150-169): per backend whose utilization exceeds
// tau_pressure (strict), flush the idle (in_flight == 0) preserved entry with the least
// last_update_ts, ties to the lexicographically smallest workflow id (the reference scans entries
// in workflow-id order and replaces only on strict <, memory.cpp:160-161). The tracker is a
// struct-of-arrays in HBM; the lexicographic (ts, wf_rank, index) minimum per backend is one
// launch: a segmented warp-shuffle argmin per CTA and a last-CTA reduction (argmin.cuh), order-
// independent, so the victim is deterministic. 21 B per entry.
//
// K7 replaces map_threshold (mapper.cpp:19-31: light iff score <= threshold) and generalises it
// to an R x C cost argmin with reroute_on_overload (orchestrator.cpp:78-87) applied in request
// order by one warp (exact sequential semantics with a 32-request fast path).
#include <mutex>
#include <vector>

#include "argmin.cuh"
#include "pool.cuh"
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace sfkv {

struct PressArgs {
  int64_t n;
  const int32_t* backend;
  const double* ts;
  const uint32_t* rank;
  const int32_t* in_flight;
  const uint8_t* preserved;
  int32_t nb;
  const double* util;
  double tau;
  Cand* part;          // [gridDim.x][nb] CTA candidates
  unsigned int* done;  // CTAs finished (the last one reduces; it leaves the counter at 0)
  long long* victim;
};

// One launch: per backend above tau', every CTA reduces its grid-stride share of the entries to
// one (ts, rank, index) candidate with warp shuffles; the last CTA to finish reduces the CTA
// candidates into the victims. The entries of a CTA stay in L1 across the per-backend passes.
__global__ void __launch_bounds__(256) press_kernel(PressArgs a) {
  __shared__ Cand red[32];
  __shared__ bool last;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int32_t b = 0; b < a.nb; ++b) {
    Cand c = cand_none();
    if (a.util[b] > a.tau) {
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        if (a.backend[i] == b && a.preserved[i] && a.in_flight[i] <= 0) {
          const Cand d{ts_order_key(a.ts[i]), a.rank[i], i};
          if (cand_less(d, c)) c = d;
        }
      }
    }
    c = block_argmin(c, red);
    if (threadIdx.x == 0) a.part[(int64_t)blockIdx.x * a.nb + b] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int32_t b = 0; b < a.nb; ++b) {
    Cand c = cand_none();
    for (int64_t p = threadIdx.x; p < gridDim.x; p += blockDim.x) {
      const Cand d = cand_load(&a.part[p * a.nb + b]);
      if (cand_less(d, c)) c = d;
    }
    c = block_argmin(c, red);
    if (threadIdx.x == 0) a.victim[b] = c.idx;
  }
  if (threadIdx.x == 0) *a.done = 0;
}

// Single-pass variant for up to PRESS_NB_MAX backends (the common case): every entry is read
// once. A warp reduces its 32 entries segmented by backend — one warp_argmin per distinct backend
// among them (__ballot groups; a warp of one backend, as in a backend-major layout, is a single
// 5-step shuffle reduction) — into its own shared-memory row of per-backend candidates; one
// __syncthreads, then the CTA's candidates go out per backend and the last CTA reduces them with
// one warp per backend. No per-backend passes over the entries, no block-wide barrier per backend.
constexpr int PRESS_NB_MAX = 64;
constexpr int PRESS_THREADS = 256;
__global__ void __launch_bounds__(PRESS_THREADS) press1_kernel(PressArgs a) {
  __shared__ Cand s_c[PRESS_THREADS / 32][PRESS_NB_MAX];
  __shared__ unsigned char s_on[PRESS_NB_MAX];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = PRESS_THREADS / 32;
  for (int i = threadIdx.x; i < NW * PRESS_NB_MAX; i += PRESS_THREADS) s_c[i / PRESS_NB_MAX][i % PRESS_NB_MAX] = cand_none();
  for (int b = threadIdx.x; b < a.nb; b += PRESS_THREADS) s_on[b] = a.util[b] > a.tau;
  __syncthreads();
  const int64_t gw = ((int64_t)blockIdx.x * PRESS_THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * PRESS_THREADS) >> 5;
  for (int64_t base = gw * 32; base < a.n; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t b = -1;
    Cand c = cand_none();
    if (i < a.n) {
      b = a.backend[i];
      if (b >= 0 && b < a.nb && s_on[b] && a.preserved[i] && a.in_flight[i] <= 0) {
        c = Cand{ts_order_key(a.ts[i]), a.rank[i], i};
      } else {
        b = -1;
      }
    }
    unsigned rem = __ballot_sync(0xffffffffu, b >= 0);
    while (rem) {
      const int32_t bb = __shfl_sync(0xffffffffu, b, __ffs(rem) - 1);
      const unsigned grp = __ballot_sync(0xffffffffu, b == bb);
      const Cand m = warp_argmin(b == bb ? c : cand_none());
      if (lane == 0 && cand_less(m, s_c[warp][bb])) s_c[warp][bb] = m;
      rem &= ~grp;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < a.nb; b += PRESS_THREADS) {
    Cand c = s_c[0][b];
#pragma unroll
    for (int w = 1; w < NW; ++w)
      if (cand_less(s_c[w][b], c)) c = s_c[w][b];
    a.part[(int64_t)blockIdx.x * a.nb + b] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int b = warp; b < a.nb; b += NW) {
    Cand c = cand_none();
    for (int64_t p = lane; p < gridDim.x; p += 32) {
      const Cand d = cand_load(&a.part[p * a.nb + b]);
      if (cand_less(d, c)) c = d;
    }
    c = warp_argmin(c);
    if (lane == 0) a.victim[b] = c.idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) *a.done = 0;
}

int pressure_dev(cudaStream_t st, int64_t n, const int32_t* backend, const double* ts,
                 const uint32_t* rank, const int32_t* in_flight, const uint8_t* preserved,
                 int32_t nb, const double* util, double tau, Cand* part, int grid,
                 unsigned int* done, long long* victim) {
  PressArgs a{n, backend, ts, rank, in_flight, preserved, nb, util, tau, part, done, victim};
  if (nb <= PRESS_NB_MAX) {
    press1_kernel<<<grid, PRESS_THREADS, 0, st>>>(a);
    SFKV_LAUNCH_CHECK("press1_kernel");
    return 0;
  }
  press_kernel<<<grid, 256, 0, st>>>(a);
  SFKV_LAUNCH_CHECK("press_kernel");
  return 0;
}

// ---- mapper --------------------------------------------------------------------------------
__global__ void threshold_kernel(int64_t n, const double* score, double thr, int32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = score[i] <= thr ? 0 : 1;
}

struct CostArgs {
  int64_t n;
  int32_t c;
  const int64_t* P;
  const int64_t* M;
  const int64_t* O;
  const double* overhead;
  const double* prefill;
  const double* decode;
  const double* qpen;
  const int32_t* alternates;
  unsigned long long* depth;  // live depth (updated by the reroute pass)
  const unsigned long long* depth0;  // batch-start snapshot
  unsigned long long limit;
  int32_t* choice;
  double* cost;
};

// Same evaluation order as the oracle, no FMA contraction: bit-identical doubles.
__global__ void cost_kernel(CostArgs a) {
  pdl_enter();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t best = 0;
    double bc = 0;
    for (int32_t j = 0; j < a.c; ++j) {
      double x = __dadd_rn(a.overhead[j], __dmul_rn(a.prefill[j], (double)(a.P[r] - a.M[r * a.c + j])));
      x = __dadd_rn(x, __dmul_rn(a.decode[j], (double)a.O[r]));
      x = __dadd_rn(x, __dmul_rn(a.qpen[j], (double)a.depth0[j]));
      if (j == 0 || x < bc) {
        bc = x;
        best = j;
      }
    }
    a.choice[r] = best;
    a.cost[r] = bc;
  }
}

// reroute_on_overload in request order (one warp). depth lives in shared memory (c <= 1024).
// The first choices of RG chunks of 32 requests are loaded together (the pass is a sequential
// walk: without the prefetch every chunk paid a dependent global round trip).
constexpr int RG = 8;
__global__ void reroute_kernel(CostArgs a) {
  pdl_enter();
  extern __shared__ unsigned long long sdepth[];
  const int lane = threadIdx.x;
  for (int j = lane; j < a.c; j += 32) sdepth[j] = a.depth[j];
  __syncwarp();
  for (int64_t group = 0; group < a.n; group += RG * 32) {
    int32_t chs[RG];
#pragma unroll
    for (int u = 0; u < RG; ++u) {
      const int64_t r = group + u * 32 + lane;
      chs[u] = r < a.n ? a.choice[r] : -1;
    }
#pragma unroll
    for (int u = 0; u < RG; ++u) {
      const int64_t base = group + u * 32;
      if (base >= a.n) break;
      const int64_t r = base + lane;
      const bool act = r < a.n;
      const int32_t ch = chs[u];
      // fast path: no request of the chunk sees its candidate at the limit
      const unsigned peers = __match_any_sync(0xffffffffu, ch);
      const unsigned lt = (1u << lane) - 1u;
      const unsigned long long live = act ? sdepth[ch] + __popc(peers & lt) : 0;
      const bool ok = !act || a.limit == 0 || live < a.limit;
      if (__all_sync(0xffffffffu, ok)) {
        __syncwarp();
        if (act && (peers & lt) == 0) sdepth[ch] += __popc(peers);  // leader of each peer group
        __syncwarp();
      } else {
        for (int j = 0; j < 32; ++j) {
          if (base + j >= a.n) break;
          const int32_t c0 = __shfl_sync(0xffffffffu, ch, j);
          if (lane == 0) {
            int32_t pick = c0;
            if (sdepth[c0] >= a.limit && a.alternates) {
              for (int32_t t = 0; t < a.c; ++t) {
                const int32_t alt = a.alternates[c0 * a.c + t];
                if (alt < 0) break;
                if (sdepth[alt] < a.limit) {
                  pick = alt;
                  break;
                }
              }
            }
            if (pick != c0) a.choice[base + j] = pick;
            sdepth[pick] += 1;
          }
          __syncwarp();
        }
      }
    }
  }
  __syncwarp();
  for (int j = lane; j < a.c; j += 32) a.depth[j] = sdepth[j];
}

// No queue limit: nothing is rerouted, the depths just count the choices (a parallel histogram).
__global__ void depth_count_kernel(CostArgs a) {
  pdl_enter();
  extern __shared__ unsigned int scount[];
  for (int j = threadIdx.x; j < a.c; j += blockDim.x) scount[j] = 0;
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&scount[a.choice[r]], 1u);
  __syncthreads();
  for (int j = threadIdx.x; j < a.c; j += blockDim.x)
    if (scount[j]) atomicAdd(a.depth + j, (unsigned long long)scount[j]);
}

// reroute_on_overload for c <= 16 candidates, one CTA, in windows of RWIN requests. Depths only grow,
// so the saturated set S = {j : depth[j] >= limit} grows monotonically (at most c times) and a
// request's pick is a pure function of (its choice, S): the first unsaturated of (choice,
// alternates...), else the choice. A window computes every pick under the current S in parallel,
// scans the picks' one-hot counts (16-bit counters packed four to a u64 word: window counts stay
// below 2^16, so plain u64 adds never carry across counters), and finds the first request whose
// increment saturates an unsaturated candidate. Requests up to it are final; S grows and the
// window restarts after it. Windows: n / RWIN + (saturation events <= c). Alternates live in shared
// memory; each window's choices are loaded during the previous window.
template <int W>
struct PackN {
  unsigned long long w[W];
};
template <int W>
struct PackAdd {
  __device__ __forceinline__ PackN<W> operator()(const PackN<W>& x, const PackN<W>& y) const {
    PackN<W> z;
#pragma unroll
    for (int i = 0; i < W; ++i) z.w[i] = x.w[i] + y.w[i];
    return z;
  }
};
// Register-only access by a runtime candidate index (a dynamically indexed register array
// would live in local memory): select / predicated add over the W words.
template <int W>
__device__ __forceinline__ unsigned lane16(const PackN<W>& p, int j) {
  unsigned long long x = 0;
#pragma unroll
  for (int i = 0; i < W; ++i) x = (j >> 2) == i ? p.w[i] : x;
  return (unsigned)((x >> (16 * (j & 3))) & 0xffffu);
}
template <int W>
__device__ __forceinline__ void bump16(PackN<W>& p, int j) {
  const unsigned long long inc = 1ull << (16 * (j & 3));
#pragma unroll
  for (int i = 0; i < W; ++i) p.w[i] += (j >> 2) == i ? inc : 0ull;
}
constexpr int RWT = 512;         // threads of the window kernel
constexpr int RK = 8;            // consecutive requests per thread
constexpr int RWIN = RWT * RK;   // requests per window (< 2^16: 16-bit counters cannot overflow)
template <int W>  // W u64 words = 4 W candidates
__global__ void __launch_bounds__(RWT) reroute_window_kernel(CostArgs a) {
  pdl_enter();
  using P = PackN<W>;
  using BS = cub::BlockScan<P, RWT, cub::BLOCK_SCAN_WARP_SCANS>;
  using BR = cub::BlockReduce<int, RWT>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ typename BR::TempStorage rtmp;
  __shared__ unsigned long long sdepth[4 * W];
  __shared__ int32_t salt[4 * W * 4 * W];
  __shared__ unsigned ssat;
  __shared__ int s_p;
  __shared__ P s_incl;
  const int tid = threadIdx.x;
  const int c = a.c;
  if (tid < c) sdepth[tid] = a.depth[tid];
  for (int i = tid; i < c * c; i += RWT) salt[i] = a.alternates ? a.alternates[i] : -1;
  __syncthreads();
  if (tid == 0) {
    unsigned m = 0;
    for (int j = 0; j < c; ++j)
      if (sdepth[j] >= a.limit) m |= 1u << j;
    ssat = m;
  }
  __syncthreads();
  int64_t base = 0;
  int32_t cn[RK];  // this thread's choices in the next window
#pragma unroll
  for (int k = 0; k < RK; ++k) cn[k] = (int64_t)tid * RK + k < a.n ? a.choice[tid * RK + k] : 0;
  __shared__ int32_t spick[4 * W];  // pick of each first choice under the current S
  unsigned sat_done = ~0u;
  while (base < a.n) {
    const unsigned sat = ssat;
    if (sat != sat_done) {  // S changed (at most c times): rebuild the pick table
      if (tid < c) {
        int32_t pk = tid;
        if ((sat >> tid) & 1u)
          for (int32_t t = 0; t < c; ++t) {
            const int32_t alt = salt[tid * c + t];
            if (alt < 0) break;
            if (!((sat >> alt) & 1u)) {
              pk = alt;
              break;
            }
          }
        spick[tid] = pk;
      }
      __syncthreads();
      sat_done = sat;
    }
    const int64_t r0 = base + (int64_t)tid * RK;
    int32_t c0[RK], pick[RK];
    P loc;  // this thread's one-hot counts
#pragma unroll
    for (int i = 0; i < W; ++i) loc.w[i] = 0ull;
#pragma unroll
    for (int k = 0; k < RK; ++k) {
      c0[k] = cn[k];
      pick[k] = spick[c0[k]];
      if (r0 + k < a.n) bump16<W>(loc, pick[k]);
      // the following window's choice, assuming no saturation event here (else reloaded below)
      cn[k] = r0 + RWIN + k < a.n ? a.choice[r0 + RWIN + k] : 0;
    }
    P zero;
#pragma unroll
    for (int i = 0; i < W; ++i) zero.w[i] = 0ull;
    P pre, total;
    BS(tmp).ExclusiveScan(loc, pre, zero, PackAdd<W>(), total);
    int ev = RWIN;  // first request of this thread that saturates an unsaturated candidate
    {
      P run = pre;
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        if (ev == RWIN && r0 + k < a.n && !((sat >> pick[k]) & 1u) &&
            sdepth[pick[k]] + lane16<W>(run, pick[k]) + 1 >= a.limit)
          ev = tid * RK + k;
        if (r0 + k < a.n) bump16<W>(run, pick[k]);
      }
    }
    const int p = BR(rtmp).Reduce(ev, cub::Min());
    if (tid == 0) s_p = p;
    __syncthreads();
    const int pp = s_p;
#pragma unroll
    for (int k = 0; k < RK; ++k)
      if (r0 + k < a.n && tid * RK + k <= pp && pick[k] != c0[k]) a.choice[r0 + k] = pick[k];
    if (pp < RWIN && tid == pp / RK) {
      P incl = pre;
#pragma unroll
      for (int k = 0; k < RK; ++k)
        if (tid * RK + k <= pp) bump16<W>(incl, pick[k]);
      s_incl = incl;
      ssat |= 1u << pick[pp % RK];
    }
    __syncthreads();
    if (tid < c) sdepth[tid] += lane16<W>(pp < RWIN ? s_incl : total, tid);
    if (pp < RWIN) {  // the window restarts after the event: reload
      base += pp + 1;
#pragma unroll
      for (int k = 0; k < RK; ++k) {
        const int64_t r = base + (int64_t)tid * RK + k;
        cn[k] = r < a.n ? a.choice[r] : 0;
      }
    } else {
      base += RWIN;
    }
    __syncthreads();
  }
  if (tid < c) a.depth[tid] = sdepth[tid];
}

int cost_dev(cudaStream_t st, CostArgs a, int sms) {
  if (a.n > 0) {
    SFKV_CUDA(launch_pdl(cost_kernel, dim3(grid_for(a.n, 256, sms * 8)), dim3(256), st, a));
    if (a.limit == 0)
      depth_count_kernel<<<grid_for(a.n, 256, sms * 2), 256, sizeof(unsigned) * a.c, st>>>(a);
    else if (a.c <= 8)
      SFKV_CUDA(launch_pdl(reroute_window_kernel<2>, dim3(1), dim3(RWT), st, a));
    else if (a.c <= 16)
      SFKV_CUDA(launch_pdl(reroute_window_kernel<4>, dim3(1), dim3(RWT), st, a));
    else
      reroute_kernel<<<1, 32, sizeof(unsigned long long) * (a.c > 0 ? a.c : 1), st>>>(a);
  }
  SFKV_LAUNCH_CHECK("mapper kernels");
  return 0;
}

int threshold_dev(cudaStream_t st, int64_t n, const double* score, double thr, int32_t* out, int sms) {
  if (n > 0) threshold_kernel<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(n, score, thr, out);
  SFKV_LAUNCH_CHECK("threshold_kernel");
  return 0;
}

}  // namespace sfkv

// ---- pool-less entry points: per-device stream + scratch ----------------------------------
namespace sfkv {
struct DevCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  Scratch buf;
  unsigned int* done = nullptr;  // K6 last-CTA counter (zero between launches)
  int sms = 148;
};
static DevCtx* ctx_for(int dev) {
  static std::mutex gmu;
  static std::vector<DevCtx*> ctxs;
  std::lock_guard<std::mutex> lk(gmu);
  if ((int)ctxs.size() <= dev) ctxs.resize(dev + 1, nullptr);
  if (!ctxs[dev]) {
    auto* c = new DevCtx;
    cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&c->done, sizeof(unsigned int)) == cudaSuccess) cudaMemset(c->done, 0, sizeof(unsigned int));
    ctxs[dev] = c;
  }
  return ctxs[dev];
}
}  // namespace sfkv

using namespace sfkv;

extern "C" int sfmm_pressure_argmin(int32_t device, int64_t n, const int32_t* backend, const double* ts,
                                    const uint32_t* wf_rank, const int32_t* in_flight,
                                    const uint8_t* preserved, int32_t n_backends, const double* util,
                                    double tau, int64_t* out_victim) {
  if (n < 0 || n_backends < 0 || (n > 0 && (!backend || !ts || !wf_rank || !in_flight || !preserved)) ||
      (n_backends > 0 && (!util || !out_victim)))
    return fail(SFKV_EINVAL, "pressure_argmin: bad argument");
  if (n_backends == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  DevCtx* c = ctx_for(device);
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->done) return fail(SFKV_ENOMEM, "pressure_argmin: device context");
  const int grid = grid_for(n, 256, c->sms * 4);
  Carver cv;
  const size_t o_b = cv.take<int32_t>(n), o_ts = cv.take<double>(n), o_rk = cv.take<uint32_t>(n),
               o_if = cv.take<int32_t>(n), o_pr = cv.take<uint8_t>(n), o_u = cv.take<double>(n_backends),
               o_p = cv.take<Cand>((size_t)grid * n_backends), o_v = cv.take<long long>(n_backends);
  if (int rc = c->buf.ensure(cv.off)) return rc;
  char* b = c->buf.as<char>();
  cudaStream_t st = c->stream;
  if (n > 0) {
    SFKV_CUDA(cudaMemcpyAsync(b + o_b, backend, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    SFKV_CUDA(cudaMemcpyAsync(b + o_ts, ts, n * sizeof(double), cudaMemcpyHostToDevice, st));
    SFKV_CUDA(cudaMemcpyAsync(b + o_rk, wf_rank, n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    SFKV_CUDA(cudaMemcpyAsync(b + o_if, in_flight, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    SFKV_CUDA(cudaMemcpyAsync(b + o_pr, preserved, n, cudaMemcpyHostToDevice, st));
  }
  SFKV_CUDA(cudaMemcpyAsync(b + o_u, util, n_backends * sizeof(double), cudaMemcpyHostToDevice, st));
  if (int rc = pressure_dev(st, n, reinterpret_cast<int32_t*>(b + o_b), reinterpret_cast<double*>(b + o_ts),
                           reinterpret_cast<uint32_t*>(b + o_rk), reinterpret_cast<int32_t*>(b + o_if),
                           reinterpret_cast<uint8_t*>(b + o_pr), n_backends,
                           reinterpret_cast<double*>(b + o_u), tau, reinterpret_cast<Cand*>(b + o_p), grid,
                           c->done, reinterpret_cast<long long*>(b + o_v)))
    return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_victim, b + o_v, n_backends * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

/* Device pointers, asynchronous on cuda_stream (NULL = legacy default stream). */
extern "C" int sfmm_pressure_argmin_dev(int32_t device, int64_t n, const int32_t* backend, const double* ts,
                                        const uint32_t* wf_rank, const int32_t* in_flight,
                                        const uint8_t* preserved, int32_t n_backends, const double* util,
                                        double tau, int64_t* out_victim, void* cuda_stream) {
  if (n < 0 || n_backends < 0 || (n > 0 && (!backend || !ts || !wf_rank || !in_flight || !preserved)) ||
      (n_backends > 0 && (!util || !out_victim)))
    return fail(SFKV_EINVAL, "pressure_argmin_dev: bad argument");
  if (n_backends == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  DevCtx* c = ctx_for(device);
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->done) return fail(SFKV_ENOMEM, "pressure_argmin_dev: device context");
  const int grid = grid_for(n, 256, c->sms * 4);
  if (int rc = c->buf.ensure((size_t)grid * n_backends * sizeof(Cand))) return rc;
  return pressure_dev(static_cast<cudaStream_t>(cuda_stream), n, backend, ts, wf_rank, in_flight, preserved,
                      n_backends, util, tau, c->buf.as<Cand>(), grid, c->done,
                      reinterpret_cast<long long*>(out_victim));
}

extern "C" int sfmap_threshold_batch(int32_t device, int64_t n, const double* score, double threshold,
                                     int32_t* out_choice) {
  if (n < 0 || (n > 0 && (!score || !out_choice))) return fail(SFKV_EINVAL, "threshold_batch: bad argument");
  if (n == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  DevCtx* c = ctx_for(device);
  std::lock_guard<std::mutex> lk(c->mu);
  Carver cv;
  const size_t o_s = cv.take<double>(n), o_o = cv.take<int32_t>(n);
  if (int rc = c->buf.ensure(cv.off)) return rc;
  char* b = c->buf.as<char>();
  SFKV_CUDA(cudaMemcpyAsync(b + o_s, score, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (int rc = threshold_dev(c->stream, n, reinterpret_cast<double*>(b + o_s), threshold,
                            reinterpret_cast<int32_t*>(b + o_o), c->sms))
    return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_choice, b + o_o, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SFKV_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

extern "C" int sfmap_cost_batch(int32_t device, int64_t n, int32_t cc, const int64_t* P, const int64_t* M,
                                const int64_t* O, const double* overhead, const double* prefill,
                                const double* decode, const double* queue_penalty,
                                const int32_t* alternates, uint64_t* depth_inout, uint64_t limit,
                                int32_t* out_choice, double* out_cost) {
  if (n < 0 || cc <= 0 || cc > 1024 || !depth_inout || !overhead || !prefill || !decode || !queue_penalty ||
      (n > 0 && (!P || !M || !O || !out_choice || !out_cost)))
    return fail(SFKV_EINVAL, "cost_batch: bad argument");
  if (n == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  DevCtx* c = ctx_for(device);
  std::lock_guard<std::mutex> lk(c->mu);
  Carver cv;
  const size_t o_P = cv.take<int64_t>(n), o_M = cv.take<int64_t>(n * (int64_t)cc), o_O = cv.take<int64_t>(n),
               o_par = cv.take<double>(4 * (size_t)cc), o_alt = cv.take<int32_t>((size_t)cc * cc),
               o_d = cv.take<unsigned long long>(cc), o_d0 = cv.take<unsigned long long>(cc),
               o_ch = cv.take<int32_t>(n), o_co = cv.take<double>(n);
  if (int rc = c->buf.ensure(cv.off)) return rc;
  char* b = c->buf.as<char>();
  cudaStream_t st = c->stream;
  SFKV_CUDA(cudaMemcpyAsync(b + o_P, P, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_M, M, n * cc * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_O, O, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  double* par = reinterpret_cast<double*>(b + o_par);
  SFKV_CUDA(cudaMemcpyAsync(par, overhead, cc * sizeof(double), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(par + cc, prefill, cc * sizeof(double), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(par + 2 * cc, decode, cc * sizeof(double), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(par + 3 * cc, queue_penalty, cc * sizeof(double), cudaMemcpyHostToDevice, st));
  if (alternates)
    SFKV_CUDA(cudaMemcpyAsync(b + o_alt, alternates, (size_t)cc * cc * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_d, depth_inout, cc * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_d0, depth_inout, cc * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CostArgs a;
  a.n = n;
  a.c = cc;
  a.P = reinterpret_cast<int64_t*>(b + o_P);
  a.M = reinterpret_cast<int64_t*>(b + o_M);
  a.O = reinterpret_cast<int64_t*>(b + o_O);
  a.overhead = par;
  a.prefill = par + cc;
  a.decode = par + 2 * cc;
  a.qpen = par + 3 * cc;
  a.alternates = alternates ? reinterpret_cast<int32_t*>(b + o_alt) : nullptr;
  a.depth = reinterpret_cast<unsigned long long*>(b + o_d);
  a.depth0 = reinterpret_cast<unsigned long long*>(b + o_d0);
  a.limit = limit;
  a.choice = reinterpret_cast<int32_t*>(b + o_ch);
  a.cost = reinterpret_cast<double*>(b + o_co);
  if (int rc = cost_dev(st, a, c->sms)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_choice, a.choice, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(out_cost, a.cost, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(depth_inout, a.depth, cc * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// Device pointers, asynchronous on `stream` (NULL: the legacy default stream). The scoring kernel
// reads depth_inout before the reroute pass (stream-ordered after it) updates it, so the batch-start
// snapshot needs no copy.
extern "C" int sfmap_cost_batch_dev(int32_t device, int64_t n, int32_t cc, const int64_t* P, const int64_t* M,
                                    const int64_t* O, const double* overhead, const double* prefill,
                                    const double* decode, const double* queue_penalty,
                                    const int32_t* alternates, uint64_t* depth_inout, uint64_t limit,
                                    int32_t* out_choice, double* out_cost, void* stream) {
  if (n < 0 || cc <= 0 || cc > 1024 || !depth_inout || !overhead || !prefill || !decode || !queue_penalty ||
      (n > 0 && (!P || !M || !O || !out_choice || !out_cost)))
    return fail(SFKV_EINVAL, "cost_batch_dev: bad argument");
  if (n == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  CostArgs a;
  a.n = n;
  a.c = cc;
  a.P = P;
  a.M = M;
  a.O = O;
  a.overhead = overhead;
  a.prefill = prefill;
  a.decode = decode;
  a.qpen = queue_penalty;
  a.alternates = alternates;
  a.depth = reinterpret_cast<unsigned long long*>(depth_inout);
  a.depth0 = reinterpret_cast<const unsigned long long*>(depth_inout);
  a.limit = limit;
  a.choice = out_choice;
  a.cost = out_cost;
  return cost_dev(static_cast<cudaStream_t>(stream), a, ctx_for(device)->sms);
}
