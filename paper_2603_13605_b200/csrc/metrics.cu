// §8f-3: batched latency model and TTFT percentiles.
//
// Replaces the per-request timing arithmetic of SimulatedBackend::start (simulated_backend.cpp:
// 99-112) and MetricsReport's nearest-rank percentiles (metrics.cpp:22-28, 57-67):
//   prefill = overhead + prefill_ms_per_token * (P - M)        (double, in this order)
//   decode  = decode_ms_per_token * O
//   ttft    = queue + prefill;   total = ttft + decode;   service delay = prefill + decode
// evaluated with __dadd_rn / __dmul_rn (no FMA contraction), so every double equals the
// reference's bit for bit. Percentiles: the samples are radix-sorted on the device and
// percentile p is sorted[max(1, ceil(p / 100 * n)) - 1], the reference's rank rule.
#include <cub/device/device_radix_sort.cuh>
#include <mutex>
#include <vector>

#include "pool.cuh"

namespace sfkv {

struct LatArgs {
  int64_t n;
  const int32_t* backend;
  const double* queue;
  const int64_t* P;
  const int64_t* M;
  const int64_t* O;
  const double* overhead;
  const double* prefill;
  const double* decode;
  double* ttft;
  double* total;
  double* service;
};

// One thread per request (no grid-stride loop: every request's loads are in flight at once; the
// per-backend parameters are a dependent gather of a few cached lines).
__global__ void __launch_bounds__(256) latency_kernel(LatArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < a.n) {
    const int32_t b = __ldg(a.backend + r);
    const double q = __ldg(a.queue + r);
    const int64_t P = __ldg(a.P + r), M = __ldg(a.M + r), O = __ldg(a.O + r);
    const double pf = __dadd_rn(__ldg(a.overhead + b), __dmul_rn(__ldg(a.prefill + b), (double)(P - M)));
    const double dc = __dmul_rn(__ldg(a.decode + b), (double)O);
    const double t = __dadd_rn(q, pf);
    a.ttft[r] = t;
    if (a.total) a.total[r] = __dadd_rn(t, dc);
    if (a.service) a.service[r] = __dadd_rn(pf, dc);
  }
}

__global__ void nearest_rank_kernel(const double* sorted, int64_t n, int32_t k, const int32_t* pct, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  // ceil(p / 100 * n) in double, exactly as std::ceil(static_cast<double>(pct) / 100.0 * n)
  int64_t rank = (int64_t)ceil(__dmul_rn(__ddiv_rn((double)pct[i], 100.0), (double)n));
  if (rank < 1) rank = 1;
  if (rank > n) rank = n;
  out[i] = sorted[rank - 1];
}

}  // namespace sfkv

namespace sfkv {
// Host-pointer entry points: a per-device scratch buffer and stream reused across calls (a
// cudaMalloc / cudaFree pair per call cost milliseconds: cudaFree synchronizes the device).
struct MetCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  Scratch buf;
};
static MetCtx* met_ctx(int dev) {
  static std::mutex gmu;
  static std::vector<MetCtx*> ctxs;
  std::lock_guard<std::mutex> lk(gmu);
  if ((int)ctxs.size() <= dev) ctxs.resize(dev + 1, nullptr);
  if (!ctxs[dev]) {
    auto* c = new MetCtx;
    cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    ctxs[dev] = c;
  }
  return ctxs[dev];
}
}  // namespace sfkv

using namespace sfkv;

extern "C" {

int sfmet_latency_batch_dev(int32_t device, int64_t n, const int32_t* backend, const double* queue_ms,
                            const int64_t* P, const int64_t* M, const int64_t* O, const double* overhead,
                            const double* prefill, const double* decode, double* out_ttft, double* out_total,
                            double* out_service, void* stream) {
  if (n < 0 || (n > 0 && (!backend || !queue_ms || !P || !M || !O || !overhead || !prefill || !decode || !out_ttft)))
    return fail(SFKV_EINVAL, "latency_batch_dev: bad argument");
  if (n == 0) return 0;
  if (n > (int64_t)INT32_MAX * 256) return fail(SFKV_EINVAL, "latency_batch_dev: too many requests");
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  LatArgs a{n, backend, queue_ms, P, M, O, overhead, prefill, decode, out_ttft, out_total, out_service};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  latency_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
  SFKV_LAUNCH_CHECK("latency_kernel");
  return 0;
}

int sfmet_latency_batch(int32_t device, int64_t n, const int32_t* backend, const double* queue_ms, const int64_t* P,
                        const int64_t* M, const int64_t* O, int32_t n_backends, const double* overhead,
                        const double* prefill, const double* decode, double* out_ttft, double* out_total,
                        double* out_service) {
  if (n < 0 || n_backends <= 0 || (n > 0 && (!backend || !queue_ms || !P || !M || !O || !overhead || !prefill ||
                                            !decode || !out_ttft)))
    return fail(SFKV_EINVAL, "latency_batch: bad argument");
  for (int64_t r = 0; r < n; ++r)
    if (backend[r] < 0 || backend[r] >= n_backends) return fail(SFKV_EINVAL, "latency_batch: backend out of range");
  if (n == 0) return 0;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  Carver cv;
  const size_t o_b = cv.take<int32_t>(n), o_q = cv.take<double>(n), o_p = cv.take<int64_t>(n),
               o_m = cv.take<int64_t>(n), o_o = cv.take<int64_t>(n), o_oh = cv.take<double>(n_backends),
               o_pf = cv.take<double>(n_backends), o_dc = cv.take<double>(n_backends), o_t = cv.take<double>(n),
               o_tt = cv.take<double>(n), o_sv = cv.take<double>(n);
  MetCtx* mc = met_ctx(device);
  std::lock_guard<std::mutex> lk(mc->mu);
  if (int rc = mc->buf.ensure(cv.off)) return rc;
  char* d = mc->buf.as<char>();
  cudaStream_t st = mc->stream;
  auto up = [&](size_t off, const void* src, size_t bytes) {
    return cudaMemcpyAsync(d + off, src, bytes, cudaMemcpyHostToDevice, st);
  };
  cudaError_t e = cudaSuccess;
  if ((e = up(o_b, backend, n * 4)) != cudaSuccess || (e = up(o_q, queue_ms, n * 8)) != cudaSuccess ||
      (e = up(o_p, P, n * 8)) != cudaSuccess || (e = up(o_m, M, n * 8)) != cudaSuccess ||
      (e = up(o_o, O, n * 8)) != cudaSuccess || (e = up(o_oh, overhead, n_backends * 8)) != cudaSuccess ||
      (e = up(o_pf, prefill, n_backends * 8)) != cudaSuccess || (e = up(o_dc, decode, n_backends * 8)) != cudaSuccess) {
    return cuda_fail(e, "latency_batch H2D");
  }
  int rc = sfmet_latency_batch_dev(device, n, reinterpret_cast<int32_t*>(d + o_b), reinterpret_cast<double*>(d + o_q),
                                   reinterpret_cast<int64_t*>(d + o_p), reinterpret_cast<int64_t*>(d + o_m),
                                   reinterpret_cast<int64_t*>(d + o_o), reinterpret_cast<double*>(d + o_oh),
                                   reinterpret_cast<double*>(d + o_pf), reinterpret_cast<double*>(d + o_dc),
                                   reinterpret_cast<double*>(d + o_t), out_total ? reinterpret_cast<double*>(d + o_tt) : nullptr,
                                   out_service ? reinterpret_cast<double*>(d + o_sv) : nullptr, st);
  if (!rc) {
    if ((e = cudaMemcpyAsync(out_ttft, d + o_t, n * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (out_total && (e = cudaMemcpyAsync(out_total, d + o_tt, n * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) ||
        (out_service && (e = cudaMemcpyAsync(out_service, d + o_sv, n * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      rc = cuda_fail(e, "latency_batch D2H");
  }
  return rc;
}

// Nearest-rank percentiles of n samples (metrics.cpp:22-28): out[i] = sorted[max(1, ceil(pct[i]/100 n)) - 1].
int sfmet_nearest_rank(int32_t device, int64_t n, const double* samples, int32_t k, const int32_t* pct, double* out) {
  if (n <= 0) return fail(SFKV_EINVAL, "nearest_rank: no samples");  // the reference throws
  if (!samples || k < 0 || (k > 0 && (!pct || !out))) return fail(SFKV_EINVAL, "nearest_rank: bad argument");
  if (n > INT32_MAX) return fail(SFKV_EINVAL, "nearest_rank: too many samples");
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  Carver cv;
  const size_t o_in = cv.take<double>(n), o_out = cv.take<double>(n), o_p = cv.take<int32_t>(k + 1),
               o_r = cv.take<double>(k + 1), o_tmp = cv.take<char>(tmp_bytes);
  MetCtx* mc = met_ctx(device);
  std::lock_guard<std::mutex> lk(mc->mu);
  if (int rc = mc->buf.ensure(cv.off)) return rc;
  char* d = mc->buf.as<char>();
  cudaStream_t st = mc->stream;
  cudaError_t e = cudaMemcpyAsync(d + o_in, samples, n * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && k) e = cudaMemcpyAsync(d + o_p, pct, k * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortKeys(d + o_tmp, tmp_bytes, reinterpret_cast<const double*>(d + o_in),
                                       reinterpret_cast<double*>(d + o_out), (int)n, 0, 64, st);
  if (e == cudaSuccess && k) {
    nearest_rank_kernel<<<(k + 127) / 128, 128, 0, st>>>(reinterpret_cast<double*>(d + o_out), n, k,
                                                         reinterpret_cast<int32_t*>(d + o_p),
                                                         reinterpret_cast<double*>(d + o_r));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && k) e = cudaMemcpyAsync(out, d + o_r, k * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "nearest_rank");
  return 0;
}

}  // extern "C"
