// Link stub for the reference's HttpBackend (oracle test infrastructure only).
//
// The reference's src/http_backend.cpp needs cpp-httplib, which is not in this
// image. src/config.cpp:170-184 (build_registry) references HttpBackend, so the
// oracle build links this stub instead. Every config the oracle replays uses
// simulated backends only; constructing an HttpBackend through this stub throws.
#include "stageflow/http_backend.hpp"

namespace stageflow {

struct HttpBackend::Pool {};

HttpBackend::HttpBackend(EventLoop& loop, BackendDescriptor descriptor, HttpBackendConfig config,
                         LogFn log)
    : loop_(loop), descriptor_(std::move(descriptor)), config_(config), log_(std::move(log)) {
  throw BackendError("oracle build: HttpBackend is stubbed (cpp-httplib absent)");
}
HttpBackend::~HttpBackend() = default;
bool HttpBackend::has_capacity() const { return false; }
void HttpBackend::complete(CompletionRequest, CompletionCallback) {
  throw BackendError("oracle build: HttpBackend is stubbed");
}
long long HttpBackend::flush(const FlushScope&) { return 0; }
double HttpBackend::cache_utilization() const { return 0.0; }
bool HttpBackend::preserve(const std::string&) { return false; }

}  // namespace stageflow
