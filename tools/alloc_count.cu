// alloc_count.cu — run-time allocation counter for librdfft.so (SURVEY §8(b) "the library allocates
// no device or host memory per call"; S:L185 zero intermediate allocation).
//
// CUPTI callback subscriber on the CUDA driver and runtime API domains: every API call made inside
// the measured window — by this program, by the static cudart inside librdfft.so, or by the library
// itself — is seen at its entry, and calls whose name belongs to an allocator (cuMemAlloc*,
// cuMemCreate, cuMemHostAlloc, cuMemAllocManaged, cuMemPool*, cuMemMap, cudaMalloc*, cudaHostAlloc,
// cudaHostRegister, ...) are counted.  All buffers are allocated BEFORE the window opens.
//
// Window "cold": the very first call of every entry point (kernel attributes, occupancy queries,
// lazy module loading of each kernel happen here).  Window "warm": the same calls repeated.
//
// Usage: alloc_count <path to librdfft.so>   -> one JSON line on stdout, exit 0 iff no allocation.
// Built and run by tests/test_gpu_alloc.py; test infrastructure, not part of the product path.
#include <cuda_runtime.h>
#include <cupti.h>
#include <dlfcn.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

namespace {
std::atomic<long> g_calls{0}, g_allocs{0};
std::mutex g_mu;
std::set<std::string> g_alloc_names, g_all_names;
bool g_on = false;

bool is_alloc(const char* f) {
  static const char* pats[] = {"Alloc", "alloc", "cuMemCreate", "cuMemMap", "HostRegister", "MemPool", "cuMemGetHandle",
                               "Malloc", "cuMemImport", "cuArrayCreate", "cuArray3DCreate", "cuMipmappedArrayCreate"};
  for (const char* p : pats)
    if (std::strstr(f, p)) return true;
  return false;
}

void CUPTIAPI on_api(void*, CUpti_CallbackDomain, CUpti_CallbackId, const void* data) {
  const auto* info = static_cast<const CUpti_CallbackData*>(data);
  if (!g_on || info->callbackSite != CUPTI_API_ENTER || !info->functionName) return;
  g_calls++;
  std::lock_guard<std::mutex> lk(g_mu);
  g_all_names.insert(info->functionName);
  if (is_alloc(info->functionName)) {
    g_allocs++;
    g_alloc_names.insert(info->functionName);
  }
}

#define CK(x)                                                                     \
  do {                                                                            \
    auto e_ = (x);                                                                \
    if (e_) {                                                                     \
      std::fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)e_); \
      std::exit(2);                                                               \
    }                                                                             \
  } while (0)

using fwd_t = int (*)(void*, int64_t, int64_t, int, void*);
using mul_t = int (*)(void*, const void*, int64_t, int64_t, int64_t, int, void*);
using bfwd_t = int (*)(const void*, const void*, void*, int64_t, int64_t, int64_t, int64_t, int, void*);
using bbwd_t = int (*)(const void*, const void*, const void*, void*, float*, int64_t, int64_t, int64_t, int64_t, int,
                       void*);
using sfwd_t = int (*)(const void*, const float*, void*, int64_t, int64_t, int64_t, int64_t, int, int, void*);
using sbwd_t = int (*)(const void*, const float*, const void*, void*, float*, int64_t, int64_t, int64_t, int64_t, int,
                       int, void*);
using dec_t = int (*)(const void*, void*, int64_t, int64_t, int, void*);
using conj_t = int (*)(void*, int64_t, int64_t, int, void*);
using axpy_t = int (*)(void*, const void*, float, int64_t, int64_t, int64_t, int, void*);
using host_t = int (*)(void*, int64_t, int64_t, int, const void*, int, void*, int64_t, void*, void*);

template <typename F>
F sym(void* h, const char* name) {
  void* p = dlsym(h, name);
  if (!p) {
    std::fprintf(stderr, "missing symbol %s\n", name);
    std::exit(2);
  }
  return reinterpret_cast<F>(p);
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s librdfft.so\n", argv[0]);
    return 2;
  }
  CK(cudaSetDevice(0));
  CK(cudaFree(nullptr));
  void* h = dlopen(argv[1], RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    std::fprintf(stderr, "dlopen: %s\n", dlerror());
    return 2;
  }
  auto fwd = sym<fwd_t>(h, "rdfft_fwd");
  auto inv = sym<fwd_t>(h, "rdfft_inv");
  auto mul = sym<mul_t>(h, "rdfft_packed_mul");
  auto cmul = sym<mul_t>(h, "rdfft_packed_conjmul");
  auto bf = sym<bfwd_t>(h, "bca_fwd");
  auto bfa = sym<bfwd_t>(h, "bca_fwd_accum");
  auto bb = sym<bbwd_t>(h, "bca_bwd");
  auto bba = sym<bbwd_t>(h, "bca_bwd_accum");
  auto sf = sym<sfwd_t>(h, "bca_fwd_spectral");
  auto sb = sym<sbwd_t>(h, "bca_bwd_spectral");
  auto dec = sym<dec_t>(h, "rdfft_decode");
  auto enc = sym<dec_t>(h, "rdfft_encode");
  auto cj = sym<conj_t>(h, "rdfft_packed_conj");
  auto ax = sym<axpy_t>(h, "rdfft_packed_axpy");
  auto fh = sym<host_t>(h, "rdfft_filter_host");

  // ---- every buffer before the window (zero-filled: the values do not matter here)
  const size_t big = (size_t)64 << 20;  // bytes
  void *a, *b, *c, *xb, *yb, *gb, *dxb, *wb, *work, *hostp;
  float *dw, *W;
  CK(cudaMalloc(&a, big));
  CK(cudaMalloc(&b, big));
  CK(cudaMalloc(&c, big + (1 << 20)));
  CK(cudaMalloc(&xb, big));
  CK(cudaMalloc(&yb, big));
  CK(cudaMalloc(&gb, big));
  CK(cudaMalloc(&dxb, big));
  CK(cudaMalloc(&wb, 1 << 20));
  CK(cudaMalloc(&dw, 1 << 20));
  CK(cudaMalloc(&W, 1 << 20));
  CK(cudaMalloc(&work, 8 << 20));
  CK(cudaMallocHost(&hostp, 4 << 20));
  for (void* p : {a, b, c, xb, yb, gb, dxb}) CK(cudaMemset(p, 0, big));
  CK(cudaMemset(wb, 0, 1 << 20));
  CK(cudaMemset(W, 0, 1 << 20));
  std::memset(hostp, 0, 4 << 20);
  cudaStream_t s0, s1;
  CK(cudaStreamCreate(&s0));
  CK(cudaStreamCreate(&s1));
  CK(cudaDeviceSynchronize());

  CUpti_SubscriberHandle sub;
  CK(cuptiSubscribe(&sub, (CUpti_CallbackFunc)on_api, nullptr));
  CK(cuptiEnableDomain(1, sub, CUPTI_CB_DOMAIN_DRIVER_API));
  CK(cuptiEnableDomain(1, sub, CUPTI_CB_DOMAIN_RUNTIME_API));

  int bad = 0;
  auto run_all = [&]() {
    for (int dt = 0; dt < 2; ++dt) {
      for (int64_t n = 2; n <= 65536; n *= 2) {
        const int64_t batch = n >= 8192 ? 7 : 257;
        bad |= fwd(a, batch, n, dt, s0);
        bad |= mul(a, b, batch, n, 1, dt, s0);
        bad |= cmul(a, b, batch, n, batch, dt, s0);
        bad |= inv(a, batch, n, dt, s0);
        if (n <= 4096) {
          bad |= dec(a, c, batch, n, dt, s0);
          bad |= enc(c, a, batch, n, dt, s0);
        }
        bad |= cj(a, batch, n, dt, s0);
        bad |= ax(a, b, -0.5f, batch, n, 1, dt, s0);
      }
      // BCA: every kernel family (fused p = 256 / 512 / 1024 / 2048 / 4096, resident spectra, tiled)
      const int64_t shapes[][4] = {{256, 3, 3, 67},  {512, 4, 4, 33}, {1024, 4, 4, 33}, {1024, 3, 3, 19},
                                   {2048, 2, 2, 9},  {4096, 1, 1, 9}, {128, 3, 2, 21},  {256, 16, 16, 5}};
      for (const auto& sh : shapes) {
        const int64_t p = sh[0], qo = sh[1], qi = sh[2], T = sh[3];
        bad |= bf(xb, wb, yb, T, qi * p, qo * p, p, dt, s0);
        bad |= bfa(xb, wb, yb, T, qi * p, qo * p, p, dt, s0);
        bad |= bb(xb, wb, gb, dxb, dw, T, qi * p, qo * p, p, dt, s0);
        bad |= bba(xb, wb, gb, dxb, dw, T, qi * p, qo * p, p, dt, s0);
        if (qi == qo) bad |= bb(xb, wb, gb, gb, dw, T, qi * p, qo * p, p, dt, s0);  // dx over g
        bad |= sf(xb, W, yb, T, qi * p, qo * p, p, dt, 0, s0);
        bad |= sb(xb, W, gb, dxb, dw, T, qi * p, qo * p, p, dt, 1, s0);
      }
      bad |= fh(hostp, 512, 1024, dt, b, 0, work, 64, s0, s1);
    }
    CK(cudaDeviceSynchronize());
  };

  g_on = true;
  run_all();
  g_on = false;
  const long cold_calls = g_calls.exchange(0), cold_allocs = g_allocs.exchange(0);
  std::set<std::string> cold_names;
  std::swap(cold_names, g_alloc_names);
  g_on = true;
  for (int r = 0; r < 3; ++r) run_all();
  g_on = false;
  const long warm_calls = g_calls.load(), warm_allocs = g_allocs.load();
  CK(cuptiUnsubscribe(sub));

  auto names = [](const std::set<std::string>& s) {
    std::string o = "[";
    for (const auto& n : s) o += (o.size() > 1 ? ", \"" : "\"") + n + "\"";
    return o + "]";
  };
  std::printf(
      "{\"cold_api_calls\": %ld, \"cold_allocs\": %ld, \"cold_alloc_names\": %s, \"warm_api_calls\": %ld, "
      "\"warm_allocs\": %ld, \"warm_alloc_names\": %s, \"status_or\": %d, \"api_names\": %s}\n",
      cold_calls, cold_allocs, names(cold_names).c_str(), warm_calls, warm_allocs, names(g_alloc_names).c_str(), bad,
      names(g_all_names).c_str());
  return (cold_allocs || warm_allocs || bad) ? 1 : 0;
}
