// Common device/host utilities for libgdsw (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace gdsw {

// ---------------------------------------------------------------------------
// error plumbing: every C entry point converts exceptions into a status code
// and a thread-local message (include/gdsw.h: GDSW_E*)
// ---------------------------------------------------------------------------
enum Status : int {
  OK = 0,
  E_VALUE = 1,   // ValueError
  E_LINALG = 2,  // numpy.linalg.LinAlgError
  E_FLOAT = 3,   // FloatingPointError
  E_ARITH = 4,   // ArithmeticError
  E_CUDA = 5,    // RuntimeError (driver / launch)
  E_TYPE = 6,    // TypeError
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::gdsw::cuda_check((x), #x)
// every kernel launch site is followed by CK_LAUNCH(): it checks the launch
// and counts it (gdsw_launch_count, reported as gpu_launches by bench.py)
inline std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}
#define CK_LAUNCH()                                                   \
  do {                                                                \
    ::gdsw::cuda_check(cudaGetLastError(), "kernel launch");          \
    ::gdsw::launch_counter().fetch_add(1, std::memory_order_relaxed); \
  } while (0)

inline void require(bool ok, const std::string& msg, int code = E_VALUE) {
  if (!ok) throw Error(code, msg);
}

// ---------------------------------------------------------------------------
// owning device buffer
// ---------------------------------------------------------------------------
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) CK(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* host, size_t count) {
    alloc(count);
    if (count) CK(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
  void zero(cudaStream_t s = 0) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  std::vector<T> download() const {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// narrow a host int64 array to int32 with a range check
inline std::vector<int32_t> to_i32(const int64_t* a, size_t n, int64_t add = 0) {
  std::vector<int32_t> out(n);
  for (size_t i = 0; i < n; ++i) {
    int64_t v = a[i] + add;
    require(v >= INT32_MIN && v <= INT32_MAX, "index exceeds the int32 device layout");
    out[i] = (int32_t)v;
  }
  return out;
}

inline int num_sms() {
  static int sms = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

inline unsigned grid_for(int64_t work, int block, int64_t cap = 1 << 30) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---------------------------------------------------------------------------
// IEEE round-to-nearest arithmetic without FMA contraction. The reference's
// numba loops (_kernels.py:12-16, no fastmath) round every product and sum
// separately; using these keeps the sequential kernels bit-identical.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float rn_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rn_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rn_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float rn_div(float a, float b) { return __fdiv_rn(a, b); }

// read-only streaming load (values/indices are read once per pass)
template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) { return __ldcs(p); }

// L2 evict_last hints (createpolicy + ld/st .L2::cache_hint): for the
// small iterate vectors that successive sweeps re-read while the factor
// values stream through with evict_first
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_last(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_last(const float* a, uint64_t pol) {
  float v;
  asm("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_last(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_last(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy primitives (sm_90+ PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace gdsw
