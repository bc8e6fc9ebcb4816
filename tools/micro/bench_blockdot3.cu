// block-dot at C2 size: the product dispatch (launch_block_dot) against a
// row-group variant (rows split over CTAs, v/z re-read through L2) and a pure
// streaming read of the same rows (the access pattern's bound)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2304_04876_b200/csrc tools/micro/bench_blockdot3.cu -o /tmp/bbd3
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "krylov.cuh"
using namespace gdsw;

// rows [g*RG, g*RG+RG) of [V[0..nv), v] for CTA row group g = blockIdx.x % ng;
// element pairs grid-strided over the CTAs of one group
template <int RG, int EP, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bd_rg(int64_t n, const double* __restrict__ V, int64_t ldv, int nv,
                                                    int nrc, const double* __restrict__ v,
                                                    const double* __restrict__ z, double* __restrict__ partial,
                                                    double* __restrict__ out, unsigned* __restrict__ counter) {
  constexpr int NW = 8;
  __shared__ double red[NW][2 * RG];
  const int ng = (nrc + RG - 1) / RG;
  const int g = blockIdx.x % ng, cta = blockIdx.x / ng, ncta = gridDim.x / ng;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = g * RG;
  const int nr = min(RG, nrc - q0);                   // rows of this group
  const int nb = max(0, min(nr, nv - q0));            // basis rows in it
  const bool self = nv - q0 >= 0 && nv - q0 < nr;
  double av[RG], az[RG], as = 0.0, zs = 0.0;
#pragma unroll
  for (int q = 0; q < RG; ++q) av[q] = az[q] = 0.0;
  const int64_t n2 = n >> 1;
  const int64_t ld2 = ldv >> 1;
  const int64_t nth = (int64_t)ncta * 256;
  const double2* Vr = reinterpret_cast<const double2*>(V + (int64_t)q0 * ldv);
  int64_t i = (int64_t)cta * 256 + threadIdx.x;
  if (EP == 2) {
#pragma unroll 1
    for (; i + nth < n2; i += 2 * nth) {
      double2 pv[2], pz[2], x[2][RG];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t ie = i + e * nth;
        pv[e] = __ldg(reinterpret_cast<const double2*>(v) + ie);
        pz[e] = __ldg(reinterpret_cast<const double2*>(z) + ie);
#pragma unroll
        for (int u = 0; u < RG; ++u)
          if (u < nb) x[e][u] = ldg_stream(Vr + u * ld2 + ie);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int u = 0; u < RG; ++u)
          if (u < nb) {
            av[u] = fma(x[e][u].y, pv[e].y, fma(x[e][u].x, pv[e].x, av[u]));
            az[u] = fma(x[e][u].y, pz[e].y, fma(x[e][u].x, pz[e].x, az[u]));
          }
        if (self) {
          as = fma(pv[e].y, pv[e].y, fma(pv[e].x, pv[e].x, as));
          zs = fma(pv[e].y, pz[e].y, fma(pv[e].x, pz[e].x, zs));
        }
      }
    }
  }
#pragma unroll 1
  for (; i < n2; i += nth) {
    const double2 pv = __ldg(reinterpret_cast<const double2*>(v) + i);
    const double2 pz = __ldg(reinterpret_cast<const double2*>(z) + i);
    double2 x[RG];
#pragma unroll
    for (int u = 0; u < RG; ++u)
      if (u < nb) x[u] = ldg_stream(Vr + u * ld2 + i);
#pragma unroll
    for (int u = 0; u < RG; ++u)
      if (u < nb) {
        av[u] = fma(x[u].y, pv.y, fma(x[u].x, pv.x, av[u]));
        az[u] = fma(x[u].y, pz.y, fma(x[u].x, pz.x, az[u]));
      }
    if (self) {
      as = fma(pv.y, pv.y, fma(pv.x, pv.x, as));
      zs = fma(pv.y, pz.y, fma(pv.x, pz.x, zs));
    }
  }
  if (self) {
#pragma unroll
    for (int q = 0; q < RG; ++q)
      if (q == nb) {
        av[q] = as;
        az[q] = zs;
      }
  }
#pragma unroll
  for (int q = 0; q < RG; ++q) {
    if (q < nr) {
      const double a = warp_sum(av[q]);
      const double c = warp_sum(az[q]);
      if (lane == 0) {
        red[warp][2 * q] = a;
        red[warp][2 * q + 1] = c;
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * nr; k += 256) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) a += red[w][k];
    partial[(int64_t)cta * KDOT_W2 + 2 * q0 + k] = a;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = warp; k < 2 * nrc; k += NW) {
    double s = 0.0;
    for (int b = lane; b < ncta; b += 32) s += __ldcg(partial + (int64_t)b * KDOT_W2 + k);
    s = warp_sum(s);
    if (lane == 0) out[k] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// pure read of nt rows + 2 vectors (sum into one value per thread)
__global__ void __launch_bounds__(256) k_read(int64_t n, const double* __restrict__ V, int64_t ld, int nt,
                                              const double* v, const double* z, double* sink) {
  const int64_t n2 = n >> 1, ld2 = ld >> 1;
  const int64_t nth = (int64_t)gridDim.x * 256;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n2; i += nth) {
    double2 a = __ldg(reinterpret_cast<const double2*>(v) + i), b = __ldg(reinterpret_cast<const double2*>(z) + i);
    s += a.x + b.y;
#pragma unroll 4
    for (int r = 0; r < nt; ++r) {
      const double2 x = ldg_stream(reinterpret_cast<const double2*>(V) + r * ld2 + i);
      s += x.x * x.y;
    }
  }
  if (s == 12345.678) *sink = s;
}

struct Ctx {
  int64_t n, ld;
  double *V, *v, *z, *part, *out, *sink;
  unsigned* ctr;
  cudaEvent_t e0, e1;
};

template <class F>
double timeit(Ctx& c, F f) {
  for (int w = 0; w < 3; ++w) f();
  const int R = 20;
  cudaEventRecord(c.e0);
  for (int w = 0; w < R; ++w) f();
  cudaEventRecord(c.e1);
  cudaEventSynchronize(c.e1);
  float ms;
  cudaEventElapsedTime(&ms, c.e0, c.e1);
  return ms * 1000.0 / R;
}

template <int RG, int EP, int MINB>
double run_rg(Ctx& c, int nt, int ctas_per_group) {
  const int ng = (nt + RG - 1) / RG;
  const int grid = ng * ctas_per_group;
  return timeit(c, [&] {
    k_bd_rg<RG, EP, MINB><<<grid, 256>>>(c.n, c.V, c.ld, nt - 1, nt, c.v, c.z, c.part, c.out, c.ctr);
  });
}

int main(int argc, char** argv) {
  Ctx c;
  c.n = 2097152;
  c.ld = c.n + (argc > 1 ? atoll(argv[1]) : 0);
  printf("ld = n + %lld\n", (long long)(c.ld - c.n));
  cudaMalloc(&c.V, 32 * c.ld * 8);
  cudaMalloc(&c.v, c.n * 8);
  cudaMalloc(&c.z, c.n * 8);
  cudaMalloc(&c.part, 16384 * KDOT_W2 * 8);
  cudaMalloc(&c.out, KDOT_W2 * 8);
  cudaMalloc(&c.sink, 8);
  cudaMalloc(&c.ctr, 4);
  cudaMemset(c.ctr, 0, 4);
  // random-ish data so the dots are not trivially zero
  std::vector<double> h(c.n);
  for (int64_t i = 0; i < c.n; ++i) h[i] = 1.0 / (1 + (i % 97));
  for (int r = 0; r < 32; ++r) cudaMemcpy(c.V + r * c.ld, h.data(), c.n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c.v, h.data(), c.n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c.z, h.data(), c.n * 8, cudaMemcpyHostToDevice);
  cudaEventCreate(&c.e0);
  cudaEventCreate(&c.e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> ref(KDOT_W2), got(KDOT_W2);
  for (int nt : {2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 28, 31}) {
    const double bytes = (nt + 1) * c.n * 8.0;
    auto gbs = [&](double us) { return bytes / us / 1e3; };
    const double t_prod = timeit(c, [&] {
      launch_block_dot(sms, 0, c.n, c.V, c.ld, nt - 1, 0, nt, c.v, c.z, c.part, c.out, c.ctr);
    });
    cudaMemcpy(ref.data(), c.out, 2 * nt * 8, cudaMemcpyDeviceToHost);
    const double t_read = timeit(c, [&] { k_read<<<8 * sms, 256>>>(c.n, c.V, c.ld, nt - 1, c.v, c.z, c.sink); });
    printf("nt %2d  prod %7.2f us %5.0f GB/s | read %7.2f us %5.0f GB/s\n", nt, t_prod, gbs(t_prod), t_read,
           gbs(t_read));
    auto report = [&](const char* tag, int cpg, double us) {
      cudaMemcpy(got.data(), c.out, 2 * nt * 8, cudaMemcpyDeviceToHost);
      double md = 0;
      for (int k = 0; k < 2 * nt; ++k) md = std::max(md, std::fabs(got[k] - ref[k]) / std::fabs(ref[k]));
      printf("   %-14s cpg %4d: %7.2f us %5.0f GB/s  maxrel %.1e\n", tag, cpg, us, gbs(us), md);
    };
    const int ng4 = (nt + 3) / 4;
    report("rg4 b4 fit", 4 * sms / ng4, run_rg<4, 1, 4>(c, nt, 4 * sms / ng4));
    report("rg4 b4 fit2", 8 * sms / ng4, run_rg<4, 1, 4>(c, nt, 8 * sms / ng4));
    report("rg4 ep2 b2 fit", 2 * sms / ng4, run_rg<4, 2, 2>(c, nt, 2 * sms / ng4));
    const int ng2 = (nt + 1) / 2;
    report("rg2 b8 fit", 8 * sms / ng2, run_rg<2, 1, 8>(c, nt, 8 * sms / ng2));
    report("rg2 b6 fit", 6 * sms / ng2, run_rg<2, 1, 6>(c, nt, 6 * sms / ng2));
    const int ng8 = (nt + 7) / 8;
    report("rg8 b2 fit", 2 * sms / ng8, run_rg<8, 1, 2>(c, nt, 2 * sms / ng8));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
