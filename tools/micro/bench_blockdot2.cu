// block-dot variants at C2 size: element pairs per step (EP) x grid multiple
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2304_04876_b200/csrc tools/micro/bench_blockdot2.cu -o /tmp/bbd2
#include <cstdio>
#include "krylov.cuh"
using namespace gdsw;
template <int NR, int EP>
void run(int grid, int64_t n, double* V, int64_t ld, int nt, double* v, double* z, double* part, double* out,
         unsigned* ctr, const char* tag) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nv = nt - 1;
  for (int w = 0; w < 3; ++w) k_block_dot<NR, EP><<<grid, KDOT_THREADS>>>(n, V, ld, nv, 0, nt, v, z, part, out, ctr, nullptr);
  cudaEventRecord(e0);
  const int R = 20;
  for (int w = 0; w < R; ++w) k_block_dot<NR, EP><<<grid, KDOT_THREADS>>>(n, V, ld, nv, 0, nt, v, z, part, out, ctr, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1000 / R, bytes = (nt + 1) * n * 8.0;
  printf("%s NR %2d EP %d grid %4d rows %2d: %7.2f us  %6.0f GB/s\n", tag, NR, EP, grid, nt, us, bytes / us / 1e3);
}
int main() {
  const int64_t n = 2097152, ld = n;
  double *V, *v, *z, *part, *out;
  unsigned* ctr;
  cudaMalloc(&V, 32 * ld * 8);
  cudaMalloc(&v, n * 8);
  cudaMalloc(&z, n * 8);
  cudaMalloc(&part, 8192 * KDOT_W2 * 8);
  cudaMalloc(&out, KDOT_W2 * 8);
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  cudaMemset(V, 0, 32 * ld * 8);
  cudaMemset(v, 0, n * 8);
  cudaMemset(z, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {2, 3, 4, 8}) {
    for (int nt : {1, 2, 3, 4}) {
      run<4, 1>(mult * sms, n, V, ld, nt, v, z, part, out, ctr, "");
      run<4, 2>(mult * sms, n, V, ld, nt, v, z, part, out, ctr, "");
    }
    for (int nt : {6, 8}) {
      run<8, 1>(mult * sms, n, V, ld, nt, v, z, part, out, ctr, "");
      run<8, 2>(mult * sms, n, V, ld, nt, v, z, part, out, ctr, "");
    }
    for (int nt : {12, 16}) {
      run<16, 1>(mult * sms / 2, n, V, ld, nt, v, z, part, out, ctr, "");
      run<16, 2>(mult * sms / 2, n, V, ld, nt, v, z, part, out, ctr, "");
    }
    for (int nt : {20, 24}) run<24, 1>(mult * sms / 2, n, V, ld, nt, v, z, part, out, ctr, "");
    for (int nt : {28, 31}) run<32, 1>(mult * sms / 2, n, V, ld, nt, v, z, part, out, ctr, "");
    for (int nt : {20, 24}) run<16, 1>(mult * sms / 2, n, V, ld, 16, v, z, part, out, ctr, "split16");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
