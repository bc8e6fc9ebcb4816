// micro-benchmark of k_block_dot per row-count bucket at C2 size
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2304_04876_b200/csrc tools/micro/bench_blockdot.cu -o /tmp/bbd
#include <cstdio>
#include <vector>
#include "krylov.cuh"
using namespace gdsw;
int main() {
  const int64_t n = 2097152, ld = n;
  double *V, *v, *z, *part, *out;
  unsigned* ctr;
  cudaMalloc(&V, 32 * ld * 8);
  cudaMalloc(&v, n * 8);
  cudaMalloc(&z, n * 8);
  cudaMalloc(&part, 4096 * KDOT_W2 * 8);
  cudaMalloc(&out, KDOT_W2 * 8);
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  cudaMemset(V, 0, 32 * ld * 8);
  cudaMemset(v, 0, n * 8);
  cudaMemset(z, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mult : {1, 2, 4}) {
    for (int nt : {2, 4, 8, 12, 16, 20, 24, 28, 31}) {
      const int nv = nt - 1;
      for (int w = 0; w < 3; ++w)
        launch_block_dot(mult * sms, 0, n, V, ld, nv, 0, nt, v, z, part, out, ctr);
      cudaEventRecord(e0);
      const int R = 20;
      for (int w = 0; w < R; ++w)
        launch_block_dot(mult * sms, 0, n, V, ld, nv, 0, nt, v, z, part, out, ctr);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1000 / R, bytes = (nt + 1) * n * 8.0;
      printf("grid %d*sms rows %2d: %7.2f us  %6.0f GB/s\n", mult, nt, us, bytes / us / 1e3);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
