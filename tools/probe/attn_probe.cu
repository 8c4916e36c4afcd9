// Back-to-back timing of the tcgen05 attention forward/backward at the c2/c3/c4 chunk
// shapes (dev tool, not part of the library).  Build: tools/probe/build_attn_probe.sh
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2510_00207_b200/csrc/kernels.h"

using namespace fm;

static void run(const char* name, int nseq, int N, int M, int H) {
  const size_t T = (size_t)nseq * N;
  void *qkv, *ctx, *dctx, *dqkv;
  float *lse, *D;
  cudaMalloc(&qkv, T * 3 * M * 2); cudaMalloc(&ctx, T * M * 2); cudaMalloc(&dctx, T * M * 2);
  cudaMalloc(&dqkv, T * 3 * M * 2); cudaMalloc(&lse, T * H * 4); cudaMalloc(&D, T * H * 4);
  std::vector<uint16_t> h(T * 3 * M);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0x3c00 ^ (uint16_t)((i * 2654435761u >> 7) & 0x3ff);
  cudaMemcpy(qkv, h.data(), T * 3 * M * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dctx, h.data(), T * M * 2, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms[2];
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < 10; ++i) {
      if (pass == 0) attn_fwd_tc(qkv, ctx, lse, nseq, N, 0, N, M, H, 1, s);
      else attn_bwd_tc(qkv, ctx, lse, dctx, dqkv, D, nseq, N, 0, N, M, H, 1, s);
    }
    cudaEventRecord(e0, s);
    for (int i = 0; i < 100; ++i) {
      if (pass == 0) attn_fwd_tc(qkv, ctx, lse, nseq, N, 0, N, M, H, 1, s);
      else attn_bwd_tc(qkv, ctx, lse, dctx, dqkv, D, nseq, N, 0, N, M, H, 1, s);
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms[pass], e0, e1);
  }
  // isolated launches (synchronised on both sides: no overlap with a neighbour launch)
  float iso[2] = {0.f, 0.f};
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < 20; ++i) {
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      if (pass == 0) attn_fwd_tc(qkv, ctx, lse, nseq, N, 0, N, M, H, 1, s);
      else attn_bwd_tc(qkv, ctx, lse, dctx, dqkv, D, nseq, N, 0, N, M, H, 1, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      iso[pass] += t * 1000.f / 20;
    }
  printf("%-4s nseq=%d N=%d M=%d H=%d: back-to-back fwd %.2f us  bwd %.2f us | isolated fwd %.2f us  bwd %.2f us (%s)\n",
         name, nseq, N, M, H, ms[0] * 10.f, ms[1] * 10.f, iso[0], iso[1], cudaGetErrorString(cudaGetLastError()));
  cudaFree(qkv); cudaFree(ctx); cudaFree(dctx); cudaFree(dqkv); cudaFree(lse); cudaFree(D);
}

int main() {
  run("c2", 1, 256, 256, 4);
  run("c3", 2, 512, 1024, 16);
  run("c4", 2, 512, 4096, 32);
  run("c3x4", 4, 512, 1024, 16);
  return 0;
}
