// Phase probe of the fused gate + routing-scan kernel at c2/c3/c4 chunk shapes
// (k_route.cu built with -DFM_PROBE).  Dev tool, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFM_PROBE -I include \
//        tools/probe/gate_probe.cu -o build/gate_probe
#include "../../paper_2510_00207_b200/csrc/k_route.cu"
#include <cstdio>
#include <vector>

namespace fm { int g_pdl_enabled = 1; }
using namespace fm;

static void run(const char* name, int T, int M, int E, int k, int C) {
  void *a, *wg;
  float *logits, *w;
  int32_t *idx, *pos, *counts, *src;
  unsigned int* done;
  cudaMalloc(&a, (size_t)T * M * 2); cudaMalloc(&wg, (size_t)M * E * 2);
  cudaMalloc(&logits, (size_t)T * E * 4); cudaMalloc(&w, (size_t)T * k * 4);
  cudaMalloc(&idx, (size_t)T * k * 4); cudaMalloc(&pos, (size_t)T * k * 4);
  cudaMalloc(&counts, E * 4); cudaMalloc(&src, (size_t)E * C * 4); cudaMalloc(&done, 4);
  cudaMemset(done, 0, 4);
  std::vector<uint16_t> h((size_t)T * M);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0x3f80 ^ (uint16_t)((i * 2654435761u) & 0x7f);
  cudaMemcpy(a, h.data(), (size_t)T * M * 2, cudaMemcpyHostToDevice);
  std::vector<uint16_t> hw((size_t)M * E);
  for (size_t i = 0; i < hw.size(); ++i) hw[i] = 0x3c00 ^ (uint16_t)((i * 40503u) & 0xff);
  cudaMemcpy(wg, hw.data(), (size_t)M * E * 2, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 20; ++i) gate_route(DT_BF16, a, wg, nullptr, logits, idx, w, pos, counts, src, done, T, M, E, k, C, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 200; ++i) gate_route(DT_BF16, a, wg, nullptr, logits, idx, w, pos, counts, src, done, T, M, E, k, C, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  gate_route(DT_BF16, a, wg, nullptr, logits, idx, w, pos, counts, src, done, T, M, E, k, C, s);
  cudaStreamSynchronize(s);
  long long g[24];
  cudaMemcpyFromSymbol(g, g_gprobe, sizeof(g));
  printf("  topk phase: sync %lld logits %lld select %lld\n", g[16] - g[0], g[17] - g[0], g[18] - g[0]);
  printf("%-6s T=%d M=%d E=%d: back-to-back %.2f us | cta0: pdl %lld gemv %lld part %lld cs1 %lld cs2 %lld topk %lld fence %lld ticket %lld | scan cta: init %lld pass1 %lld scan %lld pass2 %lld (%s)\n",
         name, T, M, E, ms * 1000.f / 200, g[1] - g[0], g[2] - g[0], g[4] - g[0], g[5] - g[0], g[6] - g[0], g[7] - g[0], g[13] - g[0], g[3] - g[0], g[9] - g[8],
         g[10] - g[9], g[11] - g[10], g[12] - g[11], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run("c2", 256, 256, 8, 2, 64);
  g_gate_force_ks = 1;
  run("c2ks1", 256, 256, 8, 2, 64);
  g_gate_force_ks = 2;
  run("c2ks2", 256, 256, 8, 2, 64);
  g_gate_force_ks = 0;
  run("c3", 1024, 1024, 16, 2, 128);
  g_gate_force_ks = 2;
  run("c3ks2", 1024, 1024, 16, 2, 128);
  g_gate_force_ks = 0;
  run("c4", 1024, 4096, 16, 2, 128);
  run("dsv2s", 512, 5120, 16, 8, 256);
  return 0;
}
