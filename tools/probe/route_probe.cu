// Back-to-back timing of the routing / token-movement kernels at one chunk shape (k_route.cu
// built in; dev tool, not part of the library).  Inputs rotate over NB buffer sets so the
// gathered rows come from HBM, not L2.  Prints µs per launch and the algorithmic GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include \
//        tools/probe/route_probe.cu -o build/route_probe && build/route_probe 512 5120 16 8 1.0 2
#include "../../paper_2510_00207_b200/csrc/k_route.cu"
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <functional>

namespace fm { int g_pdl_enabled = 1; }
using namespace fm;

static float time_it(const char* name, double bytes, int iters, cudaStream_t s, const std::function<void(int)>& f) {
  for (int i = 0; i < 5; ++i) f(i);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) f(i);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const float us = ms * 1000.f / iters;
  printf("%-22s %8.2f us  %7.0f GB/s  (%s)\n", name, us, bytes / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return us;
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 512, M = argc > 2 ? atoi(argv[2]) : 5120;
  const int E = argc > 3 ? atoi(argv[3]) : 16, k = argc > 4 ? atoi(argv[4]) : 8;
  const float f = argc > 5 ? atof(argv[5]) : 1.0f;
  const int R = argc > 6 ? atoi(argv[6]) : 2;
  const int C = (int)ceil((double)f * k * T / E), ldE = R * C;
  const int NB = 3;  // buffer sets (rotate: > L2 footprint)
  printf("T_r=%d M=%d E=%d k=%d C=%d R=%d\n", T, M, E, k, C, R);
  std::vector<void*> a(NB), y(NB), dy(NB), dA(NB), dO(NB), send(NB);
  for (int b = 0; b < NB; ++b) {
    cudaMalloc(&a[b], (size_t)T * M * 2); cudaMalloc(&dO[b], (size_t)T * M * 2); cudaMalloc(&dA[b], (size_t)T * M * 2);
    cudaMalloc(&y[b], (size_t)E * ldE * M * 2); cudaMalloc(&dy[b], (size_t)E * ldE * M * 2);
    cudaMalloc(&send[b], (size_t)E * ldE * M * 2);
    cudaMemset(a[b], 0x3c, (size_t)T * M * 2); cudaMemset(dO[b], 0x3c, (size_t)T * M * 2);
    cudaMemset(y[b], 0x3c, (size_t)E * ldE * M * 2);
  }
  void* wg; cudaMalloc(&wg, (size_t)M * E * 2);
  std::vector<uint16_t> hw((size_t)M * E);
  for (size_t i = 0; i < hw.size(); ++i) hw[i] = 0x3c00 ^ (uint16_t)((i * 40503u) & 0xff);
  cudaMemcpy(wg, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  std::vector<uint16_t> ha((size_t)T * M);
  for (size_t i = 0; i < ha.size(); ++i) ha[i] = 0x3f80 ^ (uint16_t)((i * 2654435761u) & 0x7f);
  for (int b = 0; b < NB; ++b) cudaMemcpy(a[b], ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  float *logits, *w, *dw, *dl, *part, *dwg;
  int32_t *idx, *pos, *counts, *src;
  unsigned int* done;
  cudaMalloc(&logits, (size_t)T * E * 4); cudaMalloc(&w, (size_t)T * k * 4); cudaMalloc(&dw, (size_t)T * k * 4);
  cudaMalloc(&dl, (size_t)T * E * 4); cudaMalloc(&dwg, (size_t)M * E * 4);
  cudaMalloc(&part, gate_wgrad_scratch_floats(T, M, E) * 4);
  cudaMalloc(&idx, (size_t)T * k * 4); cudaMalloc(&pos, (size_t)T * k * 4);
  cudaMalloc(&counts, E * 4); cudaMalloc(&src, (size_t)E * C * 4); cudaMalloc(&done, 4);
  cudaMemset(done, 0, 4); cudaMemset(dw, 0, (size_t)T * k * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  gate_route(DT_BF16, a[0], wg, nullptr, logits, idx, w, pos, counts, src, done, T, M, E, k, C, s);
  cudaStreamSynchronize(s);
  const int it = 100;
  const double es = 2;
  time_it("gate_route", T * M * es + M * E * es + T * E * 4.0 + T * k * 20.0, it, s, [&](int i) {
    gate_route(DT_BF16, a[i % NB], wg, nullptr, logits, idx, w, pos, counts, src, done, T, M, E, k, C, s); });
  time_it("gate_topk(no scan)", T * M * es + M * E * es + T * E * 4.0 + T * k * 8.0, it, s, [&](int i) {
    gate_topk(DT_BF16, a[i % NB], wg, nullptr, logits, idx, w, T, M, E, k, s); });
  time_it("route_scan", T * k * 12.0 + E * C * 4.0, it, s, [&](int i) {
    route_scan(idx, pos, counts, src, T, E, k, C, s); });
  time_it("permute_pack", 2.0 * E * C * M * es, it, s, [&](int i) {
    permute_pack(DT_BF16, a[i % NB], src, send[i % NB], E, C, ldE, M, k, s); });
  time_it("unpermute_combine", (double)T * k * M * es + 2.0 * T * M * es, it, s, [&](int i) {
    unpermute_combine(DT_BF16, y[i % NB], idx, pos, w, a[i % NB], dA[i % NB], T, M, k, ldE, s); });
  time_it("combine_bwd_pack", (double)T * M * es + 2.0 * T * k * M * es, it, s, [&](int i) {
    combine_bwd_pack(DT_BF16, dO[i % NB], y[i % NB], idx, pos, w, src, dy[i % NB], dw, T, M, k, E, C, ldE, s); });
  time_it("gather_gate_bwd", (double)T * k * M * es + 2.0 * T * M * es + M * E * es, it, s, [&](int i) {
    gather_gate_bwd(DT_BF16, y[i % NB], idx, pos, w, dw, logits, wg, dO[i % NB], dA[i % NB], dl, T, M, E, k, ldE, s); });
  time_it("gate_wgrad", (double)T * M * es + T * E * 4.0 + M * E * 4.0, it, s, [&](int i) {
    gate_wgrad(DT_BF16, a[i % NB], dl, dwg, part, T, M, E, 0, s); });
  const int rows = R * C;  // one expert's rows over all chunks at P = 1
  time_it("colsum(db2: M cols)", (double)E * rows * M * es, it, s, [&](int i) {
    colsum_acc(DT_BF16, y[i % NB], dwg, E, rows, M, 0, s); });
  return 0;
}
