// Phase probe of the tcgen05 GEMM at small (latency-bound) shapes: builds
// k_gemm_tc.cu with FM_PROBE so CTA 0 stamps clock64() at its phase boundaries,
// and times back-to-back launches with CUDA events.  Dev tool, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFM_PROBE -I include \
//        tools/probe/gemm_probe.cu paper_2510_00207_b200/csrc/k_gemm_simt.cu -lcuda -o build/gemm_probe
#include "../../paper_2510_00207_b200/csrc/k_gemm_tc.cu"
#include <vector>

namespace fm { int g_pdl_enabled = 1; }
using namespace fm;

static int g_variant = 0;  // 1: BN=256, 3 stages, 2 staging buffers per epilogue warp
static int call(const GemmArgs& g, cudaStream_t s) { return g_variant ? launch_tc<256, 3, 2>(g, s) : gemm_tc(g, s); }

static void run(const char* name, int M, int N, int K, int batch, int epi, int dbg = 0, int bn = 0) {
  g_tc_debug = dbg;
  gemm_tc_force_bn(bn);
  void *A, *B, *C, *Z;
  cudaMalloc(&A, (size_t)batch * M * K * 2); cudaMalloc(&B, (size_t)batch * K * N * 2);
  cudaMalloc(&C, (size_t)batch * M * N * 4); cudaMalloc(&Z, (size_t)batch * M * N * 2);
  cudaMemset(A, 0, (size_t)batch * M * K * 2); cudaMemset(B, 0, (size_t)batch * K * N * 2);
  cudaMemset(Z, 0, (size_t)batch * M * N * 2);
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.lda = K; g.sA = (int64_t)M * K;
  g.B = B; g.ldb = N; g.sB = (int64_t)K * N;
  g.C = C; g.ldc = N; g.sC = (int64_t)M * N;
  g.epi = epi;
  if (epi == EPI_DGELU || epi == EPI_BIAS_GELU || epi == EPI_BIAS_GELU_G || epi == EPI_MUL_AUX) {
    g.aux = Z; g.ldaux = N; g.sAux = (int64_t)M * N;
  }
  if (epi == EPI_BIAS_GELU || epi == EPI_BIAS_GELU_G) { g.bias = Z; g.sBias = N; }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 20; ++i) call(g, s);
  cudaStreamSynchronize(s);
  long long h[32] = {};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = (int64_t)M * N * batch > (1 << 26) ? 10 : 200;
  cudaEventRecord(e0, s);
  for (int i = 0; i < reps; ++i) call(g, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  // single isolated launch
  cudaEventRecord(e0, s);
  call(g, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms1 = 0.f;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaMemcpyFromSymbol(h, g_probe, sizeof(h));  // stamps of the isolated launch
  { long long z[32] = {}; cudaMemcpyToSymbol(g_probe, z, sizeof(z)); }
  printf("%-10s M=%d N=%d K=%d b=%d epi=%d  back-to-back %.2f us/launch  isolated %.2f us | cycles from entry:",
         name, M, N, K, batch, epi, ms * 1000.f / reps, ms1 * 1000.f);
  const char* lab[9] = {"entry", "synced", "pdl", "mma0", "commit", "epi_acc", "epi_issued", "epi_done", "exit"};
  for (int i = 1; i < 9; ++i) printf(" %s=%lld", lab[i], h[i] - h[0]);
  printf("\n    tmem_ld0=%lld  full-wait done per k-block:", h[9] - h[0]);
  for (int i = 0; i < 8; ++i) printf(" %lld", h[16 + i] ? h[16 + i] - h[0] : -1);
  printf("\n    producer issued per k-block:");
  for (int i = 0; i < 4; ++i) printf(" %lld", h[24 + i] ? h[24 + i] - h[0] : -1);
  printf("\n    mma issued+committed per k-block:");
  for (int i = 0; i < 4; ++i) printf(" %lld", h[28 + i] ? h[28 + i] - h[0] : -1);
  printf("\n    epilogue chunk0: math done %lld, staging free %lld, staged %lld, fenced %lld",
         h[10] - h[0], h[11] - h[0], h[12] - h[0], h[13] - h[0]);
  cudaMemset(0, 0, 0);
  // the same shape with PDL off (plain stream order)
  g_pdl_enabled = 0;
  cudaEventRecord(e0, s);
  for (int i = 0; i < reps; ++i) call(g, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  g_pdl_enabled = 1;
  printf(" | no-PDL back-to-back %.2f us", ms * 1000.f / reps);
  printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Z);
}

// pure-write bandwidth baselines over n bytes: cudaMemsetAsync and a 16-byte-store kernel
__global__ void write_v4(float4* p, size_t n4) {
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
static void write_bw(size_t n) {
  void* p;
  cudaMalloc(&p, n);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      for (int i = 0; i < 5; ++i) {
        if (v == 0) cudaMemsetAsync(p, 0, n, s);
        else write_v4<<<148 * (v == 1 ? 4 : 16), 512, 0, s>>>((float4*)p, n / 16);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("write %s %.2f GB: %.1f us  %.0f GB/s\n", v == 0 ? "memset" : (v == 1 ? "v4x4" : "v4x16"), n / 1e9,
           ms * 200.f, n / (ms / 5.f * 1e-3) / 1e9);
  }
  cudaFree(p);
}

int main(int argc, char** argv) {
  gemm_tc_init();
  if (argc > 1) {  // "dw": the write baselines and the c4 expert-wgrad shapes only
    write_bw((size_t)4096 * 16384 * 16 * 4);
    for (g_variant = 0; g_variant < 2; ++g_variant) {
      printf("variant %d\n", g_variant);
      run("c4_dw1", 4096, 16384, 256, 16, EPI_STORE_F32);
      run("c4_dw2", 16384, 4096, 256, 16, EPI_STORE_F32);
      run("c3_dw1", 1024, 2048, 512, 16, EPI_STORE_F32);
      run("c4_e1", 256, 16384, 4096, 16, EPI_BIAS_GELU_G);
      run("c3_e1", 256, 2048, 1024, 16, EPI_BIAS_GELU_G);
      run("c4_dx", 1024, 4096, 4096, 1, EPI_STORE);
    }
    return 0;
  }
  run("c2_dctx", 256, 256, 256, 1, EPI_STORE);
  run("c2_qkv", 256, 768, 256, 1, EPI_STORE);
  run("c2_e1", 64, 512, 256, 8, EPI_BIAS_GELU);
  run("c2_e2", 64, 256, 512, 8, EPI_STORE);
  run("c2_dgelu", 64, 512, 256, 8, EPI_DGELU);
  run("c2_dw1", 256, 512, 256, 8, EPI_STORE_F32);
  run("c3_e1", 256, 2048, 1024, 8, EPI_BIAS_GELU);
  run("c4_dw1", 4096, 16384, 256, 16, EPI_STORE_F32);
  run("c3_dw1", 1024, 2048, 512, 16, EPI_STORE_F32);
  run("c3_e1_st", 256, 2048, 1024, 8, EPI_STORE);
  run("c3_e1_bn128", 256, 2048, 1024, 8, EPI_BIAS_GELU, 0, 128);
  run("c3_e1_bn64", 256, 2048, 1024, 8, EPI_BIAS_GELU, 0, 64);
  run("c3_dg", 256, 2048, 1024, 8, EPI_DGELU);
  run("c3_dg_bn128", 256, 2048, 1024, 8, EPI_DGELU, 0, 128);
  run("c4_e1", 256, 16384, 4096, 16, EPI_BIAS_GELU);
  run("c4_e1_bn128", 256, 16384, 4096, 16, EPI_BIAS_GELU, 0, 128);
  run("c4_qkv", 1024, 12288, 4096, 1, EPI_STORE);
  run("c4_qkv_bn128", 1024, 12288, 4096, 1, EPI_STORE, 0, 128);
  return 0;
}
