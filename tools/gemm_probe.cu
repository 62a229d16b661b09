// Probe: cuBLASLt heuristic choice vs the best of its top-K candidates for
// the reuse-prefill projections (row-major y[n][m] = x[n][k] W[m][k]^T, the
// layout runtime.cu uses), LLaMA-2-13B / 7B shapes, n = new tokens per turn.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/gemm_probe tools/gemm_probe.cu -lcublasLt
//   tools/gemm_probe
//
// Weights rotate over buffers larger than L2 (as in the 40-layer loop).
// Diagnostics only.
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void fill_kernel(__nv_bfloat16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(((int)(x & 0xffff) - 32768) * (0.02f / 32768.f));
  }
}

int main(int argc, char** argv) {
  const int topk = 64;
  cublasLtHandle_t h;
  cublasLtCreate(&h);
  const size_t ws_bytes = 32 << 20;
  void* ws;
  CK(cudaMalloc(&ws, ws_bytes));
  struct Shape { const char* name; int m, k; };
  const Shape shapes[] = {{"13b qkv", 15360, 5120}, {"13b o", 5120, 5120},
                          {"13b gate|up", 27648, 5120}, {"13b down", 5120, 13824}};
  const int ns[] = {64, 128, 237, 301, 512, 746};
  const int nbuf = 3;
  void *W[nbuf], *X, *Y;
  const size_t wmax = (size_t)27648 * 5120 * 2;
  for (auto& w : W) {
    CK(cudaMalloc(&w, wmax));
    fill_kernel<<<1184, 256>>>((__nv_bfloat16*)w, wmax / 2, 17u);
  }
  CK(cudaMalloc(&X, (size_t)1024 * 13824 * 2));
  CK(cudaMalloc(&Y, (size_t)1024 * 27648 * 2));
  fill_kernel<<<1184, 256>>>((__nv_bfloat16*)X, (size_t)1024 * 13824, 99u);
  CK(cudaDeviceSynchronize());
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  double tot_h = 0, tot_b = 0;
  for (int n : ns) {
    for (const Shape& sh : shapes) {
      const int m = sh.m, k = sh.k;
      cublasLtMatmulDesc_t op;
      cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
      cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
      cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
      cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
      cublasLtMatrixLayout_t la, lb, lc;
      cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, k, m, k);
      cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, k, n, k);
      cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, m, n, m);
      cublasLtMatmulPreference_t pref;
      cublasLtMatmulPreferenceCreate(&pref);
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                           &ws_bytes, sizeof(ws_bytes));
      std::vector<cublasLtMatmulHeuristicResult_t> res(topk);
      int found = 0;
      cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, topk, res.data(), &found);
      const float alpha = 1.f, beta = 0.f;
      float best = 1e30f, first = 0.f;
      int best_i = -1;
      for (int i = 0; i < found; ++i) {
        auto run = [&](int it) {
          return cublasLtMatmul(h, op, &alpha, W[it % nbuf], la, X, lb, &beta, Y, lc, Y, lc,
                                &res[i].algo, ws, res[i].workspaceSize, s);
        };
        if (run(0) != CUBLAS_STATUS_SUCCESS) continue;
        for (int it = 0; it < 5; ++it) run(it);
        const int iters = 30;
        CK(cudaEventRecord(a, s));
        for (int it = 0; it < iters; ++it) run(it);
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const float us = ms * 1e3f / iters;
        if (i == 0) first = us;
        if (us < best) {
          best = us;
          best_i = i;
        }
      }
      const double fl = 2.0 * m * n * k;
      printf("n=%4d %-12s heuristic#0 %7.1f us (%6.0f TF/s)  best #%2d of %2d %7.1f us (%6.0f TF/s)  gain %4.1f%%\n",
             n, sh.name, first, fl / first * 1e-6, best_i, found, best, fl / best * 1e-6,
             100.0 * (first - best) / first);
      if (n == 301 || n == 237) {
        tot_h += first;
        tot_b += best;
      }
      cublasLtMatmulPreferenceDestroy(pref);
      cublasLtMatrixLayoutDestroy(la);
      cublasLtMatrixLayoutDestroy(lb);
      cublasLtMatrixLayoutDestroy(lc);
      cublasLtMatmulDescDestroy(op);
    }
  }
  printf("n in {237, 301}: heuristic %.1f us, best %.1f us per layer-pair\n", tot_h, tot_b);
  return 0;
}
