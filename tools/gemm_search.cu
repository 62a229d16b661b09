// Probe: exhaustive cuBLASLt configuration search (algo id x tile x stages x
// split-K x cluster shape) for the reuse-prefill projections at skinny n, next
// to the heuristic's top candidates.  Row-major y[n][m] = x[n][k] W[m][k]^T.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/gemm_search tools/gemm_search.cu -lcublasLt
//   tools/gemm_search [m k n]
// Diagnostics only.
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
  const int m = argc > 3 ? atoi(argv[1]) : 15360, k = argc > 3 ? atoi(argv[2]) : 5120,
            n = argc > 3 ? atoi(argv[3]) : 301;
  cublasLtHandle_t h;
  cublasLtCreate(&h);
  const size_t ws_bytes = 32 << 20;
  void *ws, *W[3], *X, *Y;
  cudaMalloc(&ws, ws_bytes);
  for (auto& w : W) {
    cudaMalloc(&w, (size_t)m * k * 2);
    fill_kernel<<<1184, 256>>>((__nv_bfloat16*)w, (size_t)m * k, 17u);
  }
  cudaMalloc(&X, (size_t)n * k * 2);
  cudaMalloc(&Y, (size_t)n * m * 2);
  fill_kernel<<<1184, 256>>>((__nv_bfloat16*)X, (size_t)n * k, 99u);
  cudaDeviceSynchronize();
  cublasLtMatmulDesc_t op;
  cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
  cublasLtMatrixLayout_t la, lb, lc;
  cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, k, m, k);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, k, n, k);
  cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, m, n, m);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const float alpha = 1.f, beta = 0.f;
  auto time_algo = [&](const cublasLtMatmulAlgo_t& algo, size_t wsz) -> float {
    auto run = [&](int it) {
      return cublasLtMatmul(h, op, &alpha, W[it % 3], la, X, lb, &beta, Y, lc, Y, lc, &algo, ws,
                            wsz, s);
    };
    if (run(0) != CUBLAS_STATUS_SUCCESS) return -1.f;
    for (int it = 1; it < 4; ++it) run(it);
    cudaEventRecord(a, s);
    for (int it = 0; it < 20; ++it) run(it);
    cudaEventRecord(b, s);
    if (cudaEventSynchronize(b) != cudaSuccess) return -1.f;
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / 20;
  };
  // heuristic top-8
  cublasLtMatmulPreference_t pref;
  cublasLtMatmulPreferenceCreate(&pref);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes,
                                       sizeof(ws_bytes));
  cublasLtMatmulHeuristicResult_t res[8];
  int found = 0;
  cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 8, res, &found);
  float heur_best = 1e30f;
  for (int i = 0; i < found; ++i) {
    const float us = time_algo(res[i].algo, res[i].workspaceSize);
    if (us > 0) heur_best = std::min(heur_best, us);
    printf("heuristic #%d: %.1f us\n", i, us);
  }
  // exhaustive
  int ids[256], nids = 0;
  cublasLtMatmulAlgoGetIds(h, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF,
                           CUDA_R_16BF, CUDA_R_16BF, 256, ids, &nids);
  printf("%d algo ids\n", nids);
  float best = 1e30f;
  int tried = 0;
  char best_desc[256] = "";
  for (int ii = 0; ii < nids; ++ii) {
    cublasLtMatmulAlgo_t algo;
    if (cublasLtMatmulAlgoInit(h, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF,
                               CUDA_R_16BF, CUDA_R_16BF, ids[ii], &algo) != CUBLAS_STATUS_SUCCESS)
      continue;
    size_t sz = 0;
    std::vector<int> tiles(1, 0), stages(1, 0), clusters(1, 0);
    if (cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, nullptr, 0, &sz) ==
            CUBLAS_STATUS_SUCCESS && sz) {
      tiles.resize(sz / sizeof(int));
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, tiles.data(), sz, &sz);
    }
    if (cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_STAGES_IDS, nullptr, 0, &sz) ==
            CUBLAS_STATUS_SUCCESS && sz) {
      stages.resize(sz / sizeof(int));
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_STAGES_IDS, stages.data(), sz,
                                        &sz);
    }
    clusters = {CUBLASLT_CLUSTER_SHAPE_AUTO, CUBLASLT_CLUSTER_SHAPE_1x1x1,
                CUBLASLT_CLUSTER_SHAPE_2x1x1, CUBLASLT_CLUSTER_SHAPE_1x2x1,
                CUBLASLT_CLUSTER_SHAPE_2x2x1};
    int splitk_support = 0;
    cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_SPLITK_SUPPORT, &splitk_support,
                                      sizeof(int), &sz);
    const int splits[] = {1, 2, 3, 4};
    for (int t : tiles)
      for (int st : stages)
        for (int cl : clusters)
          for (int sk : splits) {
            if (sk > 1 && !splitk_support) continue;
            cublasLtMatmulAlgo_t al = algo;
            cublasLtMatmulAlgoConfigSetAttribute(&al, CUBLASLT_ALGO_CONFIG_TILE_ID, &t, sizeof(t));
            cublasLtMatmulAlgoConfigSetAttribute(&al, CUBLASLT_ALGO_CONFIG_STAGES_ID, &st,
                                                 sizeof(st));
            cublasLtMatmulAlgoConfigSetAttribute(&al, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID, &cl,
                                                 sizeof(cl));
            cublasLtMatmulAlgoConfigSetAttribute(&al, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &sk,
                                                 sizeof(sk));
            cublasLtMatmulHeuristicResult_t chk = {};
            if (cublasLtMatmulAlgoCheck(h, op, la, lb, lc, lc, &al, &chk) != CUBLAS_STATUS_SUCCESS)
              continue;
            if (chk.workspaceSize > ws_bytes) continue;
            ++tried;
            const float us = time_algo(al, chk.workspaceSize);
            if (us > 0 && us < best) {
              best = us;
              snprintf(best_desc, sizeof(best_desc), "id %d tile %d stages %d cluster %d splitk %d",
                       ids[ii], t, st, cl, sk);
            }
          }
  }
  const double fl = 2.0 * m * n * k;
  printf("m=%d k=%d n=%d: heuristic best %.1f us (%.0f TF/s); exhaustive best of %d: %.1f us "
         "(%.0f TF/s) [%s]\n",
         m, k, n, heur_best, fl / heur_best * 1e-6, tried, best, fl / best * 1e-6, best_desc);
  return 0;
}
