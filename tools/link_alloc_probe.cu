// Host-link probe by host allocation kind (tools only): full-duplex pinned
// copies of N bytes each way (H2D from buffer A, D2H into buffer B, two
// streams), best of 5, for cudaHostAlloc default / write-combined /
// portable+mapped, and cudaHostRegister'ed malloc (2 MB aligned).
//   nvcc -O2 -o tools/link_alloc_probe tools/link_alloc_probe.cu && tools/link_alloc_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

static void run(const char *name, void *ha, void *hb, size_t n) {
  void *da, *db;
  CK(cudaMalloc(&da, n));
  CK(cudaMalloc(&db, n));
  cudaStream_t su, sd;
  CK(cudaStreamCreate(&su));
  CK(cudaStreamCreate(&sd));
  float best_u = 0, best_d = 0, best_both = 0, best_u1 = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEvent_t e0, e1, e2, e3;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0, su);
    cudaStreamWaitEvent(sd, e0, 0);
    CK(cudaMemcpyAsync(da, ha, n, cudaMemcpyHostToDevice, su));
    cudaEventRecord(e1, su);
    cudaEventRecord(e2, sd);
    CK(cudaMemcpyAsync(hb, db, n, cudaMemcpyDeviceToHost, sd));
    cudaEventRecord(e3, sd);
    CK(cudaDeviceSynchronize());
    float tu, td;
    cudaEventElapsedTime(&tu, e0, e1);
    cudaEventElapsedTime(&td, e0, e3);
    const float gu = n / (tu * 1e-3f) / 1e9f, gd = n / (td * 1e-3f) / 1e9f;
    if (gu > best_u) best_u = gu;
    if (gd > best_d) best_d = gd;
    const float both = 2.0f * n / ((tu > td ? tu : td) * 1e-3f) / 1e9f;
    if (both > best_both) best_both = both;
    // H2D alone
    cudaEventRecord(e0, su);
    CK(cudaMemcpyAsync(da, ha, n, cudaMemcpyHostToDevice, su));
    cudaEventRecord(e1, su);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&tu, e0, e1);
    const float g1 = n / (tu * 1e-3f) / 1e9f;
    if (g1 > best_u1) best_u1 = g1;
  }
  printf("{\"alloc\": \"%s\", \"bytes\": %zu, \"duplex_h2d_gbs\": %.2f, \"duplex_d2h_gbs\": %.2f, "
         "\"duplex_total_gbs\": %.2f, \"h2d_alone_gbs\": %.2f}\n", name, n, best_u, best_d, best_both, best_u1);
  cudaFree(da); cudaFree(db);
}

int main() {
  const size_t n = (size_t)1233125376;  // one OPT-30B block in bf16
  struct { const char *name; unsigned flags; } kinds[] = {
      {"cudaHostAlloc default", cudaHostAllocDefault},
      {"cudaHostAlloc write-combined", cudaHostAllocWriteCombined},
      {"cudaHostAlloc portable|mapped", cudaHostAllocPortable | cudaHostAllocMapped}};
  for (auto &k : kinds) {
    void *a, *b;
    CK(cudaHostAlloc(&a, n, k.flags));
    CK(cudaHostAlloc(&b, n, k.flags));
    memset(a, 1, n); memset(b, 2, n);
    run(k.name, a, b, n);
    cudaFreeHost(a); cudaFreeHost(b);
  }
  void *a = aligned_alloc(1 << 21, n), *b = aligned_alloc(1 << 21, n);
  memset(a, 1, n); memset(b, 2, n);
  CK(cudaHostRegister(a, n, cudaHostRegisterDefault));
  CK(cudaHostRegister(b, n, cudaHostRegisterDefault));
  run("malloc 2MB-aligned + cudaHostRegister", a, b, n);
  return 0;
}
