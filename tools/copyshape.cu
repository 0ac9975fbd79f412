// copyshape.cu — probe for the p2p copy grid shape on B200 (not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/copyshape tools/copyshape.cu
// For a 256 MiB copy, times (CUDA events, median of 20) each shape both when
// it copies and when it is a no-op (the side of a message that lost the
// handshake still has its grid launched behind k_proto).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// static tiles: CTA t copies tiles t, t+grid, ... ; TV = vectors per tile
template <int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_tiles(uint4* dst, const uint4* src, uint64_t nvec, const int* act) {
  if (*act == 0) return;
  constexpr uint64_t TV = (uint64_t)THREADS * UNROLL;
  for (uint64_t t = blockIdx.x; t * TV < nvec; t += gridDim.x) {
    uint64_t base = t * TV + threadIdx.x;
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) v[u] = src[base + u * THREADS];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) dst[base + u * THREADS] = v[u];
  }
}

// dynamic tiles: CTAs grab tiles from an atomic counter (persistent grid)
template <int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_dyn(uint4* dst, const uint4* src, uint64_t nvec, const int* act,
                                                 unsigned long long* ctr) {
  if (*act == 0) return;
  constexpr uint64_t TV = (uint64_t)THREADS * UNROLL;
  __shared__ uint64_t s_t;
  const uint64_t nt = (nvec + TV - 1) / TV;
  while (true) {
    if (threadIdx.x == 0) s_t = atomicAdd(ctr, 1ull);
    __syncthreads();
    uint64_t t = s_t;
    __syncthreads();
    if (t >= nt) break;
    uint64_t base = t * TV + threadIdx.x;
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) v[u] = src[base + u * THREADS];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) dst[base + u * THREADS] = v[u];
  }
}

template <typename F>
float timeit(F f, int iters = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> ts;
  f();
  cudaDeviceSynchronize();
  for (int i = 0; i < iters; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2] * 1e3f;  // us
}

int main() {
  const uint64_t n = 256ull << 20, nvec = n / 16;
  uint4 *src, *dst;
  int *on, *off;
  unsigned long long* ctr;
  CK(cudaMalloc(&src, n));
  CK(cudaMalloc(&dst, n));
  CK(cudaMalloc(&on, 4));
  CK(cudaMalloc(&off, 4));
  CK(cudaMalloc(&ctr, 8));
  int one = 1, zero = 0;
  CK(cudaMemcpy(on, &one, 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(off, &zero, 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(src, 1, n));
  int sms = 148;
  auto rep = [&](const char* name, float t_on, float t_off) {
    printf("%-34s copy %8.1f us  %7.1f GB/s(2S)   no-op %6.2f us\n", name, t_on, 2.0 * n / t_on / 1e3, t_off);
  };
#define TILES(TH, UN, GRID, NAME)                                                               \
  {                                                                                             \
    uint64_t g = (GRID);                                                                        \
    float a = timeit([&] { k_tiles<TH, UN><<<g, TH>>>(dst, src, nvec, on); });                  \
    float b = timeit([&] { k_tiles<TH, UN><<<g, TH>>>(dst, src, nvec, off); });                 \
    char buf[64]; snprintf(buf, 64, "%s g=%llu", NAME, (unsigned long long)g); rep(buf, a, b);  \
  }
  const uint64_t t1024x2 = nvec / (1024 * 2);
  TILES(1024, 2, t1024x2, "tiles 1024x2 (current)");
  TILES(1024, 2, sms * 2 * 8, "tiles 1024x2 capped 16/SM");
  TILES(1024, 2, sms * 2 * 4, "tiles 1024x2 capped 8/SM");
  TILES(1024, 2, sms * 2 * 2, "tiles 1024x2 capped 4/SM");
  TILES(512, 4, nvec / (512 * 4), "tiles 512x4");
  TILES(512, 4, sms * 4 * 4, "tiles 512x4 capped 16/SM");
  TILES(256, 8, nvec / (256 * 8), "tiles 256x8");
  TILES(256, 8, sms * 8 * 2, "tiles 256x8 capped 16/SM");
  TILES(256, 8, sms * 8 * 4, "tiles 256x8 capped 32/SM");
  TILES(512, 8, nvec / (512 * 8), "tiles 512x8");
  TILES(512, 8, sms * 4 * 4, "tiles 512x8 capped 16/SM");
  TILES(1024, 4, nvec / (1024 * 4), "tiles 1024x4");
  TILES(1024, 4, sms * 2 * 4, "tiles 1024x4 capped 8/SM");
#define DYN(TH, UN, GRID, NAME)                                                                 \
  {                                                                                             \
    uint64_t g = (GRID);                                                                        \
    float a = timeit([&] { cudaMemsetAsync(ctr, 0, 8); k_dyn<TH, UN><<<g, TH>>>(dst, src, nvec, on, ctr); }); \
    float b = timeit([&] { cudaMemsetAsync(ctr, 0, 8); k_dyn<TH, UN><<<g, TH>>>(dst, src, nvec, off, ctr); }); \
    char buf[64]; snprintf(buf, 64, "%s g=%llu", NAME, (unsigned long long)g); rep(buf, a, b);  \
  }
  DYN(1024, 2, sms * 2, "dyn 1024x2 persistent");
  DYN(1024, 4, sms * 2, "dyn 1024x4 persistent");
  DYN(512, 4, sms * 4, "dyn 512x4 persistent");
  DYN(512, 8, sms * 4, "dyn 512x8 persistent");
  DYN(256, 8, sms * 8, "dyn 256x8 persistent");
  float ms0 = timeit([&] { cudaMemsetAsync(ctr, 0, 8); });
  printf("memset alone %.2f us\n", ms0);
  float cp = timeit([&] { cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice); });
  rep("cudaMemcpyAsync D2D", cp, 0);
  return 0;
}
