// copybench.cu — design-space probe for the payload copy and the handshake
// primitives on B200 (not part of the product). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copybench tools/copybench.cu
// Prints GB/s (read+write bytes) for each copy variant at 256 MiB and the
// per-op latency of system-scope fences / acquire loads / release stores.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int UNROLL>
__global__ void k_copy_gs(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t nvec) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = t;
  for (; i + (UNROLL - 1) * nt < nvec; i += UNROLL * nt) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = src[i + u * nt];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) dst[i + u * nt] = v[u];
  }
  for (; i < nvec; i += nt) dst[i] = src[i];
}

// Contiguous chunk per CTA (each CTA streams its own range).
template <int UNROLL>
__global__ void k_copy_chunk(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t nvec) {
  uint64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  uint64_t b = per * blockIdx.x, e = b + per < nvec ? b + per : nvec;
  uint64_t i = b + threadIdx.x;
  for (; i + (UNROLL - 1) * blockDim.x < e; i += UNROLL * blockDim.x) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = src[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) dst[i + u * blockDim.x] = v[u];
  }
  for (; i < e; i += blockDim.x) dst[i] = src[i];
}

// non-coherent loads + no-allocate stores
template <int UNROLL>
__global__ void k_copy_nc(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t nvec) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = t;
  for (; i + (UNROLL - 1) * nt < nvec; i += UNROLL * nt) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * nt));
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i + u * nt),
                   "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w));
  }
  for (; i < nvec; i += nt) dst[i] = src[i];
}

// TMA bulk copy: global -> smem (mbarrier) -> global, one elected thread per
// CTA, STAGES buffers of CHUNK bytes, persistent over chunks.
template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(32) k_copy_bulk(uint8_t* dst, const uint8_t* src, uint64_t n) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  uint64_t nchunks = n / CHUNK;
  uint32_t phase[STAGES];
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  // issue loads for the first STAGES chunks of this CTA, then loop
  uint64_t c0 = blockIdx.x;
  auto issue = [&](int s, uint64_t c) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src + c * CHUNK), "r"(CHUNK), "r"(b) : "memory");
  };
  int s = 0;
  uint64_t c = c0;
  for (int k = 0; k < STAGES && c0 + (uint64_t)k * gridDim.x < nchunks; ++k)
    issue(k, c0 + (uint64_t)k * gridDim.x);
  for (; c < nchunks; c += gridDim.x) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(done) : "r"(b), "r"(phase[s]));
    }
    phase[s] ^= 1;
    uint32_t sp = (uint32_t)__cvta_generic_to_shared(smem + s * CHUNK);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CHUNK),
                 "r"(sp), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    uint64_t nxt = c + (uint64_t)STAGES * gridDim.x;
    if (nxt < nchunks) {
      // the store must have read smem before we refill it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(s, nxt);
    }
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// --- primitive latencies ---------------------------------------------------
__global__ void k_prims(uint64_t* buf, uint64_t* out, int iters) {
  uint64_t t0, t1;
  volatile uint64_t sink = 0;
  // fence.sc.sys
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) { buf[0] = i; asm volatile("fence.sc.sys;" ::: "memory"); }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = (t1 - t0) / iters;
  // fence.acq_rel.sys
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) { buf[0] = i; asm volatile("fence.acq_rel.sys;" ::: "memory"); }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[1] = (t1 - t0) / iters;
  // fence.sc.gpu
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) { buf[0] = i; asm volatile("fence.sc.gpu;" ::: "memory"); }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[2] = (t1 - t0) / iters;
  // ld.acquire.sys (dependent chain)
  uint64_t v = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    uint64_t x;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(buf + 8 + (v & 1)) : "memory");
    v += x;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[3] = (t1 - t0) / iters;
  // ld.relaxed.sys dependent chain
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    uint64_t x;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(buf + 8 + (v & 1)) : "memory");
    v += x;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[4] = (t1 - t0) / iters;
  // st.release.sys
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(buf + 16), "l"((uint64_t)i) : "memory");
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[5] = (t1 - t0) / iters;
  // atom.cas.sys
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    uint64_t o;
    asm volatile("atom.acq_rel.sys.global.cas.b64 %0, [%1], %2, %3;" : "=l"(o)
                 : "l"(buf + 24), "l"(v), "l"(v + 1) : "memory");
    v = o;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[6] = (t1 - t0) / iters;
  out[7] = v + sink;
}

__global__ void k_empty() {}

// non-persistent tiles: CTA b copies TILE_VEC vectors (UNROLL per thread)
template <int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) k_tile(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t nvec) {
  uint64_t base = (uint64_t)blockIdx.x * THREADS * UNROLL + threadIdx.x;
  uint4 v[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) v[u] = src[base + u * THREADS];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) if (base + u * THREADS < nvec) dst[base + u * THREADS] = v[u];
}
__global__ void k_exit_if(const uint64_t* flag) { if (*flag == 0) return; }

template <typename F>
float time_it(F f, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

int main() {
  const uint64_t n = 256ull << 20;
  uint8_t *a, *b;
  CK(cudaMalloc(&a, n));
  CK(cudaMalloc(&b, n));
  CK(cudaMemset(a, 1, n));
  uint64_t nvec = n / 16;
  int sms = 148;
  auto rep = [&](const char* name, float ms) {
    printf("%-40s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, 2.0 * n / (ms * 1e-3) / 1e9);
  };
  int threads_list[] = {256, 512, 1024};
  for (int th : threads_list) {
    for (int mult : {1, 2, 4, 8}) {
      int g = sms * mult * (1024 / th);
      if ((uint64_t)g * th > nvec) continue;
      char nm[96];
      snprintf(nm, sizeof nm, "gs<4> thr=%d grid=%d", th, g);
      rep(nm, time_it([&] { k_copy_gs<4><<<g, th>>>((uint4*)b, (uint4*)a, nvec); }, 20));
      snprintf(nm, sizeof nm, "gs<8> thr=%d grid=%d", th, g);
      rep(nm, time_it([&] { k_copy_gs<8><<<g, th>>>((uint4*)b, (uint4*)a, nvec); }, 20));
      snprintf(nm, sizeof nm, "nc<4> thr=%d grid=%d", th, g);
      rep(nm, time_it([&] { k_copy_nc<4><<<g, th>>>((uint4*)b, (uint4*)a, nvec); }, 20));
      snprintf(nm, sizeof nm, "chunk<4> thr=%d grid=%d", th, g);
      rep(nm, time_it([&] { k_copy_chunk<4><<<g, th>>>((uint4*)b, (uint4*)a, nvec); }, 20));
    }
  }
  // torch-like: one vector per thread, huge grid
  rep("gs<1> thr=128 grid=nvec/128", time_it([&] { k_copy_gs<1><<<(unsigned)(nvec / 128), 128>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<128,1>", time_it([&] { k_tile<128, 1><<<(unsigned)(nvec / 128), 128>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<256,1>", time_it([&] { k_tile<256, 1><<<(unsigned)(nvec / 256), 256>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<256,2>", time_it([&] { k_tile<256, 2><<<(unsigned)(nvec / 512), 256>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<256,4>", time_it([&] { k_tile<256, 4><<<(unsigned)(nvec / 1024), 256>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<256,8>", time_it([&] { k_tile<256, 8><<<(unsigned)(nvec / 2048), 256>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<512,4>", time_it([&] { k_tile<512, 4><<<(unsigned)(nvec / 2048), 512>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  rep("tile<1024,2>", time_it([&] { k_tile<1024, 2><<<(unsigned)(nvec / 2048), 1024>>>((uint4*)b, (uint4*)a, nvec); }, 20));
  {
    uint64_t* z;
    cudaMalloc(&z, 8);
    cudaMemset(z, 0, 8);
    for (unsigned g : {148u, 1184u, 4096u, 16384u, 131072u})
      printf("empty-exit grid %6u x256: %.2f us\n", g, time_it([&] { k_exit_if<<<g, 256>>>(z); }, 50) * 1e3);
  }
  rep("cudaMemcpyAsync D2D", time_it([&] { cudaMemcpyAsync(b, a, n, cudaMemcpyDeviceToDevice); }, 20));
  {
    constexpr int CH = 32768, ST = 4;
    cudaFuncSetAttribute(k_copy_bulk<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
    for (int mult : {1, 2}) {
      char nm[96];
      snprintf(nm, sizeof nm, "bulk<32K,4> grid=%d", sms * mult);
      rep(nm, time_it([&] { k_copy_bulk<CH, ST><<<sms * mult, 32, CH * ST>>>(b, a, n); }, 20));
    }
  }
  {
    constexpr int CH = 16384, ST = 4;
    cudaFuncSetAttribute(k_copy_bulk<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
    for (int mult : {2, 3}) {
      char nm[96];
      snprintf(nm, sizeof nm, "bulk<16K,4> grid=%d", sms * mult);
      rep(nm, time_it([&] { k_copy_bulk<CH, ST><<<sms * mult, 32, CH * ST>>>(b, a, n); }, 20));
    }
  }
  CK(cudaDeviceSynchronize());
  // verify last copy
  uint8_t h[16];
  CK(cudaMemcpy(h, b + n - 16, 16, cudaMemcpyDeviceToHost));
  printf("verify %d\n", h[15]);
  // primitives
  uint64_t *buf, *out;
  CK(cudaMalloc(&buf, 4096));
  CK(cudaMemset(buf, 0, 4096));
  CK(cudaMalloc(&out, 64));
  k_prims<<<1, 1>>>(buf, out, 1000);
  uint64_t o[8];
  CK(cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost));
  printf("ns/op: fence.sc.sys %lu  fence.acq_rel.sys %lu  fence.sc.gpu %lu  ld.acquire.sys %lu  ld.relaxed.sys %lu  st.release.sys %lu  cas.sys %lu\n",
         o[0], o[1], o[2], o[3], o[4], o[5], o[6]);
  printf("empty kernel back-to-back: %.2f us\n", time_it([&] { k_empty<<<1, 32>>>(); }, 1000) * 1e3);
  printf("empty kernel 296 CTAs x512: %.2f us\n", time_it([&] { k_empty<<<296, 512>>>(); }, 1000) * 1e3);
  return 0;
}
