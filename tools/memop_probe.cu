// memop_probe.cu — probe: stream memory operations (cuStreamWriteValue64 /
// cuStreamWaitValue64, no SM occupancy) against 1-thread spinning kernels
// for the flag waits of the enqueue path (VERDICT r1 "next" item 1,
// SURVEY.md §7.3.5).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/memop_probe tools/memop_probe.cu -lcuda
//   tools/memop_probe lat          latency: memop ping-pong vs kernel ping-pong vs kernel->memop chain
//   tools/memop_probe serial D     two host threads, memop barrier then a kernel each; thread 1
//                                  starts D ms late (run under ncu: does serialisation deadlock?)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <thread>

#define CKD(x)                                                     \
  do {                                                             \
    CUresult r_ = (x);                                             \
    if (r_ != CUDA_SUCCESS) {                                      \
      const char* s_ = nullptr;                                    \
      cuGetErrorString(r_, &s_);                                   \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_); \
      exit(1);                                                     \
    }                                                              \
  } while (0)

__global__ void k_set(uint64_t* f, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__global__ void k_spin(const uint64_t* f, uint64_t v) {
  uint64_t x;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
  } while (x < v);
}
__global__ void k_set_spin(uint64_t* peer, const uint64_t* mine, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(peer), "l"(v) : "memory");
  uint64_t x;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(mine) : "memory");
  } while (x < v);
}
__global__ void k_spin_set(uint64_t* peer, const uint64_t* mine, uint64_t v) {
  uint64_t x;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(mine) : "memory");
  } while (x < v);
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(peer), "l"(v) : "memory");
}
__global__ void k_touch(int* p) { atomicAdd(p, 1); }
// PDL variants: wait for the previous grid, let the next one launch at once
__global__ void k_set_spin_pdl(uint64_t* peer, const uint64_t* mine, uint64_t v) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(peer), "l"(v) : "memory");
  uint64_t x;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(mine) : "memory");
  } while (x < v);
}
__global__ void k_spin_set_pdl(uint64_t* peer, const uint64_t* mine, uint64_t v) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  uint64_t x;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(mine) : "memory");
  } while (x < v);
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(peer), "l"(v) : "memory");
}
template <typename K>
static void launch_pdl2(cudaStream_t s, K k, uint64_t* a, const uint64_t* b, uint64_t v) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, a, b, v);
}
__global__ void k_pdl_empty() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}
static void launch_pdl(cudaStream_t s, int threads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_pdl_empty);
}
__global__ void k_empty() {}

static void wr(cudaStream_t s, uint64_t* f, uint64_t v) {
  CKD(cuStreamWriteValue64((CUstream)s, (CUdeviceptr)f, v, 0));
}
static void wt(cudaStream_t s, uint64_t* f, uint64_t v) {
  CKD(cuStreamWaitValue64((CUstream)s, (CUdeviceptr)f, v, CU_STREAM_WAIT_VALUE_GEQ));
}

static double time_it(cudaStream_t s0, cudaStream_t s1, int mode, int n, uint64_t* f, uint64_t base) {
  uint64_t* f0 = f;
  uint64_t* f1 = f + 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s0);
  for (int i = 1; i <= n; ++i) {
    uint64_t v = base + i;
    switch (mode) {
      case 0:  // memop ping-pong
        wr(s0, f1, v);
        wt(s0, f0, v);
        wt(s1, f1, v);
        wr(s1, f0, v);
        break;
      case 1:  // kernel ping-pong
        k_set_spin<<<1, 1, 0, s0>>>(f1, f0, v);
        k_spin_set<<<1, 1, 0, s1>>>(f0, f1, v);
        break;
      case 2:  // kernel writes, memop waits (a completion word seen by a stream wait)
        k_set<<<1, 1, 0, s0>>>(f1, v);
        wt(s0, f0, v);
        wt(s1, f1, v);
        k_set<<<1, 1, 0, s1>>>(f0, v);
        break;
      case 3:  // empty kernels on s0 only (launch floor)
        k_empty<<<1, 1, 0, s0>>>();
        break;
      case 4:  // memop write + wait on s0 only (own flag, already satisfied)
        wr(s0, f0, v);
        wt(s0, f0, v);
        break;
      case 5:  // PDL chain of empty 32-thread kernels
        launch_pdl(s0, 32);
        break;
      case 6:  // PDL chain of empty 512-thread kernels
        launch_pdl(s0, 512);
        break;
      case 7:  // kernel ping-pong, PDL launches (each kernel pre-launched behind the previous)
        launch_pdl2(s0, k_set_spin_pdl, f1, f0, v);
        launch_pdl2(s1, k_spin_set_pdl, f0, f1, v);
        break;
    }
  }
  cudaEventRecord(e1, s0);
  cudaStreamSynchronize(s0);
  cudaStreamSynchronize(s1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3 / n;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const char* what = argc > 1 ? argv[1] : "lat";
  cudaSetDevice(0);
  cudaFree(0);
  CUdevice dev;
  CKD(cuDeviceGet(&dev, 0));
  int a64 = 0, nor = 0, flush = 0;
  cuDeviceGetAttribute(&a64, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev);
  cuDeviceGetAttribute(&nor, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, dev);
  cuDeviceGetAttribute(&flush, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, dev);
  printf("attr: 64bit_memops=%d wait_nor=%d flush_remote=%d\n", a64, nor, flush);
  uint64_t* f;
  cudaMalloc(&f, 4096);
  cudaMemset(f, 0, 4096);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  if (!strcmp(what, "lat")) {
    const char* names[] = {"memop ping-pong (us per round trip)", "kernel ping-pong", "kernel set -> memop wait",
                           "empty kernel", "memop write+wait (satisfied)",
                           "PDL empty kernel x32", "PDL empty kernel x512", "kernel ping-pong, PDL"};
    uint64_t base = 0;
    const int first = argc > 2 ? atoi(argv[2]) : 0;
    for (int mode = first; mode < 8; ++mode) {
      printf("mode %d ...\n", mode);
      cudaMemset(f, 0, 4096);
      cudaDeviceSynchronize();
      base = 0;
      time_it(s0, s1, mode, 100, f, base);
      base += 100;
      double us = time_it(s0, s1, mode, 2000, f, base);
      printf("%-40s %8.3f us\n", names[mode], us);
      fflush(stdout);
    }
    return 0;
  }
  // serial: two host threads, each: write peer flag, wait own flag, kernel
  int delay_ms = argc > 2 ? atoi(argv[2]) : 200;
  int* cnt;
  cudaMalloc(&cnt, 4);
  cudaMemset(cnt, 0, 4);
  cudaDeviceSynchronize();
  auto body = [&](int me) {
    cudaSetDevice(0);
    cudaStream_t s = me ? s1 : s0;
    if (me) std::this_thread::sleep_for(std::chrono::milliseconds(delay_ms));
    for (int it = 1; it <= 3; ++it) {
      wr(s, f + 8 * (1 - me), it);  // my arrival, in the peer's flag
      wt(s, f + 8 * me, it);        // peer's arrival
      k_touch<<<1, 32, 0, s>>>(cnt);
      wr(s, f + 16 + 8 * (1 - me), it);  // exit barrier
      wt(s, f + 16 + 8 * me, it);
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::thread t1(body, 1);
  body(0);
  t1.join();
  cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, cnt, 4, cudaMemcpyDeviceToHost);
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("serial: touched %d (expect 192), %.3f s, err=%s\n", h, s, cudaGetErrorString(cudaGetLastError()));
  return h == 192 ? 0 : 1;
}
