// taillaunch.cu — probe: cost/ordering of device-side tail launches (CDP2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O3 -o tools/taillaunch tools/taillaunch.cu -lcudadevrt
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_b(uint64_t* ts, int slot) {
  if (threadIdx.x == 0 && blockIdx.x == 0) ts[slot] = gt();
}
__global__ void k_wide(uint64_t* ts, int slot, const uint64_t* flag) {
  if (*flag == 0) return;
  if (threadIdx.x == 0 && blockIdx.x == 0) ts[slot] = gt();
}
__global__ void k_a(uint64_t* ts, int mode, const uint64_t* flag) {
  if (threadIdx.x != 0) return;
  ts[0] = gt();
  if (mode >= 1) k_b<<<1, 32, 0, cudaStreamTailLaunch>>>(ts, 1);
  if (mode >= 2) k_wide<<<8192, 1024, 0, cudaStreamTailLaunch>>>(ts, 2, flag);
  if (mode >= 3) k_b<<<1, 32, 0, cudaStreamTailLaunch>>>(ts, 3);
  ts[4] = gt();
}
__global__ void k_after(uint64_t* ts) { ts[5] = gt(); }

int main() {
  uint64_t *ts, *flag;
  cudaMalloc(&ts, 64 * 8);
  cudaMalloc(&flag, 8);
  cudaMemset(flag, 0, 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode <= 3; ++mode) {
    for (int f = 0; f < 2; ++f) {
      cudaMemsetAsync(flag, f, 1, s);
      double acc[6] = {0};
      int N = 50;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float ms_tot = 0;
      for (int i = 0; i < N + 5; ++i) {
        cudaMemsetAsync(ts, 0, 64 * 8, s);
        cudaEventRecord(e0, s);
        k_a<<<1, 32, 0, s>>>(ts, mode, flag);
        k_after<<<1, 32, 0, s>>>(ts);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        uint64_t h[8];
        cudaMemcpy(h, ts, 64, cudaMemcpyDeviceToHost);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) {
          ms_tot += ms;
          for (int k = 1; k < 6; ++k)
            if (h[k]) acc[k] += (double)(h[k] - h[0]);
        }
      }
      printf("mode %d flag %d: events %.2f us | ns after A start: B %.0f wide %.0f C %.0f A-end %.0f after %.0f\n",
             mode, f, ms_tot / N * 1e3, acc[1] / N, acc[2] / N, acc[3] / N, acc[4] / N, acc[5] / N);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
