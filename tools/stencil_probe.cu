// stencil_probe.cu — probe: shapes of the cfg5 7-point stencil (one rank's
// (n+2)^3 fp32 block) against the HBM roofline, all bit-identical to
// orc_stencil7 (explicit roundings, no FMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stencil_probe tools/stencil_probe.cu
//   tools/stencil_probe [n=512] [iters=20]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__host__ __device__ __forceinline__ uint64_t hidx(int x, int y, int z, int nx, int ny) {
  return ((uint64_t)z * (ny + 2) + y) * (uint64_t)(nx + 2) + x;
}

__device__ __forceinline__ float st7(float xm, float xp, float ym, float yp, float zm, float zp, float c,
                                     float w0, float w1) {
  float s = __fadd_rn(xm, xp);
  s = __fadd_rn(s, __fadd_rn(ym, yp));
  s = __fadd_rn(s, __fadd_rn(zm, zp));
  return __fadd_rn(__fmul_rn(w0, c), __fmul_rn(w1, s));
}

// A: the round-1 kernel (one thread per point, 128-wide rows)
__global__ void k_naive(const float* __restrict__ u, float* __restrict__ out, int nx, int ny, int nz,
                        float w0, float w1) {
  int x = blockIdx.x * blockDim.x + threadIdx.x + 1;
  int y = blockIdx.y + 1;
  int z = blockIdx.z + 1;
  if (x > nx) return;
  const uint64_t sx = 1, sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  uint64_t c = hidx(x, y, z, nx, ny);
  out[c] = st7(u[c - sx], u[c + sx], u[c - sy], u[c + sy], u[c - sz], u[c + sz], u[c], w0, w1);
}

// B: z-marching column per thread, z neighbours in registers, x/y
// neighbours through L1 (read-only path). Box [x0,x1]x[y0,y1]x[z0,z1].
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) k_zmarch(const float* __restrict__ u, float* __restrict__ out,
                                                  int nx, int ny, int x0, int x1, int y0, int y1,
                                                  int z0, int z1, float w0, float w1) {
  const int x = x0 + blockIdx.x * BX + threadIdx.x;
  const int y = y0 + blockIdx.y * BY + threadIdx.y;
  const int zs = z0 + blockIdx.z * ZC;
  if (x > x1 || y > y1 || zs > z1) return;
  const int ze = min(zs + ZC - 1, z1);
  const uint64_t sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  uint64_t c = hidx(x, y, zs, nx, ny);
  float below = __ldg(u + c - sz), cen = __ldg(u + c), above = __ldg(u + c + sz);
  for (int z = zs; z <= ze; ++z) {
    const float nxt = z < ze ? __ldg(u + c + 2 * sz) : 0.f;
    const float r = st7(__ldg(u + c - 1), __ldg(u + c + 1), __ldg(u + c - sy), __ldg(u + c + sy), below,
                        above, cen, w0, w1);
    __stcs(out + c, r);
    below = cen;
    cen = above;
    above = nxt;
    c += sz;
  }
}

// C: z-marching with the plane tile in shared memory (x/y neighbours from
// smem, halo ring loaded by edge threads).
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) k_zsmem(const float* __restrict__ u, float* __restrict__ out,
                                                 int nx, int ny, int x0, int x1, int y0, int y1,
                                                 int z0, int z1, float w0, float w1) {
  __shared__ float t[2][BY + 2][BX + 2];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = x0 + blockIdx.x * BX + tx;
  const int y = y0 + blockIdx.y * BY + ty;
  const int zs = z0 + blockIdx.z * ZC;
  const int ze = min(zs + ZC - 1, z1);
  const bool in = x <= x1 && y <= y1;
  const uint64_t sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  // clamp loads to the block (x, y <= n + 1 is always inside the array)
  const int xc = min(x, nx + 1), yc = min(y, ny + 1);
  uint64_t c = hidx(xc, yc, zs, nx, ny);
  float below = __ldg(u + c - sz), cen = __ldg(u + c), above = __ldg(u + c + sz);
  int b = 0;
  for (int z = zs; z <= ze; ++z) {
    const float nxt = z < ze ? __ldg(u + c + 2 * sz) : 0.f;
    t[b][ty + 1][tx + 1] = cen;
    if (tx == 0) t[b][ty + 1][0] = __ldg(u + c - 1);
    if (tx == BX - 1 || x == x1) t[b][ty + 1][tx + 2] = __ldg(u + c + 1);
    if (ty == 0) t[b][0][tx + 1] = __ldg(u + c - sy);
    if (ty == BY - 1 || y == y1) t[b][ty + 2][tx + 1] = __ldg(u + c + sy);
    __syncthreads();
    if (in) {
      const float r = st7(t[b][ty + 1][tx], t[b][ty + 1][tx + 2], t[b][ty][tx + 1], t[b][ty + 2][tx + 1],
                          below, above, cen, w0, w1);
      __stcs(out + c, r);
    }
    b ^= 1;
    below = cen;
    cen = above;
    above = nxt;
    c += sz;
  }
}

// D: warp = 32 consecutive x; each thread marches R consecutive y rows:
// x neighbours by shuffle (edge lanes load), inner y neighbours from the
// registers of the rows above/below, only rows y0-1 and y0+R loaded.
template <int BY, int R, int ZC>
__global__ void __launch_bounds__(32 * BY) k_zrows(const float* __restrict__ u, float* __restrict__ out,
                                                  int nx, int ny, int x0, int x1, int y0, int y1,
                                                  int z0, int z1, float w0, float w1) {
  const int lane = threadIdx.x;
  const int x = x0 + blockIdx.x * 32 + lane;
  const int yb = y0 + (blockIdx.y * BY + threadIdx.y) * R;
  const int zs = z0 + blockIdx.z * ZC;
  if (yb > y1 || zs > z1) return;  // whole warp exits together (yb per warp)
  const bool in = x <= x1;
  const int xc = min(x, nx + 1);
  const int ze = min(zs + ZC - 1, z1);
  const uint64_t sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  uint64_t c = hidx(xc, yb, zs, nx, ny);
  float bl[R], ce[R], ab[R], nx_[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int yy = min(yb + k, ny + 1);
    const uint64_t ck = c + (uint64_t)(yy - yb) * sy;
    bl[k] = __ldg(u + ck - sz);
    ce[k] = __ldg(u + ck);
    ab[k] = __ldg(u + ck + sz);
  }
  for (int z = zs; z <= ze; ++z) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int yy = min(yb + k, ny + 1);
      nx_[k] = z < ze ? __ldg(u + c + (uint64_t)(yy - yb) * sy + 2 * sz) : 0.f;
    }
    const float ylo = __ldg(u + c - sy);
    const int ytop = min(yb + R, ny + 1);
    const float yhi = __ldg(u + c + (uint64_t)(ytop - yb) * sy);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float xm = __shfl_up_sync(0xffffffffu, ce[k], 1);
      float xp = __shfl_down_sync(0xffffffffu, ce[k], 1);
      const uint64_t ck = c + (uint64_t)k * sy;
      if (lane == 0) xm = __ldg(u + ck - 1);
      if (lane == 31 || x == x1) xp = __ldg(u + ck + 1);
      const float ym = k == 0 ? ylo : ce[k - 1];
      const float yp = k == R - 1 ? yhi : ce[k + 1];
      if (in && yb + k <= y1) __stcs(out + ck, st7(xm, xp, ym, yp, bl[k], ab[k], ce[k], w0, w1));
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      bl[k] = ce[k];
      ce[k] = ab[k];
      ab[k] = nx_[k];
    }
    c += sz;
  }
}

// E: the same z-march but the output goes to a dense, 128-B aligned n^3
// array (timing only: tells whether the misaligned halo-layout stores cost)
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) k_zmarch_dense(const float* __restrict__ u, float* __restrict__ out,
                                                        int nx, int ny, int nz, float w0, float w1) {
  const int x = 1 + blockIdx.x * BX + threadIdx.x;
  const int y = 1 + blockIdx.y * BY + threadIdx.y;
  const int zs = 1 + blockIdx.z * ZC;
  if (x > nx || y > ny || zs > nz) return;
  const int ze = min(zs + ZC - 1, nz);
  const uint64_t sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  uint64_t c = hidx(x, y, zs, nx, ny);
  uint64_t o = ((uint64_t)(zs - 1) * ny + (y - 1)) * nx + (x - 1);
  float below = __ldg(u + c - sz), cen = __ldg(u + c), above = __ldg(u + c + sz);
  for (int z = zs; z <= ze; ++z) {
    const float nxt = z < ze ? __ldg(u + c + 2 * sz) : 0.f;
    __stcs(out + o, st7(__ldg(u + c - 1), __ldg(u + c + 1), __ldg(u + c - sy), __ldg(u + c + sy), below,
                        above, cen, w0, w1));
    below = cen;
    cen = above;
    above = nxt;
    c += sz;
    o += (uint64_t)nx * ny;
  }
}
// F: interior copy in the halo layout (same misaligned rows, no stencil)
__global__ void k_rowcopy(const float* __restrict__ u, float* __restrict__ out, int nx, int ny, int nz) {
  const int x = 1 + blockIdx.x * 32 + threadIdx.x;
  const int y = 1 + blockIdx.y * 8 + threadIdx.y;
  if (x > nx || y > ny) return;
  for (int z = 1 + blockIdx.z * 16; z <= min(nz, 16 + blockIdx.z * 16); ++z) {
    const uint64_t c = hidx(x, y, z, nx, ny);
    __stcs(out + c, __ldg(u + c));
  }
}
// G: plain stores instead of streaming stores
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) k_zmarch_st(const float* __restrict__ u, float* __restrict__ out,
                                                     int nx, int ny, int x0, int x1, int y0, int y1,
                                                     int z0, int z1, float w0, float w1) {
  const int x = x0 + blockIdx.x * BX + threadIdx.x;
  const int y = y0 + blockIdx.y * BY + threadIdx.y;
  const int zs = z0 + blockIdx.z * ZC;
  if (x > x1 || y > y1 || zs > z1) return;
  const int ze = min(zs + ZC - 1, z1);
  const uint64_t sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  uint64_t c = hidx(x, y, zs, nx, ny);
  float below = __ldg(u + c - sz), cen = __ldg(u + c), above = __ldg(u + c + sz);
  for (int z = zs; z <= ze; ++z) {
    const float nxt = z < ze ? __ldg(u + c + 2 * sz) : 0.f;
    out[c] = st7(__ldg(u + c - 1), __ldg(u + c + 1), __ldg(u + c - sy), __ldg(u + c + sy), below, above,
                 cen, w0, w1);
    below = cen;
    cen = above;
    above = nxt;
    c += sz;
  }
}

__global__ void k_fill(float* u, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    u[i] = (float)(h & 0xffffff) / 16777216.0f - 0.5f;
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512;
  const int iters = argc > 2 ? atoi(argv[2]) : 20;
  const uint64_t N = (uint64_t)(n + 2) * (n + 2) * (n + 2);
  float *u, *a, *b, *flush;
  cudaMalloc(&u, N * 4);
  cudaMalloc(&a, N * 4);
  cudaMalloc(&b, N * 4);
  cudaMalloc(&flush, 256 << 20);
  k_fill<<<1184, 256>>>(u, N);
  cudaMemset(a, 0, N * 4);
  cudaMemset(b, 0, N * 4);
  const float w0 = 0.5f, w1 = 1.0f / 12.0f;
  const double bytes = 2.0 * (double)n * n * n * 4.0;  // read u once + write out once (interior)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_naive<<<dim3((n + 127) / 128, n, n), 128>>>(u, a, n, n, n, w0, w1);
  cudaDeviceSynchronize();
  float* hr = (float*)malloc(N * 4);
  float* ht = (float*)malloc(N * 4);
  cudaMemcpy(hr, a, N * 4, cudaMemcpyDeviceToHost);
  auto run = [&](const char* name, auto launch) {
    cudaMemset(b, 0, N * 4);
    launch();
    cudaDeviceSynchronize();
    cudaMemcpy(ht, b, N * 4, cudaMemcpyDeviceToHost);
    bool same = memcmp(hr, ht, N * 4) == 0;
    float tot = 0;
    for (int i = 0; i < iters; ++i) {
      cudaMemsetAsync(flush, i, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    const double us = tot * 1e3 / iters;
    printf("%-28s %9.1f us  %7.1f GB/s  bitexact=%d  err=%s\n", name, us, bytes / us / 1e3, same,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("naive 128", [&] { k_naive<<<dim3((n + 127) / 128, n, n), 128>>>(u, b, n, n, n, w0, w1); });
  run("naive 128 (b)", [&] { k_naive<<<dim3((n + 127) / 128, n, n), 128>>>(u, b, n, n, n, w0, w1); });
#define ZM(BX, BY, ZC)                                                                                   \
  run("zmarch " #BX "x" #BY " z" #ZC, [&] {                                                            \
    k_zmarch<BX, BY, ZC><<<dim3((n + BX - 1) / BX, (n + BY - 1) / BY, (n + ZC - 1) / ZC), dim3(BX, BY)>>>( \
        u, b, n, n, 1, n, 1, n, 1, n, w0, w1);                                                          \
  });
#define ZS(BX, BY, ZC)                                                                                   \
  run("zsmem " #BX "x" #BY " z" #ZC, [&] {                                                             \
    k_zsmem<BX, BY, ZC><<<dim3((n + BX - 1) / BX, (n + BY - 1) / BY, (n + ZC - 1) / ZC), dim3(BX, BY)>>>(  \
        u, b, n, n, 1, n, 1, n, 1, n, w0, w1);                                                          \
  });
  ZM(32, 4, 8) ZM(32, 4, 16) ZM(32, 8, 16) ZM(32, 8, 32) ZM(64, 4, 16) ZM(64, 4, 32) ZM(128, 2, 16)
  ZM(128, 2, 64) ZM(32, 16, 64) ZM(64, 8, 64)
#define ZR(BY, R, ZC)                                                                                      \
  run("zrows 32x" #BY " R" #R " z" #ZC, [&] {                                                              \
    k_zrows<BY, R, ZC><<<dim3((n + 31) / 32, (n + BY * R - 1) / (BY * R), (n + ZC - 1) / ZC), dim3(32, BY)>>>( \
        u, b, n, n, 1, n, 1, n, 1, n, w0, w1);                                                              \
  });
  ZR(4, 2, 16) ZR(4, 4, 16) ZR(8, 2, 16) ZR(8, 4, 16) ZR(4, 8, 16) ZR(8, 4, 32) ZR(4, 4, 64) ZR(2, 8, 32)
  ZR(8, 2, 8) ZR(16, 2, 16)
  run("zmarch dense-out 32x8 z16 (timing)", [&] {
    k_zmarch_dense<32, 8, 16><<<dim3((n + 31) / 32, (n + 7) / 8, (n + 15) / 16), dim3(32, 8)>>>(u, b, n, n, n, w0, w1);
  });
  run("rowcopy halo layout (timing)", [&] {
    k_rowcopy<<<dim3((n + 31) / 32, (n + 7) / 8, (n + 15) / 16), dim3(32, 8)>>>(u, b, n, n, n);
  });
  run("zmarch plain-st 32x8 z16", [&] {
    k_zmarch_st<32, 8, 16><<<dim3((n + 31) / 32, (n + 7) / 8, (n + 15) / 16), dim3(32, 8)>>>(u, b, n, n, 1, n, 1, n, 1, n, w0, w1);
  });
  run("zmarch plain-st 32x8 z8", [&] {
    k_zmarch_st<32, 8, 8><<<dim3((n + 31) / 32, (n + 7) / 8, (n + 7) / 8), dim3(32, 8)>>>(u, b, n, n, 1, n, 1, n, 1, n, w0, w1);
  });
  ZS(32, 4, 16) ZS(32, 8, 16) ZS(32, 8, 32) ZS(64, 4, 32) ZS(64, 8, 64) ZS(128, 4, 32)
  // plain copy of the same bytes (roofline sanity)
  run("memcpy d2d (n^3*4)", [&] { cudaMemcpyAsync(b, u, (uint64_t)n * n * n * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}
