/*
 * mpix_testing.h — helper kernels for tests and the benchmark: the in-stream
 * "producer kernel -> send -> consumer kernel" chains of SURVEY.md §8(d),
 * the Listing-2 SAXPY and the cfg5 halo
 * stencil. Not part of the MPIX API; exported from the same library so the
 * chains run in the user's stream without torch ops in between.
 *
 * Every `stream` argument is a cudaStream_t passed as void*.
 */
#ifndef MPIX_TESTING_H
#define MPIX_TESTING_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* word i (uint32) = mpix_pattern_u32(seed, iter, i); see oracle/streamix_oracle.c */
int MPIXT_Fill_pattern(void *buf, uint64_t nbytes, uint32_t seed, uint32_t iter, void *stream);
/* *out_dev (device uint64) = order-independent checksum of nbytes
 * (oracle: orc_checksum64). Zeroes *out_dev first. */
int MPIXT_Checksum(const void *buf, uint64_t nbytes, uint64_t *out_dev, void *stream);
/* y[i] = a * x[i] + y[i] (fp32) — PAPER.md Listing 2 */
int MPIXT_Saxpy(int n, float a, const float *x, float *y, void *stream);
/* Busy-wait `ns` nanoseconds inside the stream (peer-delay tests). */
int MPIXT_Delay(uint64_t ns, void *stream);
/* One empty kernel (launch-floor measurement). */
int MPIXT_Empty(void *stream);
/* fill float buffer: x[i] = value */
int MPIXT_Fill_f32(float *x, uint64_t n, float value, void *stream);

/* cfg5 halo stencil on an (nx, ny, nz) fp32 block with a one-cell halo on
 * every face: storage (nx+2)*(ny+2)*(nz+2), x fastest.
 * face: 0=-x 1=+x 2=-y 3=+y 4=-z 5=+z. Pack copies the interior boundary
 * layer of `face` into buf; unpack writes buf into the halo layer of `face`. */
int MPIXT_Halo_pack(const float *u, int nx, int ny, int nz, int face, float *buf, void *stream);
int MPIXT_Halo_unpack(float *u, int nx, int ny, int nz, int face, const float *buf, void *stream);
/* out = 7-point Jacobi update of u's interior (halo read): out[c] = w0*u[c] +
 * w1*(sum of 6 neighbours); out's halo untouched. */
int MPIXT_Stencil7(const float *u, float *out, int nx, int ny, int nz, float w0, float w1,
                   void *stream);
/* Debug: device->host copy (synchronous), and the base/size of rank
 * `comm`'s peer-mapped region of that communicator. */
int MPIXT_Copy_to_host(void *host, const void *dev, uint64_t bytes);
/* Load every helper kernel on the current device (called by
 * MPIX_World_init; see lazy loading in DESIGN.md). */
int MPIXT_Preload(void);
/* Number of helper kernels launched so far. */
uint64_t MPIXT_Launch_count(void);

#ifdef __cplusplus
}
#endif

#endif
