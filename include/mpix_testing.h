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

#include "mpix.h"

#ifdef __cplusplus
extern "C" {
#endif

/* word i (uint32) = mpix_pattern_u32(seed, iter, i); see oracle/streamix_oracle.c */
int MPIXT_Fill_pattern(void *buf, uint64_t nbytes, uint32_t seed, uint32_t iter, void *stream);
/* *out_dev (device uint64) = order-independent checksum of nbytes
 * (oracle: orc_checksum64). Zeroes *out_dev first. */
int MPIXT_Checksum(const void *buf, uint64_t nbytes, uint64_t *out_dev, void *stream);
/* cfg3 inputs of rank `rank`: count elements of dt (MPI_FLOAT or
 * MPIX_BFLOAT16) from value set 0 (exact) or 1 (uniform(-1,1)); oracle:
 * orc_value_f32 / orc_value_bf16. */
int MPIXT_Fill_values(void *buf, uint64_t count, int dt, int set, uint32_t rank, void *stream);
/* y[i] = a * x[i] + y[i] (fp32) — PAPER.md Listing 2 */
int MPIXT_Saxpy(int n, float a, const float *x, float *y, void *stream);
/* Busy-wait `ns` nanoseconds inside the stream (peer-delay tests). */
int MPIXT_Delay(uint64_t ns, void *stream);
/* A fresh non-blocking CUDA stream on `device` (not from torch's 32-stream
 * pool, which aliases streams beyond 32), and its destruction. */
int MPIXT_Stream_create(int device, void **stream);
/* The same with a stream priority (0 = default/lowest, negative = higher;
 * clamped to the device's range). */
int MPIXT_Stream_create_prio(int device, int priority, void **stream);
int MPIXT_Stream_destroy(void *stream);
/* One empty kernel (launch-floor measurement). */
int MPIXT_Empty(void *stream);
/* Replay-dependent data for CUDA-Graph tests: x[i] = (*iter + 1) * a + b * (i % 7);
 * check counts mismatches into *bad_dev; bump advances *iter (all in-stream). */
int MPIXT_Iter_fill(float *x, uint64_t n, const uint32_t *iter, float a, float b, void *stream);
int MPIXT_Iter_check(const float *x, uint64_t n, const uint32_t *iter, float a, float b,
                     uint64_t *bad_dev, void *stream);
int MPIXT_Iter_bump(uint32_t *iter, void *stream);
/* CUDA-Graph capture of one stream (thread-local capture mode), instantiate,
 * replay, destroy. */
int MPIXT_Graph_begin(void *stream);
int MPIXT_Graph_end(void *stream, void **exec);
int MPIXT_Graph_launch(void *exec, void *stream);
int MPIXT_Graph_destroy(void *exec);
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
/* The same update restricted to the box [x0,x1]x[y0,y1]x[z0,z1] (1-based
 * interior coordinates; an empty box is a no-op), and to the boundary shell
 * (every point with a coordinate 1 or n: exactly the points that read a
 * halo). Interior box [2,n-1]^3 + shell = the whole update, so a pipelined
 * step runs the interior while the faces are in flight. */
int MPIXT_Stencil7_box(const float *u, float *out, int nx, int ny, int nz, int x0, int x1, int y0,
                       int y1, int z0, int z1, float w0, float w1, void *stream);
int MPIXT_Stencil7_shell(const float *u, float *out, int nx, int ny, int nz, float w0, float w1,
                         void *stream);
/* All six faces in one launch: bufs[face] for face 0..5. */
int MPIXT_Halo_pack6(const float *u, int nx, int ny, int nz, float *const *bufs, void *stream);
int MPIXT_Halo_unpack6(float *u, int nx, int ny, int nz, float *const *bufs, void *stream);
/* Debug: device->host copy (synchronous), and the base/size of rank
 * `comm`'s peer-mapped region of that communicator. */
int MPIXT_Copy_to_host(void *host, const void *dev, uint64_t bytes);
/* Load every helper kernel on the current device (called by
 * MPIX_World_init; see lazy loading in DESIGN.md). */
int MPIXT_Preload(void);
/* Native benchmark drivers (csrc/mpix_drivers.cpp): one host thread per
 * rank, every call through the C ABI, device time from CUDA events.
 * Msgrate (cfg4): P ranks x S single-stream comms (index r*S+k); per batch
 * and stream, W x {Irecv_enqueue(left, tag i) + Isend_enqueue(right, tag i)}
 * of 8 bytes, then Waitall_enqueue. rbufs hold W*8 bytes. host_s[0] = enqueue
 * time, host_s[1] = until the last stream drained; *dev_s = max over streams
 * of event time. */
int MPIXT_Msgrate(int P, int S, int W, int batches, MPI_Comm *comms, void **streams, void **sbufs,
                  void **rbufs, int *devices, double *host_s, double *dev_s);
/* The reference's lock-regime message-rate bench (paper Fig. 3,
 * proj/src/bench.cpp:118-235) over conventional p2p: 2 ranks x T threads,
 * windows of W MPI_Isend / MPI_Irecv + MPI_Waitall + a 1-byte credit.
 * comms/bufs: [r * T + t]; bufs hold W slots of max(bytes, 1) + 1 byte. */
int MPIXT_Fig3(int T, int W, int batches, int bytes, MPI_Comm *comms, void **bufs, int *devices,
               double *elapsed_s, long *messages);
/* The world's host exclusion regime (MPIX_HOST_EXCLUSION at init):
 * 0 global lock, 1 per communicator, 2 serial contexts lock-free. Call with
 * no operation in flight. Returns the previous regime in *prev. */
int MPIXT_Set_exclusion(int regime, int *prev);
/* Bidirectional exchange of `bytes` between ranks 0 and 1: per step each
 * rank enqueues Irecv + Isend + Waitall (one host thread per rank);
 * *dev_s = max over the two streams of event time for `iters` steps. */
int MPIXT_Exchange(MPI_Comm c0, MPI_Comm c1, void *s0buf, void *r0buf, void *s1buf, void *r1buf,
                   uint64_t bytes, int iters, void *st0, void *st1, int dev0, int dev1,
                   double *dev_s);
/* Blocking ping-pong of `bytes` between ranks 0 (c0, s0) and 1 (c1, s1):
 * Send+Recv / Recv+Send, `iters` round trips; *dev_s = event time on s0. */
int MPIXT_Pingpong(MPI_Comm c0, MPI_Comm c1, void *b0, void *b1, uint64_t bytes, int iters,
                   void *s0, void *s1, int dev0, int dev1, double *dev_s, double *host_s);
/* One side of a blocking ping-pong with `peer` (multi-process mode, one
 * process per rank): the initiator sends then receives. */
int MPIXT_Pingpong_side(MPI_Comm c, void *buf, uint64_t bytes, int iters, int peer, int initiator,
                        void *stream, double *dev_s);
/* producer kernel -> Send_enqueue -> Recv_enqueue -> consumer kernel (self
 * messages of n floats on one stream), `iters` times. */
/* cfg2 streaming bandwidth, one side of a pair: reps windows of W (<= 64)
 * Isend/Irecv_enqueue of `bytes` + Waitall_enqueue; receive i of a window
 * lands at buf + i * bytes. Device seconds of the windows. */
int MPIXT_Stream_window(MPI_Comm c, void *buf, uint64_t bytes, int W, int reps, int peer, int sender,
                        void *stream, double *dev_s, double *host_s);
int MPIXT_Selfchain(MPI_Comm c, float *prod, float *cons, int n, int iters, void *stream,
                    double *dev_s, double *host_s);
/* cfg5: `steps` halo steps of the 2x2x2 periodic 8-rank decomposition (pack
 * 6 faces, 6 Irecv + 6 Isend_enqueue, Waitall_enqueue, unpack, stencil),
 * one native thread per rank. Arrays are indexed by rank (u, v, comms,
 * streams, devices) or rank*6+face (sbuf, rbuf). u and v swap every step
 * (not in HALO_EXCHANGE). Modes: */
enum { HALO_SEQ = 0, HALO_PIPE = 1, HALO_COMPUTE = 2, HALO_EXCHANGE = 3 };
int MPIXT_Halo_steps(int n, int steps, int mode, MPI_Comm *comms, void **streams, int *devices, float **u,
                     float **v, float **sbuf, float **rbuf, float w0, float w1, double *dev_s,
                     double *host_s);
/* `iters` x {Isend + Irecv + Waitall_enqueue} of a self-message of `bytes`
 * on the comm's stream (the benchmark's N=1 step, native loop). */
int MPIXT_Loopback(MPI_Comm c, const void *src, void *dst, uint64_t bytes, int iters, void *stream,
                   double *dev_s, double *host_s);
/* `iters` x Allreduce_enqueue per rank from one native thread per rank
 * (arrays indexed by rank); *dev_s = max over ranks of event time. */
int MPIXT_Allreduce_loop(int P, MPI_Comm *comms, void **streams, int *devices, void **sbufs,
                         void **rbufs, int count, MPI_Datatype dt, MPI_Op op, int iters,
                         double *dev_s, double *host_s);
/* `iters` back-to-back empty kernels launched from C++ (launch floor). */
int MPIXT_Empty_loop(int iters, void *stream, double *dev_s, double *host_s);
/* The Allreduce_enqueue reduce stage alone (no entry/exit barrier): rank
 * `me`'s share of a P-rank allreduce over P send/recv buffers on the current
 * GPU (one-shot: all of rank me's output; two-shot: chunk me into every
 * output). For ncu, which serialises kernels and so cannot run the spinning
 * barriers of several ranks sharing one GPU. Not thread-safe. */
int MPIXT_Reduce_only(int P, int me, void **sendbufs, void **recvbufs, int count,
                      MPI_Datatype datatype, MPI_Op op, int twoshot, void *stream);
/* Timing probe for the benchmark's roofline: while enabled, the runtime
 * records CUDA events around every copy grid (k_gcopy / k_copy) it launches,
 * on both sides of a message; read returns the summed duration, count and
 * bytes of the grids whose decision records say they copied (the second
 * arriver's; the other side's grid is empty). Enabling clears. */
int MPIXT_Copy_timing(int enable);
int MPIXT_Copy_timing_read(double *total_ms, int *n, uint64_t *bytes);
/* Number of helper kernels launched so far. */
uint64_t MPIXT_Launch_count(void);

#ifdef __cplusplus
}
#endif

#endif
