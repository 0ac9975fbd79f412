// mpix_drivers.cpp — native benchmark drivers over the public C ABI
// (include/mpix_testing.h, MPIXT_Msgrate / MPIXT_Pingpong / MPIXT_Selfchain).
//
// The reference's own benchmark drivers are C++ threads calling Proc methods
// (proj/src/bench.cpp:118-235, oracle/ref_driver.cpp mirrors them for the
// enqueue path). These do the same against include/mpix.h: one host thread
// per rank, every call through the C ABI, device time from CUDA events on
// the ranks' streams. Python (ctypes) would otherwise bound the host side of
// the message-rate and latency measurements.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <vector>

#include "mpix.h"
#include "mpix_testing.h"

namespace {

struct Spin {  // host-thread barrier (all ranks start enqueueing together)
  std::atomic<int> n{0};
  int total;
  explicit Spin(int t) : total(t) {}
  void arrive_and_wait() {
    n.fetch_add(1);
    while (n.load() < total) std::this_thread::yield();
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

int MPIXT_Msgrate(int P, int S, int W, int batches, MPI_Comm* comms, void** streams, void** sbufs,
                  void** rbufs, int* devices, double* host_s, double* dev_s) {
  if (P < 1 || S < 1 || W < 1 || W > 4096 || batches < 1) return MPIX_ERR_INVALID_ARG;
  std::vector<cudaEvent_t> e0(P * S), e1(P * S);
  for (int i = 0; i < P * S; ++i) {
    cudaSetDevice(devices[i / S]);
    if (cudaEventCreate(&e0[i]) != cudaSuccess || cudaEventCreate(&e1[i]) != cudaSuccess)
      return MPIX_ERR_CUDA;
  }
  std::atomic<int> err{0};
  Spin go(P);
  double t0 = 0, t1 = 0;
  auto rank = [&](int r) {
    cudaSetDevice(devices[r]);
    MPIX_Rank_bind(r);
    const int right = (r + 1) % P, left = (r + P - 1) % P;
    std::vector<MPI_Request> reqs(2 * W);
    for (int k = 0; k < S; ++k) cudaEventRecord(e0[r * S + k], (cudaStream_t)streams[r * S + k]);
    go.arrive_and_wait();
    if (r == 0) t0 = now_s();
    for (int b = 0; b < batches && !err.load(); ++b) {
      for (int k = 0; k < S; ++k) {
        MPI_Comm c = comms[r * S + k];
        uint8_t* rb = static_cast<uint8_t*>(rbufs[r * S + k]);
        for (int i = 0; i < W; ++i) {
          int rc = MPIX_Irecv_enqueue(rb + 8 * i, 2, MPI_INT, left, i, c, &reqs[2 * i]);
          rc |= MPIX_Isend_enqueue(sbufs[r * S + k], 2, MPI_INT, right, i, c, &reqs[2 * i + 1]);
          if (rc) err.store(rc);
        }
        int rc = MPIX_Waitall_enqueue(2 * W, reqs.data(), MPI_STATUSES_IGNORE);
        if (rc) err.store(rc);
      }
    }
    for (int k = 0; k < S; ++k) cudaEventRecord(e1[r * S + k], (cudaStream_t)streams[r * S + k]);
  };
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r) th.emplace_back(rank, r);
  for (auto& t : th) t.join();
  t1 = now_s();
  for (int i = 0; i < P * S; ++i) cudaEventSynchronize(e1[i]);
  double tend = now_s();
  float mx = 0;
  for (int i = 0; i < P * S; ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e0[i], e1[i]);
    mx = std::max(mx, ms);
    cudaEventDestroy(e0[i]);
    cudaEventDestroy(e1[i]);
  }
  if (host_s) host_s[0] = t1 - t0, host_s[1] = tend - t0;
  if (dev_s) *dev_s = mx / 1e3;
  return err.load();
}

// The reference's lock-regime message-rate bench (paper Fig. 3,
// proj/src/bench.cpp:118-235: sender_loop / receiver_loop): two ranks, T
// driver threads each, thread t of rank 0 streams W conventional MPI_Isend of
// `bytes` to thread t of rank 1 over their own communicator, MPI_Waitall, then
// waits for a 1-byte credit (MPI_Recv) that rank 1 returns after its W
// MPI_Irecv + MPI_Waitall (tag 0 data, tag 1 credit). The regime is the
// world's host exclusion (MPIXT_Set_exclusion). bufs[r * T + t] holds W
// message slots plus one credit byte; *elapsed_s = last stop - first start
// over all threads (host clock, as the reference); *messages = T * W *
// batches (counted on the receive side).
int MPIXT_Fig3(int T, int W, int batches, int bytes, MPI_Comm* comms, void** bufs, int* devices,
               double* elapsed_s, long* messages) {
  if (T < 1 || W < 1 || W > 4096 || batches < 1 || bytes < 0) return MPIX_ERR_INVALID_ARG;
  std::atomic<int> err{0};
  Spin go(2 * T);
  std::vector<double> t_start(2 * T), t_stop(2 * T);
  const uint64_t slot = bytes > 0 ? (uint64_t)bytes : 1;
  auto body = [&](int r, int t) {
    cudaSetDevice(devices[r]);
    MPIX_Rank_bind(r);
    MPI_Comm c = comms[r * T + t];
    uint8_t* b = static_cast<uint8_t*>(bufs[r * T + t]);
    uint8_t* credit = b + slot * W;
    std::vector<MPI_Request> reqs(W);
    auto round = [&]() -> int {
      int rc = 0;
      if (r == 0) {
        for (int i = 0; i < W && !rc; ++i) rc = MPI_Isend(b, bytes, MPI_BYTE, 1, 0, c, &reqs[i]);
        if (!rc) rc = MPI_Waitall(W, reqs.data(), MPI_STATUSES_IGNORE);
        if (!rc) rc = MPI_Recv(credit, 1, MPI_BYTE, 1, 1, c, MPI_STATUS_IGNORE);
      } else {
        for (int i = 0; i < W && !rc; ++i) rc = MPI_Irecv(b + slot * i, bytes, MPI_BYTE, 0, 0, c, &reqs[i]);
        if (!rc) rc = MPI_Waitall(W, reqs.data(), MPI_STATUSES_IGNORE);
        if (!rc) rc = MPI_Send(credit, 1, MPI_BYTE, 0, 1, c);
      }
      return rc;
    };
    int rc = round();  // warm-up window
    if (rc) err.store(rc);
    go.arrive_and_wait();
    t_start[r * T + t] = now_s();
    for (int k = 0; k < batches && !rc && !err.load(); ++k) rc = round();
    if (rc) err.store(rc);
    t_stop[r * T + t] = now_s();
  };
  std::vector<std::thread> th;
  for (int r = 0; r < 2; ++r)
    for (int t = 0; t < T; ++t) th.emplace_back(body, r, t);
  for (auto& x : th) x.join();
  const double t0 = *std::min_element(t_start.begin(), t_start.end());
  const double t1 = *std::max_element(t_stop.begin(), t_stop.end());
  if (elapsed_s) *elapsed_s = t1 - t0;
  if (messages) *messages = (long)T * W * batches;
  return err.load();
}

// Bidirectional exchange between ranks 0 and 1 (one host thread each):
// per step Irecv_enqueue + Isend_enqueue of `bytes` + Waitall_enqueue, the
// cross-rank device handshake on both messages. *dev_s = max over the two
// streams of event time for `iters` steps.
int MPIXT_Exchange(MPI_Comm c0, MPI_Comm c1, void* s0buf, void* r0buf, void* s1buf, void* r1buf,
                   uint64_t bytes, int iters, void* st0, void* st1, int dev0, int dev1,
                   double* dev_s) {
  if (iters < 1) return MPIX_ERR_INVALID_ARG;
  cudaEvent_t ev[2][2];
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(r ? dev1 : dev0);
    if (cudaEventCreate(&ev[r][0]) != cudaSuccess || cudaEventCreate(&ev[r][1]) != cudaSuccess)
      return MPIX_ERR_CUDA;
  }
  std::atomic<int> err{0};
  Spin go(2);
  const int count = (int)bytes;
  auto side = [&](int r) {
    cudaSetDevice(r ? dev1 : dev0);
    MPIX_Rank_bind(r);
    MPI_Comm c = r ? c1 : c0;
    void* sb = r ? s1buf : s0buf;
    void* rb = r ? r1buf : r0buf;
    cudaStream_t s = (cudaStream_t)(r ? st1 : st0);
    cudaEventRecord(ev[r][0], s);
    go.arrive_and_wait();
    for (int i = 0; i < iters && !err.load(); ++i) {
      MPI_Request q[2];
      int rc = MPIX_Irecv_enqueue(rb, count, MPI_BYTE, 1 - r, 9, c, &q[0]);
      rc |= MPIX_Isend_enqueue(sb, count, MPI_BYTE, 1 - r, 9, c, &q[1]);
      rc |= MPIX_Waitall_enqueue(2, q, MPI_STATUSES_IGNORE);
      if (rc) err.store(rc);
    }
    cudaEventRecord(ev[r][1], s);
  };
  std::thread t(side, 1);
  side(0);
  t.join();
  float mx = 0;
  for (int r = 0; r < 2; ++r) {
    cudaSetDevice(r ? dev1 : dev0);
    cudaEventSynchronize(ev[r][1]);
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[r][0], ev[r][1]);
    mx = std::max(mx, ms);
    cudaEventDestroy(ev[r][0]);
    cudaEventDestroy(ev[r][1]);
  }
  cudaSetDevice(dev0);
  if (dev_s) *dev_s = mx / 1e3;
  return err.load();
}

int MPIXT_Pingpong(MPI_Comm c0, MPI_Comm c1, void* b0, void* b1, uint64_t bytes, int iters,
                   void* s0, void* s1, int dev0, int dev1, double* dev_s, double* host_s) {
  if (iters < 1) return MPIX_ERR_INVALID_ARG;
  cudaEvent_t a, b;
  cudaSetDevice(dev0);
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  std::atomic<int> err{0};
  Spin go(2);
  double t0 = 0, t1 = 0;
  const int count = (int)bytes;
  auto side = [&](int r) {
    cudaSetDevice(r ? dev1 : dev0);
    MPIX_Rank_bind(r);
    if (r == 0) cudaEventRecord(a, (cudaStream_t)s0);
    go.arrive_and_wait();
    if (r == 0) t0 = now_s();
    for (int i = 0; i < iters && !err.load(); ++i) {
      int rc;
      if (r == 0) {
        rc = MPIX_Send_enqueue(b0, count, MPI_BYTE, 1, 1, c0);
        rc |= MPIX_Recv_enqueue(b0, count, MPI_BYTE, 1, 2, c0, MPI_STATUS_IGNORE);
      } else {
        rc = MPIX_Recv_enqueue(b1, count, MPI_BYTE, 0, 1, c1, MPI_STATUS_IGNORE);
        rc |= MPIX_Send_enqueue(b1, count, MPI_BYTE, 0, 2, c1);
      }
      if (rc) err.store(rc);
    }
    if (r == 0) {
      cudaEventRecord(b, (cudaStream_t)s0);
      t1 = now_s();
    }
  };
  std::thread t(side, 1);
  side(0);
  t.join();
  cudaEventSynchronize(b);
  cudaSetDevice(dev1);
  cudaStreamSynchronize((cudaStream_t)s1);  // rank 1's last send retired too
  cudaSetDevice(dev0);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err.load();
}

// One side of a blocking ping-pong (multi-process mode: each process drives
// its own rank): the initiator sends then receives, the other side receives
// then sends; *dev_s = event time on this side's stream.
int MPIXT_Pingpong_side(MPI_Comm c, void* buf, uint64_t bytes, int iters, int peer, int initiator,
                        void* stream, double* dev_s) {
  if (iters < 1) return MPIX_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  const int count = (int)bytes;
  int err = 0;
  cudaEventRecord(a, s);
  for (int i = 0; i < iters && !err; ++i) {
    if (initiator) {
      err |= MPIX_Send_enqueue(buf, count, MPI_BYTE, peer, 1, c);
      err |= MPIX_Recv_enqueue(buf, count, MPI_BYTE, peer, 2, c, MPI_STATUS_IGNORE);
    } else {
      err |= MPIX_Recv_enqueue(buf, count, MPI_BYTE, peer, 1, c, MPI_STATUS_IGNORE);
      err |= MPIX_Send_enqueue(buf, count, MPI_BYTE, peer, 2, c);
    }
  }
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  return err;
}

// cfg2 streaming bandwidth, one side of a pair ("window of
// 16 Isend/Irecv_enqueue + Waitall_enqueue"): `reps` windows of W messages
// of `bytes`; the sender sends every message from buf, the receiver
// receives message i of a window at buf + i * bytes. Device time of the
// windows on the stream.
int MPIXT_Stream_window(MPI_Comm c, void* buf, uint64_t bytes, int W, int reps, int peer, int sender,
                        void* stream, double* dev_s, double* host_s) {
  if (W < 1 || W > 64 || reps < 1) return MPIX_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  const int count = (int)bytes;
  int err = 0;
  MPI_Request reqs[64];
  cudaEventRecord(a, s);
  const double t0 = now_s();
  for (int k = 0; k < reps && !err; ++k) {
    for (int i = 0; i < W && !err; ++i) {
      if (sender)
        err |= MPIX_Isend_enqueue(buf, count, MPI_BYTE, peer, 100 + i, c, &reqs[i]);
      else
        err |= MPIX_Irecv_enqueue(static_cast<uint8_t*>(buf) + (uint64_t)i * bytes, count, MPI_BYTE, peer,
                                  100 + i, c, &reqs[i]);
    }
    if (!err) err |= MPIX_Waitall_enqueue(W, reqs, MPI_STATUSES_IGNORE);
  }
  cudaEventRecord(b, s);
  const double t1 = now_s();
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err;
}

// producer kernel -> Send_enqueue -> Recv_enqueue -> consumer kernel, all on
// one stream (self messages), `iters` times.
int MPIXT_Selfchain(MPI_Comm c, float* prod, float* cons, int n, int iters, void* stream,
                    double* dev_s, double* host_s) {
  if (iters < 1) return MPIX_ERR_INVALID_ARG;
  int me = 0;
  MPI_Comm_rank(c, &me);
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  int err = 0;
  cudaEventRecord(a, s);
  double t0 = now_s();
  for (int i = 0; i < iters && !err; ++i) {
    err |= MPIXT_Fill_f32(prod, n, (float)i, s);
    err |= MPIX_Send_enqueue(prod, n, MPI_FLOAT, me, 3, c);
    err |= MPIX_Recv_enqueue(cons, n, MPI_FLOAT, me, 3, c, MPI_STATUS_IGNORE);
    err |= MPIXT_Fill_f32(cons, 0, 0.f, s);  // consumer kernel
  }
  cudaEventRecord(b, s);
  double t1 = now_s();
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err;
}

// cfg5: `steps` halo-exchange steps of a 2x2x2 periodic decomposition, one
// host thread per rank (8 ranks), all in the rank's stream (the structure of
// workloads.HaloStencil.step). u/v[r] are the rank's two (n+2)^3 blocks
// (swapped each step), sbuf/rbuf[r*6+d] its n*n face buffers. mode:
//   HALO_SEQ       pack6 -> 6 Irecv + 6 Isend_enqueue -> Waitall_enqueue ->
//                  unpack6 -> stencil (the whole block)
//   HALO_PIPE      the interior [2,n-1]^3 runs on a second stream while the
//                  faces are packed, exchanged and unpacked; the boundary
//                  shell runs after the unpack (same results, bit for bit)
//   HALO_COMPUTE   the stencil alone (no exchange)
//   HALO_EXCHANGE  pack6 -> exchange -> unpack6 alone (no stencil)
int MPIXT_Halo_steps(int n, int steps, int mode, MPI_Comm* comms, void** streams, int* devices,
                     float** u, float** v, float** sbuf, float** rbuf, float w0, float w1,
                     double* dev_s, double* host_s) {
  const int P = 8;
  if (mode < HALO_SEQ || mode > HALO_EXCHANGE) return MPIX_ERR_INVALID_ARG;
  static const int opp[6] = {1, 0, 3, 2, 5, 4};
  auto neighbour = [](int r, int d) {
    int c[3] = {r & 1, (r >> 1) & 1, (r >> 2) & 1};
    const int axis = d >> 1;
    c[axis] = (c[axis] + ((d & 1) ? 1 : -1) + 2) % 2;
    return c[0] | (c[1] << 1) | (c[2] << 2);
  };
  std::vector<cudaEvent_t> e0(P), e1(P), ea(P), eb(P);
  std::vector<cudaStream_t> s2(P, nullptr);
  for (int r = 0; r < P; ++r) {
    cudaSetDevice(devices[r]);
    if (cudaEventCreate(&e0[r]) != cudaSuccess || cudaEventCreate(&e1[r]) != cudaSuccess ||
        cudaEventCreateWithFlags(&ea[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&eb[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s2[r], cudaStreamNonBlocking) != cudaSuccess)
      return MPIX_ERR_CUDA;
  }
  std::atomic<int> err{0};
  Spin go(P);
  double t0 = 0, t1 = 0;
  auto rank = [&](int r) {
    cudaSetDevice(devices[r]);
    MPIX_Rank_bind(r);
    void* s = streams[r];
    float* a = u[r];
    float* b = v[r];
    cudaEventRecord(e0[r], (cudaStream_t)s);
    go.arrive_and_wait();
    if (r == 0) t0 = now_s();
    MPI_Request reqs[12];
    for (int it = 0; it < steps && !err.load(); ++it) {
      int rc = 0;
      if (mode == HALO_PIPE) {  // interior on s2, behind everything before this step
        cudaEventRecord(ea[r], (cudaStream_t)s);
        cudaStreamWaitEvent(s2[r], ea[r], 0);
        rc |= MPIXT_Stencil7_box(a, b, n, n, n, 2, n - 1, 2, n - 1, 2, n - 1, w0, w1, s2[r]);
        cudaEventRecord(eb[r], s2[r]);
      }
      if (mode != HALO_COMPUTE) {
        rc |= MPIXT_Halo_pack6(a, n, n, n, sbuf + r * 6, s);
        for (int d = 0; d < 6; ++d)
          rc |= MPIX_Irecv_enqueue(rbuf[r * 6 + d], n * n, MPI_FLOAT, neighbour(r, d), opp[d],
                                   comms[r], &reqs[d]);
        for (int d = 0; d < 6; ++d)
          rc |= MPIX_Isend_enqueue(sbuf[r * 6 + d], n * n, MPI_FLOAT, neighbour(r, d), d, comms[r],
                                   &reqs[6 + d]);
        rc |= MPIX_Waitall_enqueue(12, reqs, MPI_STATUSES_IGNORE);
        rc |= MPIXT_Halo_unpack6(a, n, n, n, rbuf + r * 6, s);
      }
      if (mode == HALO_PIPE) {
        rc |= MPIXT_Stencil7_shell(a, b, n, n, n, w0, w1, s);
        cudaStreamWaitEvent((cudaStream_t)s, eb[r], 0);
      } else if (mode != HALO_EXCHANGE) {
        rc |= MPIXT_Stencil7(a, b, n, n, n, w0, w1, s);
      }
      if (mode != HALO_EXCHANGE) std::swap(a, b);
      if (rc) err.store(rc);
    }
    cudaEventRecord(e1[r], (cudaStream_t)s);
  };
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r) th.emplace_back(rank, r);
  for (auto& t : th) t.join();
  t1 = now_s();
  float mx = 0;
  for (int r = 0; r < P; ++r) {
    cudaEventSynchronize(e1[r]);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0[r], e1[r]);
    mx = std::max(mx, ms);
    cudaEventDestroy(e0[r]);
    cudaEventDestroy(e1[r]);
    cudaStreamSynchronize(s2[r]);
    cudaEventDestroy(ea[r]);
    cudaEventDestroy(eb[r]);
    cudaStreamDestroy(s2[r]);
  }
  if (dev_s) *dev_s = mx / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err.load();
}

// Loopback: `iters` x {Isend_enqueue + Irecv_enqueue + Waitall_enqueue} of a
// self-message on one stream (the bench's N=1 step, any size).
int MPIXT_Loopback(MPI_Comm c, const void* src, void* dst, uint64_t bytes, int iters, void* stream,
                   double* dev_s, double* host_s) {
  if (iters < 1) return MPIX_ERR_INVALID_ARG;
  int me = 0;
  MPI_Comm_rank(c, &me);
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  int err = 0;
  cudaEventRecord(a, s);
  double t0 = now_s();
  for (int i = 0; i < iters && !err; ++i) {
    MPI_Request r[2];
    err |= MPIX_Isend_enqueue(src, (int)bytes, MPI_BYTE, me, 7, c, &r[0]);
    err |= MPIX_Irecv_enqueue(dst, (int)bytes, MPI_BYTE, me, 7, c, &r[1]);
    err |= MPIX_Waitall_enqueue(2, r, MPI_STATUSES_IGNORE);
  }
  cudaEventRecord(b, s);
  double t1 = now_s();
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err;
}

// `iters` x MPIX_Allreduce_enqueue(sbuf[r] -> rbuf[r], count, dt, op) per
// rank, one native thread per rank; *dev_s = max over ranks of event time.
int MPIXT_Allreduce_loop(int P, MPI_Comm* comms, void** streams, int* devices, void** sbufs,
                         void** rbufs, int count, MPI_Datatype dt, MPI_Op op, int iters,
                         double* dev_s, double* host_s) {
  if (P < 1 || iters < 1) return MPIX_ERR_INVALID_ARG;
  std::vector<cudaEvent_t> e0(P), e1(P);
  for (int r = 0; r < P; ++r) {
    cudaSetDevice(devices[r]);
    if (cudaEventCreate(&e0[r]) != cudaSuccess || cudaEventCreate(&e1[r]) != cudaSuccess)
      return MPIX_ERR_CUDA;
  }
  std::atomic<int> err{0};
  Spin go(P);
  double t0 = 0, t1 = 0;
  auto rank = [&](int r) {
    cudaSetDevice(devices[r]);
    MPIX_Rank_bind(r);
    cudaEventRecord(e0[r], (cudaStream_t)streams[r]);
    go.arrive_and_wait();
    if (r == 0) t0 = now_s();
    for (int i = 0; i < iters && !err.load(); ++i) {
      int rc = MPIX_Allreduce_enqueue(sbufs[r], rbufs[r], count, dt, op, comms[r]);
      if (rc) err.store(rc);
    }
    cudaEventRecord(e1[r], (cudaStream_t)streams[r]);
  };
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r) th.emplace_back(rank, r);
  for (auto& t : th) t.join();
  t1 = now_s();
  float mx = 0;
  for (int r = 0; r < P; ++r) {
    cudaEventSynchronize(e1[r]);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0[r], e1[r]);
    mx = std::max(mx, ms);
    cudaEventDestroy(e0[r]);
    cudaEventDestroy(e1[r]);
  }
  if (dev_s) *dev_s = mx / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err.load();
}

// Back-to-back empty kernels from C++ (the in-stream launch floor).
int MPIXT_Empty_loop(int iters, void* stream, double* dev_s, double* host_s) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t a, b;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return MPIX_ERR_CUDA;
  cudaEventRecord(a, s);
  double t0 = now_s();
  int err = 0;
  for (int i = 0; i < iters && !err; ++i) err |= MPIXT_Empty(s);
  cudaEventRecord(b, s);
  double t1 = now_s();
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (dev_s) *dev_s = ms / 1e3;
  if (host_s) *host_s = t1 - t0;
  return err;
}

}  // extern "C"
