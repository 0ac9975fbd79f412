// mpix_kernels.cu — sm_100a kernels of the MPIX-stream GPU-enqueue path.
//
// One kernel per enqueued operation, launched into the user's CUDA stream:
//
//   k_p2p       Send/Isend/Recv/Irecv_enqueue. Replaces the reference's queue
//               worker running post_send/post_recv/wait closures
//               (proj/src/proc_enqueue.cpp:30-114, proj/src/proc_p2p.cpp:27-94)
//               and its matching/progress engine (proj/src/endpoint.cpp:15-69,
//               proj/src/fabric.cpp:93-110). CTA 0, warp 0 runs the handshake
//               on descriptor rings in peer-mapped memory; the copy (push or
//               pull, 128-bit vectors, grid-stride) is spread over the grid.
//   k_wait      Wait/Waitall_enqueue: spins on local completion words
//               (replaces proj/src/proc_enqueue.cpp:116-141).
//   k_allreduce Allreduce_enqueue (no reference): one-shot / two-shot P2P
//               reduce over peer buffers, rank-ordered fp32/fp64/int32 folds.
//
// Memory-model conventions: descriptor states and completion words are
// 64-bit, written with st.release.sys and read with ld.acquire.sys; the
// post->scan step of each side is separated by fence.sc.sys so that at least
// one of the two sides sees the other's descriptor (store-buffering litmus).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpix_internal.h"

namespace mpix {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t cas_sys(uint64_t* p, uint64_t cmp, uint64_t val) {
  uint64_t old;
  asm volatile("atom.acq_rel.sys.global.cas.b64 %0, [%1], %2, %3;"
               : "=l"(old)
               : "l"(p), "l"(cmp), "l"(val)
               : "memory");
  return old;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Error codes written to the per-rank error word (host-mapped) on watchdog
// expiry. The kernel then exits instead of hanging the GPU.
enum : uint64_t {
  ERRW_WAIT_SLOT = 1,
  ERRW_WAIT_DONE = 2,
  ERRW_WAIT_COLL = 3,
  ERRW_PROTOCOL = 4,
};

// Spin until *p >= target (acquire, system scope). Returns false on watchdog
// expiry after recording `code`.
__device__ __noinline__ bool spin_ge(const uint64_t* p, uint64_t target, uint64_t* err_word,
                                     uint64_t limit_ns, uint64_t code) {
  if (ld_acquire_sys(p) >= target) return true;
  uint64_t t0 = limit_ns ? globaltimer() : 0;
  unsigned ns = 32;
  while (ld_acquire_sys(p) < target) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (limit_ns && globaltimer() - t0 > limit_ns) {
      if (err_word) st_relaxed_sys(err_word, code);
      return false;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Copy: 128-bit vectors, UNROLL loads in flight per thread, grid-stride over
// `nparts` cooperating CTAs. Handles co-aligned heads/tails; falls back to a
// byte loop when source and destination disagree modulo 16.
// ---------------------------------------------------------------------------
template <int UNROLL>
__device__ __forceinline__ void copy_vec(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                         uint64_t nvec, uint64_t t, uint64_t nt) {
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

__device__ void part_copy(uint8_t* dst, const uint8_t* src, uint64_t n, uint64_t part,
                          uint64_t nparts) {
  if (n == 0 || dst == src) return;
  const uint64_t t = part * blockDim.x + threadIdx.x;
  const uint64_t nt = nparts * blockDim.x;
  uint64_t mis = (uint64_t)dst & 15;
  if ((((uint64_t)src) & 15) == mis) {
    uint64_t head = mis ? (16 - mis) : 0;
    if (head > n) head = n;
    if (t < head) dst[t] = src[t];
    uint64_t nvec = (n - head) >> 4;
    copy_vec<4>(reinterpret_cast<uint4*>(dst + head),
                reinterpret_cast<const uint4*>(src + head), nvec, t, nt);
    uint64_t done = head + (nvec << 4);
    uint64_t tail = n - done;
    if (t < tail) dst[done + t] = src[done + t];
  } else {
    for (uint64_t i = t; i < n; i += nt) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------------------
// Descriptor-ring scan (warp 0). Returns the slot index and a consistent
// snapshot (seqlock on the state word, which carries the pair sequence so it
// never repeats), or -1.
// ---------------------------------------------------------------------------
struct Snap {
  uint64_t state, key, addr, bytes, done_addr, done_val;
};

__device__ int warp_scan(SlotDesc* ring, int R, uint64_t key, Snap* out) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < R; base += 32) {
    int i = base + lane;
    bool hit = false;
    if (i < R) {
      uint64_t st = ld_acquire_sys(&ring[i].state);
      if ((st & 0xff) == ST_POSTED) hit = ld_relaxed_sys(&ring[i].key) == key;
    }
    unsigned m = __ballot_sync(0xffffffffu, hit);
    while (m) {
      int src = __ffs(m) - 1;
      m &= m - 1;
      int ok = 0;
      Snap sn = {};
      if (lane == src) {
        SlotDesc* s = &ring[i];
        sn.state = ld_acquire_sys(&s->state);
        sn.key = ld_relaxed_sys(&s->key);
        sn.addr = ld_relaxed_sys(&s->addr);
        sn.bytes = ld_relaxed_sys(&s->bytes);
        sn.done_addr = ld_relaxed_sys(&s->done_addr);
        sn.done_val = ld_relaxed_sys(&s->done_val);
        fence_acq_rel_sys();
        uint64_t st2 = ld_relaxed_sys(&s->state);
        ok = (sn.state == st2) && ((sn.state & 0xff) == ST_POSTED) && sn.key == key;
      }
      ok = __shfl_sync(0xffffffffu, ok, src);
      if (ok) {
        out->state = __shfl_sync(0xffffffffu, sn.state, src);
        out->key = __shfl_sync(0xffffffffu, sn.key, src);
        out->addr = __shfl_sync(0xffffffffu, sn.addr, src);
        out->bytes = __shfl_sync(0xffffffffu, sn.bytes, src);
        out->done_addr = __shfl_sync(0xffffffffu, sn.done_addr, src);
        out->done_val = __shfl_sync(0xffffffffu, sn.done_val, src);
        return base + src;
      }
    }
  }
  return -1;
}

// Completion stores performed (in order, st.release.sys) after the copy.
struct Fin {
  uint32_t n;
  uint64_t addr[8];
  uint64_t val[8];
  __device__ void add(void* a, uint64_t v) {
    if (a) {
      addr[n] = (uint64_t)a;
      val[n] = v;
      ++n;
    }
  }
  __device__ void run() const {
    fence_sc_sys();
    for (uint32_t k = 0; k < n; ++k) st_release_sys(reinterpret_cast<uint64_t*>(addr[k]), val[k]);
  }
};

struct Decision {
  uint64_t action;
  uint64_t src, dst, bytes;
  Fin fin;
  int wait_own;  // NONE + blocking receive: CTA 0 waits for my_done
  int err;
};

__device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Posts my descriptor into post_ring[pseq % R] after the slot's previous
// occupant is gone. Called by lane 0 of warp 0.
__device__ bool post_desc(const P2PArgs& a, uint64_t addr, uint64_t bytes, uint64_t done_addr,
                          uint64_t done_val) {
  const int slot = (int)(a.pseq % (uint64_t)a.R);
  SlotDesc* d = &a.post_ring[slot];
  st_relaxed_sys(&d->key, a.key);
  st_relaxed_sys(&d->addr, addr);
  st_relaxed_sys(&d->bytes, bytes);
  st_relaxed_sys(&d->done_addr, done_addr);
  st_relaxed_sys(&d->done_val, done_val);
  fence_sc_sys();  // payload (eager/staged) and fields before the state
  st_release_sys(&d->state, st_word(a.pseq, ST_POSTED));
  fence_sc_sys();  // Dekker: my post is visible before I rescan
  return true;
}

__device__ bool wait_post_slot(const P2PArgs& a) {
  const int slot = (int)(a.pseq % (uint64_t)a.R);
  uint64_t need = a.pseq >= (uint64_t)a.R ? a.pseq - a.R + 1 : 0;
  if (need == 0) return true;
  return spin_ge(&a.post_mirror[slot], need, a.err_word, a.spin_limit_ns, ERRW_WAIT_SLOT);
}

// Send: my descriptor (if posted) at post_ring[slot]; the matched receive at
// scan_ring[j] (snapshot r). Fills the push decision.
__device__ void send_win(const P2PArgs& a, Decision& dc, int j, const Snap& r, bool posted,
                         const uint8_t* src) {
  const uint64_t rpseq = r.state >> 8;
  const int slot = (int)(a.pseq % (uint64_t)a.R);
  dc.action = ACT_COPY;
  dc.src = (uint64_t)src;
  dc.dst = r.addr;
  dc.bytes = umin(a.bytes, r.bytes);  // truncation: endpoint.cpp:17
  dc.fin.n = 0;
  dc.fin.add(&a.scan_ring[j].state, st_word(rpseq, ST_FREE));
  if (posted) dc.fin.add(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));
  dc.fin.add(&a.scan_mirror[j], rpseq + 1);
  if (posted) dc.fin.add(&a.post_mirror[slot], a.pseq + 1);
  dc.fin.add(reinterpret_cast<void*>(r.done_addr), r.done_val);
  dc.fin.add(a.my_done, a.my_gen);
  if (a.mode == MODE_STAGED) dc.fin.add(a.stage_done, a.stage_gen);
}

// Receive: the matched send at scan_ring[j] (snapshot s, already TAKEN by me).
__device__ void recv_win(const P2PArgs& a, Decision& dc, int j, const Snap& s, bool posted) {
  const uint64_t spseq = s.state >> 8;
  const int slot = (int)(a.pseq % (uint64_t)a.R);
  dc.action = ACT_COPY;
  dc.src = s.addr;
  dc.dst = (uint64_t)a.buf;
  dc.bytes = umin(s.bytes, a.bytes);
  dc.fin.n = 0;
  dc.fin.add(&a.scan_ring[j].state, st_word(spseq, ST_FREE));
  if (posted) dc.fin.add(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));
  dc.fin.add(&a.scan_mirror[j], spseq + 1);
  if (posted) dc.fin.add(&a.post_mirror[slot], a.pseq + 1);
  dc.fin.add(reinterpret_cast<void*>(s.done_addr), s.done_val);
  dc.fin.add(a.my_done, a.my_gen);
}

// Phase 1 (CTA 0). All threads of CTA 0 call it; warp 0 does the protocol,
// the whole CTA does the eager payload copy.
__device__ void decide(const P2PArgs& a, Decision& dc) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  __shared__ int s_phase;  // 0 = decided, 1 = need eager copy
  if (warp == 0) {
    Snap sn;
    int j = warp_scan(a.scan_ring, a.R, a.key, &sn);
    if (lane == 0) {
      dc.err = 0;
      dc.wait_own = 0;
      dc.fin.n = 0;
      if (!a.is_recv) {
        if (j >= 0) {
          send_win(a, dc, j, sn, false, a.buf);  // receive already posted: push
          s_phase = 0;
        } else if (a.mode == MODE_STAGED) {
          dc.action = ACT_STAGE;  // copy to local staging first (all CTAs)
          s_phase = 0;
        } else if (!wait_post_slot(a)) {
          dc.action = ACT_NONE;
          dc.err = 1;
          s_phase = 0;
        } else if (a.mode == MODE_EAGER) {
          s_phase = 1;
        } else {  // MODE_ISEND: publish the user buffer
          post_desc(a, (uint64_t)a.buf, a.bytes, (uint64_t)a.my_done, a.my_gen);
          s_phase = 2;
        }
      } else {
        if (j >= 0) {
          uint64_t want = st_word(sn.state >> 8, ST_POSTED);
          uint64_t old = cas_sys(&a.scan_ring[j].state, want, st_word(sn.state >> 8, ST_TAKEN));
          if (old == want) {
            recv_win(a, dc, j, sn, false);
          } else {
            dc.action = ACT_NONE;  // impossible: nobody else can take it
            dc.err = 1;
            if (a.err_word) st_relaxed_sys(a.err_word, ERRW_PROTOCOL);
          }
          s_phase = 0;
        } else if (!wait_post_slot(a)) {
          dc.action = ACT_NONE;
          dc.err = 1;
          s_phase = 0;
        } else {
          post_desc(a, (uint64_t)a.buf, a.bytes, (uint64_t)a.my_done, a.my_gen);
          s_phase = 2;
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  int phase = s_phase;
  if (phase == 1) {
    // Eager: payload into the receiver's eager slot (remote stores).
    const int slot = (int)(a.pseq % (uint64_t)a.R);
    part_copy(a.eager_ring + (uint64_t)slot * a.E, a.buf, a.bytes, 0, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      post_desc(a, (uint64_t)(a.eager_ring + (uint64_t)slot * a.E), a.bytes, 0, 0);
      s_phase = 2;
    }
    __syncthreads();
    phase = 2;
  }
  if (phase == 2) {
    // Posted: rescan; if the other side's descriptor is there, race for the
    // send descriptor's state word.
    if (warp == 0) {
      Snap sn;
      int j = warp_scan(a.scan_ring, a.R, a.key, &sn);
      if (lane == 0) {
        dc.action = ACT_NONE;
        if (j >= 0) {
          if (!a.is_recv) {
            const int slot = (int)(a.pseq % (uint64_t)a.R);
            uint64_t want = st_word(a.pseq, ST_POSTED);
            if (cas_sys(&a.post_ring[slot].state, want, st_word(a.pseq, ST_TAKEN)) == want)
              send_win(a, dc, j, sn, true, a.buf);
          } else {
            uint64_t want = st_word(sn.state >> 8, ST_POSTED);
            if (cas_sys(&a.scan_ring[j].state, want, st_word(sn.state >> 8, ST_TAKEN)) == want)
              recv_win(a, dc, j, sn, true);
          }
        }
        if (dc.action == ACT_NONE && a.is_recv && a.blocking) dc.wait_own = 1;
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 2) k_p2p(const P2PArgs a) {
  __shared__ Decision s_dc;
  __shared__ int s_last;
  const bool multi = gridDim.x > 1;
  OpRecord* rec = a.rec;

  if (blockIdx.x == 0) {
    decide(a, s_dc);
    if (multi && threadIdx.x == 0) {
      rec->action = s_dc.action;
      rec->src = s_dc.src;
      rec->dst = s_dc.dst;
      rec->bytes = s_dc.bytes;
      rec->counter = 0;
      rec->nfin = s_dc.fin.n;
      for (uint32_t k = 0; k < s_dc.fin.n; ++k) {
        rec->fin_addr[k] = s_dc.fin.addr[k];
        rec->fin_val[k] = s_dc.fin.val[k];
      }
      __threadfence();
      st_release_gpu(&rec->opid, a.opid);
    }
  } else {
    if (threadIdx.x == 0) {
      unsigned ns = 32;
      while (ld_acquire_gpu(&rec->opid) != a.opid) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
      s_dc.action = rec->action;
      s_dc.src = rec->src;
      s_dc.dst = rec->dst;
      s_dc.bytes = rec->bytes;
      s_dc.fin.n = rec->nfin;
      for (uint32_t k = 0; k < s_dc.fin.n; ++k) {
        s_dc.fin.addr[k] = rec->fin_addr[k];
        s_dc.fin.val[k] = rec->fin_val[k];
      }
      s_dc.wait_own = 0;
    }
    __syncthreads();
  }

  const uint64_t action = s_dc.action;
  if (action == ACT_NONE) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && s_dc.wait_own)
      spin_ge(a.my_done, a.my_gen, a.err_word, a.spin_limit_ns, ERRW_WAIT_DONE);
    return;
  }

  if (action == ACT_COPY) {
    part_copy(reinterpret_cast<uint8_t*>(s_dc.dst), reinterpret_cast<const uint8_t*>(s_dc.src),
              s_dc.bytes, blockIdx.x, gridDim.x);
  } else {  // ACT_STAGE: user buffer -> local staging
    part_copy(a.staging, a.buf, a.bytes, blockIdx.x, gridDim.x);
  }

  // Grid completion: the last CTA finishes the operation.
  __syncthreads();
  if (threadIdx.x == 0) {
    if (multi) {
      __threadfence_system();
      unsigned old = atomicAdd(&rec->counter, 1u);
      s_last = (old == gridDim.x - 1);
      if (s_last) __threadfence_system();
    } else {
      s_last = 1;
    }
  }
  __syncthreads();
  if (!s_last) return;

  if (action == ACT_COPY) {
    if (threadIdx.x == 0) s_dc.fin.run();
    return;
  }

  // ACT_STAGE, last CTA: publish the staged copy, rescan, maybe push.
  __shared__ int s_push;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      s_push = 0;
      if (wait_post_slot(a)) {
        post_desc(a, (uint64_t)a.staging, a.bytes, (uint64_t)a.stage_done, a.stage_gen);
      } else {
        s_push = -1;
      }
    }
    __syncwarp();
    int ok = __shfl_sync(0xffffffffu, s_push, 0);
    if (ok == 0) {
      Snap sn;
      int j = warp_scan(a.scan_ring, a.R, a.key, &sn);
      if (threadIdx.x == 0 && j >= 0) {
        const int slot = (int)(a.pseq % (uint64_t)a.R);
        uint64_t want = st_word(a.pseq, ST_POSTED);
        if (cas_sys(&a.post_ring[slot].state, want, st_word(a.pseq, ST_TAKEN)) == want) {
          send_win(a, s_dc, j, sn, true, a.staging);
          s_push = 1;
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_push == 1) {
    part_copy(reinterpret_cast<uint8_t*>(s_dc.dst), reinterpret_cast<const uint8_t*>(s_dc.src),
              s_dc.bytes, 0, 1);
    __syncthreads();
    if (threadIdx.x == 0) s_dc.fin.run();
  }
}

// ---------------------------------------------------------------------------
// Wait / Waitall
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32) k_wait(const WaitArgs a) {
  for (int i = threadIdx.x; i < a.n; i += 32) {
    if (!spin_ge(a.e[i].flag, a.e[i].gen, a.err_word, a.spin_limit_ns, ERRW_WAIT_DONE)) break;
  }
}

// ---------------------------------------------------------------------------
// Allreduce
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t f2bf_rne(float f) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f));
}

template <int OP>
__device__ __forceinline__ float opf(float a, float b) {
  if (OP == AR_SUM) return __fadd_rn(a, b);
  if (OP == AR_MAX) return b > a ? b : a;
  return b < a ? b : a;
}
template <int OP>
__device__ __forceinline__ double opd(double a, double b) {
  if (OP == AR_SUM) return __dadd_rn(a, b);
  if (OP == AR_MAX) return b > a ? b : a;
  return b < a ? b : a;
}
template <int OP>
__device__ __forceinline__ int32_t opi(int32_t a, int32_t b) {
  if (OP == AR_SUM) return (int32_t)((uint32_t)a + (uint32_t)b);
  if (OP == AR_MAX) return b > a ? b : a;
  return b < a ? b : a;
}

// Accumulator for one 16-B vector.
template <int DT>
struct Acc;
template <>
struct Acc<AR_F32> {
  float v[4];
  __device__ void init(const uint4& x) {
    v[0] = __uint_as_float(x.x); v[1] = __uint_as_float(x.y);
    v[2] = __uint_as_float(x.z); v[3] = __uint_as_float(x.w);
  }
  template <int OP>
  __device__ void add(const uint4& x) {
    v[0] = opf<OP>(v[0], __uint_as_float(x.x)); v[1] = opf<OP>(v[1], __uint_as_float(x.y));
    v[2] = opf<OP>(v[2], __uint_as_float(x.z)); v[3] = opf<OP>(v[3], __uint_as_float(x.w));
  }
  __device__ uint4 out() const {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
};
template <>
struct Acc<AR_BF16> {
  float v[8];
  __device__ void init(const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[2 * k] = bf16_lo(w[k]); v[2 * k + 1] = bf16_hi(w[k]); }
  }
  template <int OP>
  __device__ void add(const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[2 * k] = opf<OP>(v[2 * k], bf16_lo(w[k]));
      v[2 * k + 1] = opf<OP>(v[2 * k + 1], bf16_hi(w[k]));
    }
  }
  __device__ uint4 out() const {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = f2bf_rne(v[2 * k]) | (f2bf_rne(v[2 * k + 1]) << 16);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Acc<AR_I32> {
  int32_t v[4];
  __device__ void init(const uint4& x) {
    v[0] = (int32_t)x.x; v[1] = (int32_t)x.y; v[2] = (int32_t)x.z; v[3] = (int32_t)x.w;
  }
  template <int OP>
  __device__ void add(const uint4& x) {
    v[0] = opi<OP>(v[0], (int32_t)x.x); v[1] = opi<OP>(v[1], (int32_t)x.y);
    v[2] = opi<OP>(v[2], (int32_t)x.z); v[3] = opi<OP>(v[3], (int32_t)x.w);
  }
  __device__ uint4 out() const {
    return make_uint4((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3]);
  }
};
template <>
struct Acc<AR_F64> {
  double v[2];
  __device__ void init(const uint4& x) {
    v[0] = __hiloint2double((int)x.y, (int)x.x);
    v[1] = __hiloint2double((int)x.w, (int)x.z);
  }
  template <int OP>
  __device__ void add(const uint4& x) {
    v[0] = opd<OP>(v[0], __hiloint2double((int)x.y, (int)x.x));
    v[1] = opd<OP>(v[1], __hiloint2double((int)x.w, (int)x.z));
  }
  __device__ uint4 out() const {
    return make_uint4((uint32_t)__double2loint(v[0]), (uint32_t)__double2hiint(v[0]),
                      (uint32_t)__double2loint(v[1]), (uint32_t)__double2hiint(v[1]));
  }
};

// Scalar element fold (unaligned buffers and tails).
template <int DT, int OP>
__device__ void reduce_elem(const uint64_t* sb, uint8_t* const* outs, int nout, int P,
                            uint64_t e) {
  if (DT == AR_F32 || DT == AR_BF16) {
    float acc = 0.f;
    for (int q = 0; q < P; ++q) {
      float x;
      if (DT == AR_F32) {
        x = reinterpret_cast<const float*>(sb[q])[e];
      } else {
        uint16_t h = reinterpret_cast<const uint16_t*>(sb[q])[e];
        x = __uint_as_float((uint32_t)h << 16);
      }
      acc = q == 0 ? x : opf<OP>(acc, x);
    }
    for (int o = 0; o < nout; ++o) {
      if (DT == AR_F32) reinterpret_cast<float*>(outs[o])[e] = acc;
      else reinterpret_cast<uint16_t*>(outs[o])[e] = (uint16_t)f2bf_rne(acc);
    }
  } else if (DT == AR_I32) {
    int32_t acc = 0;
    for (int q = 0; q < P; ++q) {
      int32_t x = reinterpret_cast<const int32_t*>(sb[q])[e];
      acc = q == 0 ? x : opi<OP>(acc, x);
    }
    for (int o = 0; o < nout; ++o) reinterpret_cast<int32_t*>(outs[o])[e] = acc;
  } else {
    double acc = 0.0;
    for (int q = 0; q < P; ++q) {
      double x = reinterpret_cast<const double*>(sb[q])[e];
      acc = q == 0 ? x : opd<OP>(acc, x);
    }
    for (int o = 0; o < nout; ++o) reinterpret_cast<double*>(outs[o])[e] = acc;
  }
}

// Vector range [v0, v1) of 16-B vectors, grid-stride over (part, nparts).
template <int DT, int OP, int UNROLL>
__device__ void reduce_range(const uint64_t* sb, uint8_t* const* outs, int nout, int P,
                             uint64_t v0, uint64_t v1, uint64_t t, uint64_t nt) {
  uint64_t i = v0 + t;
  for (; i + (UNROLL - 1) * nt < v1; i += UNROLL * nt) {
    Acc<DT> acc[UNROLL];
    {
      const uint4* s0 = reinterpret_cast<const uint4*>(sb[0]);
      uint4 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) x[u] = s0[i + u * nt];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc[u].init(x[u]);
    }
    for (int q = 1; q < P; ++q) {
      const uint4* sq = reinterpret_cast<const uint4*>(sb[q]);
      uint4 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) x[u] = sq[i + u * nt];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc[u].template add<OP>(x[u]);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      uint4 o = acc[u].out();
      for (int k = 0; k < nout; ++k) reinterpret_cast<uint4*>(outs[k])[i + u * nt] = o;
    }
  }
  for (; i < v1; i += nt) {
    Acc<DT> acc;
    acc.init(reinterpret_cast<const uint4*>(sb[0])[i]);
    for (int q = 1; q < P; ++q) acc.template add<OP>(reinterpret_cast<const uint4*>(sb[q])[i]);
    uint4 o = acc.out();
    for (int k = 0; k < nout; ++k) reinterpret_cast<uint4*>(outs[k])[i] = o;
  }
}

template <int DT, int OP>
__device__ void ar_compute(const ARArgs& a, const uint64_t* sb, const uint64_t* rb, int algo) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  const int P = a.P;
  const uint64_t nbytes = a.count * (uint64_t)a.esize;
  bool aligned = true;
  for (int q = 0; q < P; ++q) aligned &= ((sb[q] | rb[q]) & 15) == 0;
  uint8_t* outs[kMaxCollRanks];
  if (!aligned) {
    // Scalar path: every element on its owner (two-shot) or locally.
    if (algo == AR_TWOSHOT) {
      for (int q = 0; q < P; ++q) outs[q] = reinterpret_cast<uint8_t*>(rb[q]);
      uint64_t per = (a.count + P - 1) / P;
      uint64_t e0 = per * a.me, e1 = umin(a.count, e0 + per);
      for (uint64_t e = e0 + t; e < e1; e += nt) reduce_elem<DT, OP>(sb, outs, P, P, e);
    } else {
      outs[0] = reinterpret_cast<uint8_t*>(rb[a.me]);
      for (uint64_t e = t; e < a.count; e += nt) reduce_elem<DT, OP>(sb, outs, 1, P, e);
    }
    return;
  }
  const uint64_t nvec = nbytes >> 4;
  const uint64_t tail_e0 = (nvec << 4) / a.esize;  // first element not in a vector
  if (algo == AR_TWOSHOT) {
    for (int q = 0; q < P; ++q) outs[q] = reinterpret_cast<uint8_t*>(rb[q]);
    uint64_t per = (nvec + P - 1) / P;
    uint64_t v0 = umin(nvec, per * a.me), v1 = umin(nvec, v0 + per);
    reduce_range<DT, OP, 4>(sb, outs, P, P, v0, v1, t, nt);
    if (a.me == P - 1)
      for (uint64_t e = tail_e0 + t; e < a.count; e += nt) reduce_elem<DT, OP>(sb, outs, P, P, e);
  } else {
    outs[0] = reinterpret_cast<uint8_t*>(rb[a.me]);
    reduce_range<DT, OP, 4>(sb, outs, 1, P, 0, nvec, t, nt);
    for (uint64_t e = tail_e0 + t; e < a.count; e += nt) reduce_elem<DT, OP>(sb, outs, 1, P, e);
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_allreduce(const ARArgs a) {
  __shared__ uint64_t s_sb[kMaxCollRanks], s_rb[kMaxCollRanks];
  __shared__ int s_algo, s_ok, s_last;
  const int P = a.P;
  const bool multi = gridDim.x > 1;
  OpRecord* rec = a.rec;

  if (blockIdx.x == 0) {
    if (threadIdx.x < 32) {
      const int q = threadIdx.x;
      int ok = 1;
      if (P > 1) {
        // Entry: publish my buffers to every peer, then wait for theirs.
        if (q < P) {
          CollSlot* dst = a.peer_in[q];
          st_relaxed_sys(&dst->sbuf, (uint64_t)a.sbuf);
          st_relaxed_sys(&dst->rbuf, (uint64_t)a.rbuf);
          fence_sc_sys();
          st_release_sys(&dst->flag, a.epoch);
        }
        if (q < P) {
          ok = spin_ge(&a.my_in[q].flag, a.epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL);
          s_sb[q] = ld_relaxed_sys(&a.my_in[q].sbuf);
          s_rb[q] = ld_relaxed_sys(&a.my_in[q].rbuf);
        }
      } else if (q == 0) {
        s_sb[0] = (uint64_t)a.sbuf;
        s_rb[0] = (uint64_t)a.rbuf;
      }
      ok = __all_sync(0xffffffffu, ok);
      __syncwarp();
      if (q == 0) {
        int algo = a.algo;
        // One-shot reads every peer's full buffer while peers write theirs:
        // unsafe if any rank reduces in place.
        for (int k = 0; k < P; ++k)
          if (s_sb[k] == s_rb[k] && P > 1) algo = AR_TWOSHOT;
        s_algo = algo;
        s_ok = ok;
      }
    }
    __syncthreads();
    if (multi && threadIdx.x == 0) {
      for (int k = 0; k < P; ++k) {
        rec->coll[k] = s_sb[k];
        rec->coll[kMaxCollRanks + k] = s_rb[k];
      }
      rec->action = s_ok ? (uint64_t)s_algo + 1 : 0;
      rec->counter = 0;
      __threadfence();
      st_release_gpu(&rec->opid, a.opid);
    }
  } else {
    if (threadIdx.x == 0) {
      unsigned ns = 32;
      while (ld_acquire_gpu(&rec->opid) != a.opid) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
      for (int k = 0; k < P; ++k) {
        s_sb[k] = rec->coll[k];
        s_rb[k] = rec->coll[kMaxCollRanks + k];
      }
      uint64_t act = rec->action;
      s_ok = act != 0;
      s_algo = act ? (int)act - 1 : 0;
    }
    __syncthreads();
  }
  if (!s_ok) return;

  const int algo = s_algo;
#define AR_DISPATCH(DT)                                             \
  if (a.op == AR_SUM) ar_compute<DT, AR_SUM>(a, s_sb, s_rb, algo);  \
  else if (a.op == AR_MAX) ar_compute<DT, AR_MAX>(a, s_sb, s_rb, algo); \
  else ar_compute<DT, AR_MIN>(a, s_sb, s_rb, algo);
  switch (a.dtype) {
    case AR_F32: AR_DISPATCH(AR_F32) break;
    case AR_BF16: AR_DISPATCH(AR_BF16) break;
    case AR_I32: AR_DISPATCH(AR_I32) break;
    default: AR_DISPATCH(AR_F64) break;
  }
#undef AR_DISPATCH

  if (P == 1) return;
  // Exit: every CTA done -> tell every peer; wait for all peers.
  __syncthreads();
  if (threadIdx.x == 0) {
    if (multi) {
      __threadfence_system();
      unsigned old = atomicAdd(&rec->counter, 1u);
      s_last = (old == gridDim.x - 1);
      if (s_last) __threadfence_system();
    } else {
      s_last = 1;
      __threadfence_system();
    }
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x < 32) {
    const int q = threadIdx.x;
    if (q < P) st_release_sys(a.peer_exit[q], a.epoch);
    if (q < P) spin_ge(&a.my_exit[q], a.epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL);
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
cudaError_t launch_p2p(const P2PArgs& a, int grid, cudaStream_t s) {
  k_p2p<<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_wait(const WaitArgs& a, cudaStream_t s) {
  k_wait<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_allreduce(const ARArgs& a, int grid, cudaStream_t s) {
  k_allreduce<<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

int p2p_occupancy() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_p2p, kThreads, 0) != cudaSuccess) n = 1;
  return n > 0 ? n : 1;
}

int allreduce_occupancy() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_allreduce, kThreads, 0) != cudaSuccess)
    n = 1;
  return n > 0 ? n : 1;
}

}  // namespace mpix
