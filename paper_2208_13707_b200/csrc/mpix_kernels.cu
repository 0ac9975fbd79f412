// mpix_kernels.cu — sm_100a kernels of the MPIX-stream GPU-enqueue path.
//
// Point-to-point (Send/Isend/Recv/Irecv_enqueue). Replaces the reference's
// queue worker running post_send/post_recv/wait closures
// (proj/src/proc_enqueue.cpp:30-114, proj/src/proc_p2p.cpp:27-94) and its
// matching/progress engine (proj/src/endpoint.cpp:15-69,
// proj/src/fabric.cpp:93-110):
//
//   k_proto  1 CTA. Warp 0 runs the handshake on the descriptor rings in
//            peer-mapped memory (scan, post, fence, rescan, CAS). Messages up
//            to the inline limit are also copied and completed here, so a
//            small message costs exactly one launch.
//   k_copy   large messages only; launched with programmatic dependent launch
//            right behind k_proto, never spins: every CTA reads the decision
//            and streams one 64-KiB tile (128-bit loads/stores, 4 in flight
//            per thread), push to or pull from the peer's buffer.
//   k_fin    1 CTA, PDL: completion stores (slot frees, free-mirrors, done
//            words) after the whole copy grid retired; publishes staged
//            blocking sends.
//   k_batch  coalesced launch: the inline operations enqueued on a stream
//            since its last launch (one CTA each) plus the Wait/Waitall or
//            blocking operation that closed the batch.
//
// Allreduce_enqueue (no reference): k_ar_entry (1 CTA: publish buffers,
// wait for every peer) -> k_ar_reduce (wide, rank-ordered fold, one-shot or
// two-shot over peer pointers) -> k_ar_exit (1 CTA: exit barrier).
//
// Only 1-CTA kernels ever spin, so any number of ranks sharing a GPU (and
// the user's own streams) always make progress.
//
// Scope: every primitive is templated on SYS. Ranks on the same GPU use
// .gpu scope (fence ~0.2 us); ranks on different GPUs use .sys scope
// (fence/release/CAS ~1.7-1.9 us on B200, tools/copybench.cu), so the
// protocol keeps system-scope fences to two per side on the critical path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#include "mpix_internal.h"

namespace mpix {

// ---------------------------------------------------------------------------
// Scoped memory primitives
// ---------------------------------------------------------------------------
#define MPIX_DEFINE_SCOPE(NAME, SC)                                                               \
  struct NAME {                                                                                   \
    static __device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {                        \
      uint64_t v;                                                                                 \
      asm volatile("ld.acquire." SC ".global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");     \
      return v;                                                                                   \
    }                                                                                             \
    static __device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) {                        \
      uint64_t v;                                                                                 \
      asm volatile("ld.relaxed." SC ".global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");     \
      return v;                                                                                   \
    }                                                                                             \
    static __device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {                      \
      asm volatile("st.release." SC ".global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");       \
    }                                                                                             \
    static __device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) {                      \
      asm volatile("st.relaxed." SC ".global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");       \
    }                                                                                             \
    static __device__ __forceinline__ uint64_t cas(uint64_t* p, uint64_t c, uint64_t v) {         \
      uint64_t o;                                                                                 \
      asm volatile("atom.acq_rel." SC ".global.cas.b64 %0, [%1], %2, %3;"                       \
                   : "=l"(o)                                                                      \
                   : "l"(p), "l"(c), "l"(v)                                                       \
                   : "memory");                                                                   \
      return o;                                                                                   \
    }                                                                                             \
    static __device__ __forceinline__ uint64_t cas_acq(uint64_t* p, uint64_t c, uint64_t v) {     \
      uint64_t o;                                                                                 \
      asm volatile("atom.acquire." SC ".global.cas.b64 %0, [%1], %2, %3;"                       \
                   : "=l"(o)                                                                      \
                   : "l"(p), "l"(c), "l"(v)                                                       \
                   : "memory");                                                                   \
      return o;                                                                                   \
    }                                                                                             \
    static __device__ __forceinline__ uint64_t exch(uint64_t* p, uint64_t v) {                  \
      uint64_t o;                                                                                 \
      asm volatile("atom.relaxed." SC ".global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory"); \
      return o;                                                                                   \
    }                                                                                             \
    static __device__ __forceinline__ void fence_sc() { asm volatile("fence.sc." SC ";" ::: "memory"); } \
    static __device__ __forceinline__ void fence_ar() {                                           \
      asm volatile("fence.acq_rel." SC ";" ::: "memory");                                        \
    }                                                                                             \
  };
MPIX_DEFINE_SCOPE(ScopeSys, "sys")
MPIX_DEFINE_SCOPE(ScopeGpu, "gpu")
#undef MPIX_DEFINE_SCOPE

template <bool SYS>
struct Scope;
template <>
struct Scope<true> : ScopeSys {};
template <>
struct Scope<false> : ScopeGpu {};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// Spin until *p >= target. Returns false on watchdog expiry after recording
// `code` in the rank's host-mapped error word (the kernel then exits rather
// than hanging the GPU).
// Polls with relaxed loads (an acquire load invalidates the SM's L1 on every
// poll — the stacks and cached reads of every CTA on the SM with it) and
// orders what follows with one acquire load once the value is there.
template <bool SYS>
__device__ __noinline__ bool spin_ge(const uint64_t* p, uint64_t target, uint64_t* err_word,
                                     uint64_t limit_ns, uint64_t code) {
  using M = Scope<SYS>;
  if (M::ld_acq(p) >= target) return true;
  uint64_t t0 = limit_ns ? globaltimer() : 0;
  unsigned ns = 32;
  while (M::ld_rlx(p) < target) {
    __nanosleep(ns);
    if (ns < 64) ns <<= 1;  // short cap: the poll's own round trip dominates (256: +0.3-0.5 us latency)
    if (limit_ns && globaltimer() - t0 > limit_ns) {
      if (err_word) ScopeSys::st_rlx(err_word, code);
      return false;
    }
  }
  (void)M::ld_acq(p);  // acquire: what the writer released is visible from here
  return true;
}

__device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }

constexpr uint64_t kPollMaxBytes = 65536;  // blocking receives up to this capacity poll (§3c)

// Ring slot of a pair sequence. A 64-bit modulo is a software division
// (a call of ~150 cycles, and the handshake needs several per operation);
// the default ring sizes are powers of two, so it is a mask.
__device__ __forceinline__ int ring_slot(uint64_t pseq, int R) {
  return (R & (R - 1)) == 0 ? (int)(pseq & (uint64_t)(R - 1)) : (int)(pseq % (uint64_t)R);
}

// Phase stamps (globaltimer ns): one time base for the kernels of every
// rank, so two ranks' phases can be lined up.
__device__ __forceinline__ void trace_t(TraceRec* tr, int k) {
  if (tr) tr->t[k] = globaltimer();
}

// ---------------------------------------------------------------------------
// Copies
// ---------------------------------------------------------------------------
constexpr int kCopyThreads = 1024;
constexpr int kCopyUnroll = 4;  // 64-KiB tiles (tools/copyshape.cu)
constexpr uint64_t kTileVec = (uint64_t)kCopyThreads * kCopyUnroll;  // 16-B vectors per tile

// Whole-CTA copy of n bytes (k_proto inline path and the rare staged push).
__device__ void cta_copy(uint8_t* dst, const uint8_t* src, uint64_t n) {
  if (n == 0 || dst == src) return;
  const uint64_t t = threadIdx.x, nt = blockDim.x;
  uint64_t mis = (uint64_t)dst & 15;
  if ((((uint64_t)src) & 15) != mis) {
    for (uint64_t i = t; i < n; i += nt) dst[i] = src[i];
    return;
  }
  uint64_t head = mis ? umin(16 - mis, n) : 0;
  if (t < head) dst[t] = src[t];
  uint64_t nvec = (n - head) >> 4;
  uint4* d = reinterpret_cast<uint4*>(dst + head);
  const uint4* s = reinterpret_cast<const uint4*>(src + head);
  uint64_t i = t;
  for (; i + 3 * nt < nvec; i += 4 * nt) {
    uint4 v0 = s[i], v1 = s[i + nt], v2 = s[i + 2 * nt], v3 = s[i + 3 * nt];
    d[i] = v0; d[i + nt] = v1; d[i + 2 * nt] = v2; d[i + 3 * nt] = v3;
  }
  for (; i < nvec; i += nt) d[i] = s[i];
  uint64_t done = head + (nvec << 4);
  if (t < n - done) dst[done + t] = src[done + t];
}

// One tile of a grid-wide copy: CTA `tile` moves vectors
// [tile*kTileVec, (tile+1)*kTileVec) after the co-aligned head; extra tiles
// (grid sized from a receive capacity larger than the message) loop nothing.
__device__ __forceinline__ void tile_copy(uint8_t* dst, const uint8_t* src, uint64_t n,
                                          uint64_t tile, uint64_t ntiles) {
  if (n == 0 || dst == src) return;
  uint64_t mis = (uint64_t)dst & 15;
  if ((((uint64_t)src) & 15) != mis) {  // not co-aligned: byte loop over the grid
    uint64_t t = tile * blockDim.x + threadIdx.x, nt = ntiles * blockDim.x;
    for (uint64_t i = t; i < n; i += nt) dst[i] = src[i];
    return;
  }
  uint64_t head = mis ? umin(16 - mis, n) : 0;
  uint64_t nvec = (n - head) >> 4;
  if (tile == 0 && threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
  uint64_t done = head + (nvec << 4);
  if (tile == 0 && threadIdx.x < n - done) dst[done + threadIdx.x] = src[done + threadIdx.x];
  uint4* d = reinterpret_cast<uint4*>(dst + head);
  const uint4* s = reinterpret_cast<const uint4*>(src + head);
  for (uint64_t t = tile; t * kTileVec < nvec; t += ntiles) {
    uint64_t base = t * kTileVec + threadIdx.x;
    if (base + (kCopyUnroll - 1) * kCopyThreads < nvec) {
      uint4 v[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) v[u] = s[base + u * kCopyThreads];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) d[base + u * kCopyThreads] = v[u];
    } else {
      for (int u = 0; u < kCopyUnroll; ++u) {
        uint64_t i = base + u * kCopyThreads;
        if (i < nvec) d[i] = s[i];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Descriptor-ring scan (warp 0). Returns the slot index and a consistent
// snapshot, or -1. Relaxed loads filter; the candidate is validated seqlock
// style (the state word carries the pair sequence, so it never repeats).
// ---------------------------------------------------------------------------
struct Snap {
  uint64_t state, key, addr, bytes, done_addr, done_val, p0, p1;  // p0, p1: an LL post's words
};

template <bool SYS>
__device__ __forceinline__ void ld_pair(const SlotDesc* s, uint64_t& st, uint64_t& key) {
  if (SYS)
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(st), "=l"(key) : "l"(s) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(st), "=l"(key) : "l"(s) : "memory");
}

constexpr int kMaxScanPerLane = 8;  // R <= 256

// Inlined: the snapshot stays in registers (a call would pass it through
// the stack, i.e. local memory, which every acquire's L1 invalidation evicts).
template <bool SYS>
__device__ __forceinline__ int warp_scan(SlotDesc* ring, int R, uint64_t key, Snap* out) {
  using M = Scope<SYS>;
  const int lane = threadIdx.x & 31;
  // Issue every (state, key) load of this lane before looking at any.
  uint64_t st[kMaxScanPerLane], ky[kMaxScanPerLane];
#pragma unroll
  for (int k = 0; k < kMaxScanPerLane; ++k) {
    int i = k * 32 + lane;
    st[k] = 0;
    ky[k] = 0;
    if (i < R) ld_pair<SYS>(&ring[i], st[k], ky[k]);
  }
  uint32_t hits = 0;  // bit k: slot k * 32 + lane is posted with my key
#pragma unroll
  for (int k = 0; k < kMaxScanPerLane; ++k)
    if (k * 32 + lane < R && (st[k] & ~(ST_LL | ST_LLE) & 0xff) == ST_POSTED && ky[k] == key) hits |= 1u << k;
#pragma unroll 1
  for (int k = 0; k < kMaxScanPerLane && k * 32 < R; ++k) {
    unsigned m = __ballot_sync(0xffffffffu, (hits >> k) & 1u);
    while (m) {
      int src = __ffs(m) - 1;
      m &= m - 1;
      int ok = 0;
      Snap sn = {};
      if (lane == src) {
        SlotDesc* s = &ring[k * 32 + lane];
        // an LL post validates its own words (flags), so the scan's relaxed
        // state suffices; any other post's fields are read behind an acquire
        uint64_t stk = 0;
#pragma unroll
        for (int kk = 0; kk < kMaxScanPerLane; ++kk)
          if (kk == k) stk = st[kk];
        sn.state = (stk & ST_LL) ? stk : M::ld_acq(&s->state);
        sn.key = M::ld_rlx(&s->key);
        sn.addr = M::ld_rlx(&s->addr);
        sn.bytes = M::ld_rlx(&s->bytes);
        sn.done_addr = M::ld_rlx(&s->done_addr);
        sn.done_val = M::ld_rlx(&s->done_val);
        sn.p0 = M::ld_rlx(&s->pad[0]);
        sn.p1 = M::ld_rlx(&s->pad[1]);
        // No re-validation: a state moves POSTED(pseq) -> TAKEN -> FREE ->
        // POSTED(pseq + R) only, and the fields change only with a new post,
        // so they belong to this post as long as the state does — which the
        // snapshot's user either proves by CAS on exactly sn.state (taking a
        // send descriptor) or owns (a receive descriptor only its one
        // matching sender reads).
        ok = ((sn.state & ~(ST_LL | ST_LLE) & 0xff) == ST_POSTED) && sn.key == key;
      }
      ok = __shfl_sync(0xffffffffu, ok, src);
      if (ok) {
        out->state = __shfl_sync(0xffffffffu, sn.state, src);
        out->key = __shfl_sync(0xffffffffu, sn.key, src);
        out->addr = __shfl_sync(0xffffffffu, sn.addr, src);
        out->bytes = __shfl_sync(0xffffffffu, sn.bytes, src);
        out->done_addr = __shfl_sync(0xffffffffu, sn.done_addr, src);
        out->done_val = __shfl_sync(0xffffffffu, sn.done_val, src);
        out->p0 = __shfl_sync(0xffffffffu, sn.p0, src);
        out->p1 = __shfl_sync(0xffffffffu, sn.p1, src);
        return k * 32 + src;
      }
    }
  }
  return -1;
}

// Completion stores: group A (slot frees) then group B (free-mirrors and
// done words), a fence before each group. A poster reuses a slot only after
// seeing its mirror, so the FREE state must land first.
struct Fin {
  uint32_t na, nb;
  uint64_t a_addr[2], a_val[2];
  uint64_t b_addr[5], b_val[5];
  // the completed receive's status (its completion word's status planes)
  uint64_t s_addr, s_bytes, s_srctag;
  __device__ void clear() { na = nb = 0; s_addr = 0; }
  __device__ void add_a(void* p, uint64_t v) {
    if (p) { a_addr[na] = (uint64_t)p; a_val[na] = v; ++na; }
  }
  __device__ void add_b(void* p, uint64_t v) {
    if (p) { b_addr[nb] = (uint64_t)p; b_val[nb] = v; ++nb; }
  }
  // deliver's status (endpoint.cpp:17-24): bytes = min(len, cap), truncated = len > cap
  // sidx_enc: the sender's multiplex stream index + 2 (0 = none)
  __device__ void status(void* done, uint64_t len, uint64_t cap, int src, int tag, uint64_t sidx_enc) {
    if (!done) return;
    s_addr = (uint64_t)done;
    s_bytes = (len < cap ? len : cap) | (len > cap ? kTruncBit : 0);
    s_srctag = ((uint64_t)(src & 0xffffff) << 40) | ((sidx_enc & 0xff) << 32) | (uint32_t)tag;
  }
  template <bool SYS>
  // One fence: the payload (written by the whole CTA or grid before this)
  // and the slot frees must both be visible before any mirror or done word;
  // nothing orders the frees against the payload (a freed slot is reused only
  // after its mirror), so group A (and the status) is stored before the fence.
  __device__ void run() const {
    using M = Scope<SYS>;
    if (s_addr) {
      M::st_rlx(reinterpret_cast<uint64_t*>(s_addr + kStatusOff), s_bytes);
      M::st_rlx(reinterpret_cast<uint64_t*>(s_addr + 2 * kStatusOff), s_srctag);
    }
    for (uint32_t k = 0; k < na; ++k) M::st_rlx(reinterpret_cast<uint64_t*>(a_addr[k]), a_val[k]);
    M::fence_ar();
    for (uint32_t k = 0; k < nb; ++k) M::st_rlx(reinterpret_cast<uint64_t*>(b_addr[k]), b_val[k]);
  }
};

struct Decision {
  uint64_t action, src, dst, bytes;
  Fin fin;
  int wait_own;
  int now;  // copy + complete in the deciding CTA even on the split path
  // staged blocking send: the staging buffer and its release word/value
  // (host-provided, or claimed from the rank's device arena)
  uint8_t* stage_ptr;
  uint64_t* stage_done;
  uint64_t stage_gen;
  // ACT_LLE: a taken LL-eager send (src = its eager slot of LL words, dst =
  // my buffer, bytes = what I keep); completed by the CTA after the copy
  uint64_t lle_len, lle_spseq, lle_key, lle_gate, lle_sgen;
  uint64_t* lle_sdone;
  int lle_j, lle_posted;
};

template <bool SYS>
__device__ void post_desc(const P2PArgs& a, uint64_t addr, uint64_t bytes, uint64_t done_addr,
                          uint64_t done_val, bool others_wrote) {
  using M = Scope<SYS>;
  const int slot = ring_slot(a.pseq, a.R);
  SlotDesc* d = &a.post_ring[slot];
  M::st_rlx(&d->key, a.key);
  M::st_rlx(&d->addr, addr);
  M::st_rlx(&d->bytes, bytes);
  M::st_rlx(&d->done_addr, done_addr);
  M::st_rlx(&d->done_val, done_val);
  // Payload written by other threads of the CTA (others_wrote): ordered by
  // the CTA barrier before this call plus the release store's fence (one
  // MEMBAR; a separate fence here would emit a second).
  (void)others_wrote;
  M::st_rel(&d->state, st_word(a.pseq, ST_POSTED));
  M::fence_sc();  // Dekker: my post is visible before I rescan
}

template <bool SYS>
__device__ bool wait_post_slot(const P2PArgs& a, uint64_t prefetched = 0) {
  const int slot = ring_slot(a.pseq, a.R);
  uint64_t need = a.pseq >= (uint64_t)a.R ? a.pseq - a.R + 1 : 0;
  if (need == 0 || prefetched >= need) return true;
  return spin_ge<SYS>(&a.post_mirror[slot], need, a.err_word, a.spin_limit_ns, ERRW_WAIT_SLOT);
}

// Sender wins: push src -> receiver's buffer.
__device__ void send_win(const P2PArgs& a, Decision& dc, int j, const Snap& r, bool posted,
                         const uint8_t* src) {
  const uint64_t rpseq = r.state >> 8;
  const int slot = ring_slot(a.pseq, a.R);
  dc.action = ACT_COPY;
  dc.src = (uint64_t)src;
  dc.dst = r.addr;
  dc.bytes = umin(a.bytes, r.bytes);  // truncation: endpoint.cpp:17
  dc.fin.clear();
  dc.fin.add_a(&a.scan_ring[j].state, st_word(rpseq, ST_FREE));
  if (posted) dc.fin.add_a(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));
  dc.fin.add_b(&a.scan_mirror[j], rpseq + 1);
  // My slot pseq % R is consumed either way (posted, or skipped by the
  // fast path after its previous occupant retired): advance its mirror.
  dc.fin.add_b(&a.post_mirror[slot], a.pseq + 1);
  dc.fin.add_b(reinterpret_cast<void*>(r.done_addr), r.done_val);
  dc.fin.add_b(a.my_done, a.my_gen);
  if (a.mode == MODE_STAGED && dc.stage_done) dc.fin.add_b(dc.stage_done, dc.stage_gen);
  dc.fin.status(reinterpret_cast<void*>(r.done_addr), a.bytes, r.bytes, a.me, (int)(a.key >> 32),
                (uint64_t)(a.sidx + 2));
}

// Receiver wins (send descriptor already TAKEN by me): pull.
__device__ void recv_win(const P2PArgs& a, Decision& dc, int j, const Snap& s, bool posted) {
  const uint64_t spseq = s.state >> 8;
  const int slot = ring_slot(a.pseq, a.R);
  dc.action = ACT_COPY;
  dc.src = s.addr;
  dc.dst = (uint64_t)a.buf;
  dc.bytes = umin(s.bytes, a.bytes);
  dc.fin.clear();
  dc.fin.add_a(&a.scan_ring[j].state, st_word(spseq, ST_FREE));
  if (posted) dc.fin.add_a(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));
  dc.fin.add_b(&a.scan_mirror[j], spseq + 1);
  dc.fin.add_b(&a.post_mirror[slot], a.pseq + 1);  // consumed either way
  dc.fin.add_b(reinterpret_cast<void*>(s.done_addr), s.done_val);
  dc.fin.add_b(a.my_done, a.my_gen);
  dc.fin.status(a.my_done, s.bytes, a.bytes, a.peer, (int)(s.key >> 32), (uint64_t)(a.sidx + 2));
}

// Claim a slot of the rank's device staging arena (warp 0, all lanes). A
// slot's state word is even when free; the claimer moves v -> v+1 and the
// consumer of the staged copy releases it by storing v+2 (the descriptor's
// done word/value). Returns false on watchdog expiry.
template <bool SYS>
__device__ bool claim_stage_slot(const P2PArgs& a, Decision& dc) {
  using M = Scope<SYS>;
  const int lane = threadIdx.x & 31;
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  unsigned ns = 32;
  for (;;) {
    for (int base = 0; base < (int)a.arena_slots; base += 32) {
      const int i = base + lane;
      uint64_t v = i < (int)a.arena_slots ? M::ld_rlx(&a.arena_state[i]) : 1;
      unsigned m = __ballot_sync(0xffffffffu, (v & 1) == 0);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        int won = 0;
        if (lane == src) won = M::cas(&a.arena_state[i], v, v + 1) == v;
        if (__shfl_sync(0xffffffffu, won, src)) {
          const uint64_t vv = __shfl_sync(0xffffffffu, v, src);
          const int slot = base + src;
          if (lane == 0) {
            dc.stage_ptr = a.arena + (uint64_t)slot * a.arena_chunk;
            dc.stage_done = &a.arena_state[slot];
            dc.stage_gen = vv + 2;
          }
          __syncwarp();
          return true;
        }
      }
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
      if (lane == 0 && a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
      return false;
    }
  }
}

// ---------------------------------------------------------------------------
// Dynamic matching (MPIX_MATCHING=dynamic): the reference's single-queue
// matcher (proj/src/endpoint.cpp:29-69) per (comm, receiver d), serialised by
// a lock in d's region. Unexpected messages are the send descriptors in d's
// SR rings, stamped with an arrival sequence; posted receives live in d's
// posted-receive queue (PQ), possibly with ANY_SOURCE / ANY_TAG.
//   receive (ticket = d's receive sequence, so a batch matches in post
//     order): take the earliest-arrived acceptable send descriptor, else
//     append to PQ;
//   send (ticket = pseq per source, so sends of a source stay ordered): take
//     the earliest-posted acceptable receive, else post a descriptor.
// The winner copies and completes exactly as in the static protocol.
// ---------------------------------------------------------------------------
struct Dom {
  uint64_t* lock;
  uint64_t* next_rpost;
  uint64_t* arrival;
  uint64_t* next_spost;  // [P]
  SlotDesc* pq;          // [R]
};

__device__ __forceinline__ Dom dom_at(uint8_t* base, const RegionLayout& L) {
  Dom d;
  d.lock = reinterpret_cast<uint64_t*>(base + L.dom_lock());
  d.next_rpost = reinterpret_cast<uint64_t*>(base + L.dom_next_rpost());
  d.arrival = reinterpret_cast<uint64_t*>(base + L.dom_arrival());
  d.next_spost = reinterpret_cast<uint64_t*>(base + L.dom_next_spost(0));
  d.pq = reinterpret_cast<SlotDesc*>(base + L.pq());
  return d;
}

template <bool SYS>
__device__ bool dom_lock(uint64_t* lock, const P2PArgs& a) {
  using M = Scope<SYS>;
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  unsigned ns = 32;
  // acquire only: everything of the previous holder is published by its
  // release (dom_unlock); nothing of mine precedes the lock
  while (M::cas_acq(lock, 0, 1) != 0) {
    __nanosleep(ns);
    if (ns < 512) ns <<= 1;
    if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
      if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
      return false;
    }
  }
  return true;
}

template <bool SYS>
__device__ __forceinline__ void dom_unlock(uint64_t* lock) {
  Scope<SYS>::st_rel(lock, 0);
}

// Warp-wide argmin of (v, idx); lanes without a candidate pass v = ~0.
__device__ __forceinline__ void warp_argmin(uint64_t& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov < v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
}

__device__ __forceinline__ bool tag_ok(int32_t want, int32_t have) { return want < 0 || want == have; }

// Multiplex stream indices in the dynamic engine (endpoint.hpp:26-32): a
// send descriptor carries (src_idx, dst_idx) in key bits 24..31 / 16..23, a
// posted receive its (src_idx filter, dst_idx) in pad[0]; encoded idx + 2
// (-2 = none, -1 = ANY source index).
__device__ __forceinline__ uint64_t idx_enc(int idx) { return (uint64_t)((idx + 2) & 0xff); }
__device__ __forceinline__ bool idx_ok(uint64_t want_src, uint64_t want_dst, uint64_t have_src,
                                       uint64_t have_dst) {
  return want_dst == have_dst && (want_src == 1 /* ANY */ || want_src == have_src);
}

// Receive side (warp 0, lock held): the earliest-arrived POSTED send
// descriptor from an acceptable source with an acceptable tag. Returns the
// source (or -1) and the slot; every lane gets the result.
template <bool SYS>
__device__ int dyn_scan_sends(const P2PArgs& a, uint8_t* my_base, const RegionLayout& L, int* slot_out) {
  const int lane = threadIdx.x & 31;
  uint64_t best = ~0ull;
  int best_idx = 0x7fffffff;
  const int q0 = a.peer >= 0 ? a.peer : 0, q1 = a.peer >= 0 ? a.peer + 1 : a.P;
  for (int q = q0; q < q1; ++q) {
    SlotDesc* ring = reinterpret_cast<SlotDesc*>(my_base + L.sr(q));
    // every load of this source's ring first (one round trip, not one per
    // slot): under the lock no descriptor can become POSTED meanwhile
    uint64_t st[kMaxScanPerLane], ky[kMaxScanPerLane], ar[kMaxScanPerLane];
#pragma unroll
    for (int k = 0; k < kMaxScanPerLane; ++k) {
      const int i = k * 32 + lane;
      st[k] = 0;
      ky[k] = 0;
      ar[k] = ~0ull;
      if (i < a.R) {
        ld_pair<SYS>(&ring[i], st[k], ky[k]);
        ar[k] = Scope<SYS>::ld_rlx(&ring[i].pad[0]);
      }
    }
#pragma unroll
    for (int k = 0; k < kMaxScanPerLane; ++k) {
      const int i = k * 32 + lane;
      if (i < a.R && (st[k] & 0xff) == ST_POSTED && tag_ok(a.tag, (int32_t)(ky[k] >> 32)) &&
          idx_ok(idx_enc(a.sidx), idx_enc(a.didx), (ky[k] >> 24) & 0xff, (ky[k] >> 16) & 0xff) &&
          ar[k] < best) {
        best = ar[k];
        best_idx = q * a.R + i;
      }
    }
  }
  warp_argmin(best, best_idx);
  if (best == ~0ull) return -1;
  *slot_out = best_idx % a.R;  // (32-bit, once per dynamic scan)
  return best_idx / a.R;
}

// Send side (warp 0, lock held): the earliest-posted POSTED receive in the
// receiver's PQ accepting (me, tag). Returns the PQ index or -1.
template <bool SYS>
__device__ int dyn_scan_recvs(const P2PArgs& a, SlotDesc* pq) {
  const int lane = threadIdx.x & 31;
  uint64_t best = ~0ull;
  int best_idx = 0x7fffffff;
  uint64_t st[kMaxScanPerLane], ky[kMaxScanPerLane], fl[kMaxScanPerLane];
#pragma unroll
  for (int k = 0; k < kMaxScanPerLane; ++k) {  // all loads first (lock held)
    const int i = k * 32 + lane;
    st[k] = 0;
    ky[k] = 0;
    fl[k] = 0;
    if (i < a.R) {
      ld_pair<SYS>(&pq[i], st[k], ky[k]);
      fl[k] = Scope<SYS>::ld_rlx(&pq[i].pad[0]);
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxScanPerLane; ++k) {
    const int i = k * 32 + lane;
    const int32_t src = (int32_t)(ky[k] >> 32), tg = (int32_t)(uint32_t)ky[k];
    if (i < a.R && (st[k] & 0xff) == ST_POSTED && (src < 0 || src == a.me) && tag_ok(tg, a.tag) &&
        idx_ok((fl[k] >> 8) & 0xff, fl[k] & 0xff, idx_enc(a.sidx), idx_enc(a.didx))) {
      const uint64_t rseq = st[k] >> 8;
      if (rseq < best) {
        best = rseq;
        best_idx = i;
      }
    }
  }
  warp_argmin(best, best_idx);
  return best == ~0ull ? -1 : best_idx;
}

// Sender takes posted receive pq[j] (lock held, lane 0): push src -> its buffer.
template <bool SYS>
__device__ void dyn_send_take(const P2PArgs& a, Decision& dc, SlotDesc* pq, int j, const Dom& D,
                              const uint8_t* src) {
  using M = Scope<SYS>;
  SlotDesc* e = &pq[j];
  const uint64_t st = M::ld_rlx(&e->state);
  const uint64_t addr = M::ld_rlx(&e->addr), cap = M::ld_rlx(&e->bytes);
  const uint64_t done_addr = M::ld_rlx(&e->done_addr), done_val = M::ld_rlx(&e->done_val);
  M::st_rlx(&e->state, st_word(st >> 8, ST_TAKEN));
  M::st_rlx(&D.next_spost[a.me], a.pseq + 1);
  const int slot = ring_slot(a.pseq, a.R);
  dc.action = ACT_COPY;
  dc.src = (uint64_t)src;
  dc.dst = addr;
  dc.bytes = umin(a.bytes, cap);  // truncation: endpoint.cpp:17
  dc.fin.clear();
  // TAKEN is final for a PQ entry: the receiver reposts into the slot as soon
  // as it is not POSTED, so no later FREE store may follow.
  dc.fin.add_b(&a.post_mirror[slot], a.pseq + 1);  // my SR slot is skipped
  dc.fin.add_b(reinterpret_cast<void*>(done_addr), done_val);
  dc.fin.add_b(a.my_done, a.my_gen);
  if (a.mode == MODE_STAGED && dc.stage_done) dc.fin.add_b(dc.stage_done, dc.stage_gen);
  dc.fin.status(reinterpret_cast<void*>(done_addr), a.bytes, cap, a.me, a.tag, idx_enc(a.sidx));
}

// Sender posts its descriptor (lock held, lane 0), stamped with the arrival.
// key = tag << 32 | 1 if the payload sits in the eager ring slot.
template <bool SYS>
__device__ void dyn_send_post(const P2PArgs& a, const Dom& D, uint64_t addr, uint64_t done_addr,
                              uint64_t done_val, bool eager) {
  using M = Scope<SYS>;
  const int slot = ring_slot(a.pseq, a.R);
  SlotDesc* d = &a.post_ring[slot];
  const uint64_t arr = M::ld_rlx(D.arrival);
  M::st_rlx(D.arrival, arr + 1);
  M::st_rlx(&d->key, ((uint64_t)(uint32_t)a.tag << 32) | (idx_enc(a.sidx) << 24) |
                         (idx_enc(a.didx) << 16) | (eager ? 1u : 0u));
  M::st_rlx(&d->addr, addr);
  M::st_rlx(&d->bytes, a.bytes);
  M::st_rlx(&d->done_addr, done_addr);
  M::st_rlx(&d->done_val, done_val);
  M::st_rlx(&d->pad[0], arr);
  M::st_rlx(&d->state, st_word(a.pseq, ST_POSTED));
  M::st_rlx(&D.next_spost[a.me], a.pseq + 1);
}

template <bool SYS>
__device__ void decide_dyn(const P2PArgs& a, Decision& dc) {
  using M = Scope<SYS>;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const RegionLayout L{a.P, a.R, a.E};
  __shared__ int s_stage;  // 1: eager payload to copy first
  uint8_t* my_base = reinterpret_cast<uint8_t*>(a.bases[a.me]);
  if (threadIdx.x == 0) {
    dc.wait_own = 0;
    dc.now = 0;
    dc.fin.clear();
    dc.action = ACT_NONE;
    dc.stage_ptr = a.staging;
    dc.stage_done = a.stage_done;
    dc.stage_gen = a.stage_gen;
    s_stage = 0;
  }
  __syncthreads();
  if (!a.is_recv) {
    const Dom D = dom_at(reinterpret_cast<uint8_t*>(a.bases[a.peer]), L);
    if (threadIdx.x == 0) {
      bool ok = spin_ge<SYS>(&D.next_spost[a.me], a.pseq, a.err_word, a.spin_limit_ns, ERRW_WAIT_SLOT) &&
                wait_post_slot<SYS>(a);
      s_stage = ok ? (a.mode == MODE_EAGER ? 1 : 2) : 0;
    }
    __syncthreads();
    if (s_stage == 1) {  // eager: payload into my slot of the receiver's eager ring first
      const int slot = ring_slot(a.pseq, a.R);
      cta_copy(a.eager_ring + (uint64_t)slot * 2 * a.E, a.buf, a.bytes);
      __syncthreads();  // published by the unlock's release (after the CTA barrier)
    }
    if (warp == 0 && s_stage != 0) {
      int got = lane == 0 ? (int)dom_lock<SYS>(D.lock, a) : 0;
      got = __shfl_sync(0xffffffffu, got, 0);
      if (got) {
        __syncwarp();  // lane 0's acquire orders the other lanes' scan loads
        const int j = dyn_scan_recvs<SYS>(a, D.pq);
        if (lane == 0) {
          if (j >= 0) {
            dyn_send_take<SYS>(a, dc, D.pq, j, D, a.buf);
          } else if (a.mode == MODE_STAGED) {
            dc.action = ACT_STAGE;  // ticket kept until the staged copy is published
          } else {
            const int slot = ring_slot(a.pseq, a.R);
            const uint64_t addr = a.mode == MODE_EAGER ? (uint64_t)(a.eager_ring + (uint64_t)slot * 2 * a.E)
                                                       : (uint64_t)a.buf;
            if (a.mode == MODE_EAGER) dyn_send_post<SYS>(a, D, addr, 0, 0, true);
            else dyn_send_post<SYS>(a, D, addr, (uint64_t)a.my_done, a.my_gen, false);
          }
          dom_unlock<SYS>(D.lock);
        }
        __syncwarp();
        if (s_stage == 2 && a.mode == MODE_STAGED && !dc.stage_ptr) {
          // claim staging only now that it is needed (lane 0 wrote dc first)
          if (dc.action == ACT_STAGE && !claim_stage_slot<SYS>(a, dc) && lane == 0) dc.action = ACT_NONE;
          __syncwarp();
        }
      }
    }
  } else if (warp == 0) {
    const Dom D = dom_at(my_base, L);
    const int qslot = ring_slot(a.pseq, a.R);
    int got = 0;
    if (lane == 0) {
      // my receive ticket, my PQ slot no longer POSTED, then the lock
      got = spin_ge<SYS>(D.next_rpost, a.pseq, a.err_word, a.spin_limit_ns, ERRW_WAIT_SLOT);
      if (got) {
        const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
        while ((M::ld_rlx(&D.pq[qslot].state) & 0xff) == ST_POSTED) {
          __nanosleep(128);
          if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
            if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
            got = 0;
            break;
          }
        }
      }
      if (got) got = dom_lock<SYS>(D.lock, a);
    }
    got = __shfl_sync(0xffffffffu, got, 0);
    if (got) {
      __syncwarp();  // lane 0's acquire orders the other lanes' scan loads
      int sslot = 0;
      const int q = dyn_scan_sends<SYS>(a, my_base, L, &sslot);
      if (lane == 0) {
        if (q >= 0) {
          SlotDesc* sd = reinterpret_cast<SlotDesc*>(my_base + L.sr(q)) + sslot;
          const uint64_t st = M::ld_rlx(&sd->state);
          const uint64_t key = M::ld_rlx(&sd->key);
          const uint64_t addr = M::ld_rlx(&sd->addr), len = M::ld_rlx(&sd->bytes);
          const uint64_t done_addr = M::ld_rlx(&sd->done_addr), done_val = M::ld_rlx(&sd->done_val);
          const uint64_t spseq = st >> 8;
          uint8_t* qbase = reinterpret_cast<uint8_t*>(a.bases[q]);
          uint64_t* qmirror = reinterpret_cast<uint64_t*>(qbase + L.sr_free(a.me)) + sslot;
          M::st_rlx(D.next_rpost, a.pseq + 1);
          dc.action = ACT_COPY;
          dc.src = addr;
          dc.dst = (uint64_t)a.buf;
          dc.bytes = umin(len, a.bytes);
          dc.fin.clear();
          if (key & 1) {
            // payload in the eager ring slot: copy it now, then free the slot
            M::st_rlx(&sd->state, st_word(spseq, ST_TAKEN));
            dc.now = 1;
            dc.fin.add_a(&sd->state, st_word(spseq, ST_FREE));
            dc.fin.add_b(qmirror, spseq + 1);
          } else {
            // payload elsewhere (user buffer / staging): the slot is free as
            // soon as it is taken, so a sender waiting for it never waits on
            // this copy (or on the rest of this batch)
            M::st_rlx(&sd->state, st_word(spseq, ST_FREE));
            M::fence_ar();
            M::st_rlx(qmirror, spseq + 1);
          }
          dc.fin.add_b(reinterpret_cast<void*>(done_addr), done_val);
          dc.fin.add_b(a.my_done, a.my_gen);
          dc.fin.status(a.my_done, len, a.bytes, q, (int32_t)(key >> 32), (key >> 24) & 0xff);
        } else {
          SlotDesc* e = &D.pq[qslot];
          M::st_rlx(&e->key, ((uint64_t)(uint32_t)a.peer << 32) | (uint32_t)a.tag);
          M::st_rlx(&e->pad[0], (idx_enc(a.sidx) << 8) | idx_enc(a.didx));
          M::st_rlx(&e->addr, (uint64_t)a.buf);
          M::st_rlx(&e->bytes, a.bytes);
          M::st_rlx(&e->done_addr, (uint64_t)a.my_done);
          M::st_rlx(&e->done_val, a.my_gen);
          M::st_rlx(&e->state, st_word(a.pseq, ST_POSTED));
          M::st_rlx(D.next_rpost, a.pseq + 1);
          if (a.blocking) dc.wait_own = 1;
        }
        dom_unlock<SYS>(D.lock);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// Publish a staged blocking send under dynamic matching (whole CTA): under
// the lock, take a receive posted meanwhile (push from staging) or post the
// staging buffer, then release the send ticket.
template <bool SYS>
__device__ void stage_publish_dyn(const P2PArgs& a, Decision& dc) {
  using M = Scope<SYS>;
  const RegionLayout L{a.P, a.R, a.E};
  const Dom D = dom_at(reinterpret_cast<uint8_t*>(a.bases[a.peer]), L);
  __shared__ int s_push;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int got = lane == 0 ? (int)dom_lock<SYS>(D.lock, a) : 0;
    got = __shfl_sync(0xffffffffu, got, 0);
    if (lane == 0) s_push = 0;
    if (got) {
      __syncwarp();  // lane 0's acquire orders the other lanes' scan loads
      const int j = dyn_scan_recvs<SYS>(a, D.pq);
      if (lane == 0) {
        if (j >= 0) {
          dyn_send_take<SYS>(a, dc, D.pq, j, D, dc.stage_ptr);
          s_push = 1;
        } else {
          dyn_send_post<SYS>(a, D, (uint64_t)dc.stage_ptr, (uint64_t)dc.stage_done, dc.stage_gen,
                             false);
        }
        dom_unlock<SYS>(D.lock);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_push == 1) {
    cta_copy(reinterpret_cast<uint8_t*>(dc.dst), reinterpret_cast<const uint8_t*>(dc.src), dc.bytes);
    __syncthreads();
    if (threadIdx.x == 0) dc.fin.run<SYS>();
  }
}

// A self-message whose send and receive the host found in one batch (same
// comm, same key): no descriptors and no scan. Both ring slots are consumed
// only after their previous occupants retired, so the free-mirrors stay
// monotonic; the receive then copies the send buffer and completes both.
template <bool SYS>
__device__ void decide_paired(const P2PArgs& a, Decision& dc) {
  if (threadIdx.x == 0) {
    dc.wait_own = 0;
    dc.now = 0;
    dc.fin.clear();
    dc.action = ACT_NONE;
    dc.stage_ptr = nullptr;
    dc.stage_done = nullptr;
    dc.stage_gen = 0;
    const int rslot = ring_slot(a.pseq, a.R);
    const int sslot = ring_slot(a.pair_pseq, a.R);
    const uint64_t rneed = a.pseq >= (uint64_t)a.R ? a.pseq - a.R + 1 : 0;
    const uint64_t sneed = a.pair_pseq >= (uint64_t)a.R ? a.pair_pseq - a.R + 1 : 0;
    if ((rneed == 0 || spin_ge<SYS>(&a.post_mirror[rslot], rneed, a.err_word, a.spin_limit_ns,
                                    ERRW_WAIT_SLOT)) &&
        (sneed == 0 || spin_ge<SYS>(&a.pair_mirror[sslot], sneed, a.err_word, a.spin_limit_ns,
                                    ERRW_WAIT_SLOT))) {
      dc.action = ACT_COPY;
      dc.src = (uint64_t)a.pair_src;
      dc.dst = (uint64_t)a.buf;
      dc.bytes = umin(a.pair_bytes, a.bytes);  // truncation: endpoint.cpp:17
      dc.fin.add_b(&a.post_mirror[rslot], a.pseq + 1);
      dc.fin.add_b(&a.pair_mirror[sslot], a.pair_pseq + 1);
      dc.fin.add_b(a.pair_done, a.pair_gen);
      dc.fin.add_b(a.my_done, a.my_gen);
      dc.fin.status(a.my_done, a.pair_bytes, a.bytes, a.me, (int)(a.key >> 32), 0);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Flag-in-data (LL) small sends and polling blocking receives
// ---------------------------------------------------------------------------
// Payload bytes (<= kLLBytes) into three 32-bit words: byte loads, all in
// flight together (no read past the user's buffer).
__device__ __forceinline__ void ll_load(const uint8_t* src, uint64_t n, uint32_t w[3]) {
  uint8_t b[kLLBytes];
  if (n == 0) {
#pragma unroll
    for (int i = 0; i < (int)kLLBytes; ++i) b[i] = 0;
  } else {
    // branch-free: every load is issued before any result is used (a
    // conditional load per byte compiled to a chain of dependent round
    // trips); bytes past n re-read the last byte and are masked below
    uint8_t v[kLLBytes];
#pragma unroll
    for (int i = 0; i < (int)kLLBytes; ++i) v[i] = __ldcg(src + (i < (int)n ? i : (int)n - 1));
#pragma unroll
    for (int i = 0; i < (int)kLLBytes; ++i) b[i] = i < (int)n ? v[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    w[k] = (uint32_t)b[4 * k] | ((uint32_t)b[4 * k + 1] << 8) | ((uint32_t)b[4 * k + 2] << 16) |
           ((uint32_t)b[4 * k + 3] << 24);
}

// Post an LL send descriptor (lane 0): three payload words and the length as
// LL words, the sender's completion word/value check-tagged (ll_chk), the key,
// then the state — all relaxed: a reader validates every word by its flag or
// check, and a stale key never matches (keys are unique per pair), so nothing
// has to be ordered before the state store. Like an Isend's descriptor, the
// post completes the sender's request only when a receiver consumes it (the
// windows of a stream stay flow-controlled by their receivers).
template <bool SYS>
__device__ void ll_post(const P2PArgs& a, const uint32_t w[3]) {
  using M = Scope<SYS>;
  SlotDesc* d = &a.post_ring[ring_slot(a.pseq, a.R)];
  const uint32_t f = ll_flag(a.pseq);
  const uint64_t chk = ll_chk(a.pseq);
  M::st_rlx(&d->addr, ll_word(w[0], f));
  M::st_rlx(&d->pad[0], ll_word(w[1], f));
  M::st_rlx(&d->pad[1], ll_word(w[2], f));
  M::st_rlx(&d->bytes, ll_word((uint32_t)a.bytes, f));
  M::st_rlx(&d->done_addr, ((uint64_t)a.my_done & kLLPtrMask) | chk);
  M::st_rlx(&d->done_val, (a.my_done ? (a.my_gen & kLLPtrMask) : 0) | chk);
  M::st_rlx(&d->key, a.key);
  M::st_rlx(&d->state, st_word(a.pseq, ST_POSTED | ST_LL));
}

struct LLMsg {
  uint32_t w[3];
  uint64_t len;
  uint64_t* sdone;  // the sender's completion word (null: a blocking send)
  uint64_t sgen;
};

// Read an LL send descriptor's words (lane 0) until every flag and check is
// its post's (the scan's snapshot first: usually everything has landed).
// Returns false on watchdog expiry.
template <bool SYS>
__device__ bool ll_read(const SlotDesc* s, const Snap& sn, LLMsg& m, const P2PArgs& a) {
  using M = Scope<SYS>;
  const uint64_t pseq = sn.state >> 8;
  const uint32_t f = ll_flag(pseq);
  const uint64_t chk = ll_chk(pseq);
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  uint64_t w0 = sn.addr, w1 = sn.p0, w2 = sn.p1, wl = sn.bytes, da = sn.done_addr, dv = sn.done_val;
  for (;;) {
    if ((uint32_t)(w0 >> 32) == f && (uint32_t)(w1 >> 32) == f && (uint32_t)(w2 >> 32) == f &&
        (uint32_t)(wl >> 32) == f && (da & ~kLLPtrMask) == chk && (dv & ~kLLPtrMask) == chk) {
      m.w[0] = (uint32_t)w0;
      m.w[1] = (uint32_t)w1;
      m.w[2] = (uint32_t)w2;
      m.len = (uint32_t)wl;
      m.sdone = reinterpret_cast<uint64_t*>(da & kLLPtrMask);
      m.sgen = dv & kLLPtrMask;
      return true;
    }
    __nanosleep(32);
    if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
      if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
      return false;
    }
    w0 = M::ld_rlx(&s->addr);
    w1 = M::ld_rlx(&s->pad[0]);
    w2 = M::ld_rlx(&s->pad[1]);
    wl = M::ld_rlx(&s->bytes);
    da = M::ld_rlx(&s->done_addr);
    dv = M::ld_rlx(&s->done_val);
  }
}

// Complete my receive from an LL send descriptor (lane 0; the descriptor is
// mine: taken by CAS, or never contended): payload and status, my post slot
// consumed (and my posted descriptor retracted if I had posted one), my
// completion word, then the sender's free-mirror (it may reuse its slot) and
// its completion word.
template <bool SYS>
__device__ void ll_complete(const P2PArgs& a, int j, const Snap& sn, const LLMsg& m, bool posted,
                            uint64_t gate = 0) {
  using M = Scope<SYS>;
  const uint64_t n = umin(m.len, a.bytes);  // truncation: endpoint.cpp:17
  for (uint64_t i = 0; i < n; ++i) a.buf[i] = (uint8_t)(m.w[i >> 2] >> (8 * (i & 3)));
  if (a.my_done) {
    uint8_t* d = reinterpret_cast<uint8_t*>(a.my_done);
    ScopeGpu::st_rlx(reinterpret_cast<uint64_t*>(d + kStatusOff), n | (m.len > a.bytes ? kTruncBit : 0));
    ScopeGpu::st_rlx(reinterpret_cast<uint64_t*>(d + 2 * kStatusOff),
                     ((uint64_t)(a.peer & 0xffffff) << 40) | (((uint64_t)(a.sidx + 2) & 0xff) << 32) |
                         (uint32_t)(sn.key >> 32));
  }
  const int slot = ring_slot(a.pseq, a.R);
  if (posted) M::st_rlx(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));  // retract
  ScopeGpu::st_rlx(&a.post_mirror[slot], a.pseq + 1);  // consumed either way (local)
  // my completion: read only by this rank (its waits, the host after a
  // synchronisation), so device scope orders the payload and status before
  // it; a blocking receive completes in its own kernel, whose end publishes
  // everything to later stream work and to the host (no fence)
  if (a.my_done) {
    if (a.blocking) ScopeGpu::st_rlx(a.my_done, a.my_gen);
    else ScopeGpu::st_rel(a.my_done, a.my_gen);
  }
  // `gate`: the result of the atomic that took the slot (first-scan take);
  // branching on it makes the free-mirror wait until that atomic has been
  // performed, so the TAKEN state can never land after the sender's next post
  if (gate == ~0ull) return;
  M::st_rlx(&a.scan_mirror[j], (sn.state >> 8) + 1);
  if (m.sdone) M::st_rlx(m.sdone, m.sgen);
}

// LL-eager: an eager send of 13 B .. E writes its payload
// into its eager slot as LL words (4 bytes + the post's flag each; the slot
// holds 2E bytes) and posts an LL-style descriptor — the whole CTA stores,
// nothing orders them (every word carries the flag), thread 0 then does the
// Dekker fence. The descriptor's addr holds the slot with a check like the
// completion words (a stale addr must not send the reader elsewhere).
template <bool SYS>
__device__ void lle_post(const P2PArgs& a) {  // whole CTA
  using M = Scope<SYS>;
  const int slot = ring_slot(a.pseq, a.R);
  uint64_t* w = reinterpret_cast<uint64_t*>(a.eager_ring + (uint64_t)slot * 2 * a.E);
  const uint32_t f = ll_flag(a.pseq);
  const uint64_t n = a.bytes, nw = (n + 3) / 4;
  for (uint64_t i = threadIdx.x; i < nw; i += blockDim.x) {
    uint32_t d = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint64_t k = 4 * i + b;
      if (k < n) d |= (uint32_t)a.buf[k] << (8 * b);
    }
    M::st_rlx(&w[i], ll_word(d, f));
  }
  if (threadIdx.x == 0) {
    SlotDesc* d = &a.post_ring[slot];
    const uint64_t chk = ll_chk(a.pseq);
    M::st_rlx(&d->addr, ((uint64_t)w & kLLPtrMask) | chk);
    M::st_rlx(&d->pad[0], ll_word(0, f));
    M::st_rlx(&d->pad[1], ll_word(0, f));
    M::st_rlx(&d->bytes, ll_word((uint32_t)n, f));
    M::st_rlx(&d->done_addr, ((uint64_t)a.my_done & kLLPtrMask) | chk);
    M::st_rlx(&d->done_val, (a.my_done ? (a.my_gen & kLLPtrMask) : 0) | chk);
    M::st_rlx(&d->key, a.key);
    M::st_rlx(&d->state, st_word(a.pseq, ST_POSTED | ST_LL | ST_LLE));
    M::fence_sc();
  }
}

// Take an LL-eager descriptor (lane 0; taken already by CAS or exchange):
// validate its words, record what the CTA copies and completes (ACT_LLE).
// Returns false on watchdog expiry.
template <bool SYS>
__device__ bool lle_take(const P2PArgs& a, Decision& dc, int j, const Snap& sn, bool posted,
                         uint64_t gate) {
  using M = Scope<SYS>;
  const SlotDesc* s = &a.scan_ring[j];
  const uint64_t pseq = sn.state >> 8;
  const uint32_t f = ll_flag(pseq);
  const uint64_t chk = ll_chk(pseq);
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  uint64_t ad = sn.addr, w1 = sn.p0, w2 = sn.p1, wl = sn.bytes, da = sn.done_addr, dv = sn.done_val;
  while (!((ad & ~kLLPtrMask) == chk && (uint32_t)(w1 >> 32) == f && (uint32_t)(w2 >> 32) == f &&
           (uint32_t)(wl >> 32) == f && (da & ~kLLPtrMask) == chk && (dv & ~kLLPtrMask) == chk)) {
    __nanosleep(32);
    if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
      if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
      return false;
    }
    ad = M::ld_rlx(&s->addr);
    w1 = M::ld_rlx(&s->pad[0]);
    w2 = M::ld_rlx(&s->pad[1]);
    wl = M::ld_rlx(&s->bytes);
    da = M::ld_rlx(&s->done_addr);
    dv = M::ld_rlx(&s->done_val);
  }
  const uint64_t len = (uint32_t)wl;
  dc.action = ACT_LLE;
  dc.src = ad & kLLPtrMask;
  dc.dst = (uint64_t)a.buf;
  dc.bytes = umin(len, a.bytes);  // truncation: endpoint.cpp:17
  dc.lle_len = len;
  dc.lle_spseq = pseq;
  dc.lle_key = sn.key;
  dc.lle_gate = gate;
  dc.lle_sdone = reinterpret_cast<uint64_t*>(da & kLLPtrMask);
  dc.lle_sgen = dv & kLLPtrMask;
  dc.lle_j = j;
  dc.lle_posted = posted ? 1 : 0;
  return true;
}

// The CTA copies the LL words of a taken LL-eager send into my buffer (each
// word re-read until its flag is the post's), then thread 0 completes as
// ll_complete does.
template <bool SYS>
__device__ void lle_finish(const P2PArgs& a, Decision& dc) {  // whole CTA
  using M = Scope<SYS>;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(dc.src);
  const uint32_t f = ll_flag(dc.lle_spseq);
  const uint64_t n = dc.bytes, nw = (n + 3) / 4;
  uint8_t* out = reinterpret_cast<uint8_t*>(dc.dst);
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  for (uint64_t i = threadIdx.x; i < nw; i += blockDim.x) {
    uint64_t v = M::ld_rlx(&w[i]);
    while ((uint32_t)(v >> 32) != f) {
      __nanosleep(32);
      if (a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
        if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_SLOT);
        break;
      }
      v = M::ld_rlx(&w[i]);
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint64_t k = 4 * i + b;
      if (k < n) out[k] = (uint8_t)(v >> (8 * b));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.my_done) {
      uint8_t* d = reinterpret_cast<uint8_t*>(a.my_done);
      ScopeGpu::st_rlx(reinterpret_cast<uint64_t*>(d + kStatusOff),
                       n | (dc.lle_len > a.bytes ? kTruncBit : 0));
      ScopeGpu::st_rlx(reinterpret_cast<uint64_t*>(d + 2 * kStatusOff),
                       ((uint64_t)(a.peer & 0xffffff) << 40) | (((uint64_t)(a.sidx + 2) & 0xff) << 32) |
                           (uint32_t)(dc.lle_key >> 32));
    }
    const int slot = ring_slot(a.pseq, a.R);
    if (dc.lle_posted) M::st_rlx(&a.post_ring[slot].state, st_word(a.pseq, ST_FREE));  // retract
    ScopeGpu::st_rlx(&a.post_mirror[slot], a.pseq + 1);
    if (a.my_done) {
      if (a.blocking) ScopeGpu::st_rlx(a.my_done, a.my_gen);
      else ScopeGpu::st_rel(a.my_done, a.my_gen);
    }
    // the payload loads have returned (their bytes are stored, barrier
    // above) and the slot is TAKEN (gate: the exchange has been performed)
    // before the sender may reuse it
    if (dc.lle_gate != ~0ull) {
      M::st_rlx(&a.scan_mirror[dc.lle_j], dc.lle_spseq + 1);
      if (dc.lle_sdone) M::st_rlx(dc.lle_sdone, dc.lle_sgen);
    }
    dc.action = ACT_NONE;
  }
  __syncthreads();
}

// A blocking receive (static matching) never posts a descriptor: no sender
// waits for one (eager and staged sends complete on their own, an Isend
// leaves its descriptor), so it polls its scan ring until the send with its
// key is there and takes it as the second arriver — no Dekker fence on the
// receive side. Warp 0; returns the slot or -1 on watchdog expiry.
template <bool SYS>
__device__ int poll_scan(const P2PArgs& a, Snap* sn) {
  const int lane = threadIdx.x & 31;
  const uint64_t t0 = a.spin_limit_ns ? globaltimer() : 0;
  unsigned ns = 32;
  for (;;) {
    const int j = warp_scan<SYS>(a.scan_ring, a.R, a.key, sn);
    if (j >= 0) return j;
    int expired = 0;
    if (lane == 0 && a.spin_limit_ns && globaltimer() - t0 > a.spin_limit_ns) {
      if (a.err_word) ScopeSys::st_rlx(a.err_word, ERRW_WAIT_DONE);
      expired = 1;
    }
    if (__shfl_sync(0xffffffffu, expired, 0)) return -1;
    __nanosleep(ns);
    if (ns < 64) ns <<= 1;
  }
}

// The handshake (whole CTA calls; warp 0 works, the CTA copies eager
// payloads). On return dc holds ACT_NONE / ACT_COPY / ACT_STAGE.
// TINY: the lean instantiation of k_batch_tiny (no staged sends, no trace):
// less code to fetch into a cold SM's instruction cache.
template <bool SYS, bool TINY = false>
__device__ void decide(const P2PArgs& a, Decision& dc) {
  using M = Scope<SYS>;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  __shared__ int s_phase;  // 0 decided, 1 eager copy then post, 2 posted, 3 claim staging
  // LL: a small send's payload travels in its descriptor; a blocking
  // receive polls instead of posting
  const bool ll_send = a.ll && !a.is_recv && a.bytes <= kLLBytes && a.mode != MODE_STAGED;
  // (only receives of at most kPollMaxBytes: a larger one posts, as in round
  // 1, so that a large blocking send finds it and pushes straight into the
  // receive buffer instead of staging its payload first — an extra copy
  // grid and three more launches: 1 MiB ping-pong 16.8 -> 23.3 us when every
  // blocking receive polled; up to 64 KiB polling wins, the receiver's post
  // fences cost more than the sender's staging copy)
  const bool poll_recv = a.ll && a.is_recv && a.blocking && a.bytes <= kPollMaxBytes;
  // (an Isend too: its descriptor carries its completion word, signalled by
  // the receiver that consumes it, as for any Isend)
  const bool lle_send = a.ll && !a.is_recv && (a.mode == MODE_EAGER || a.mode == MODE_ISEND) &&
                        a.bytes > kLLBytes && a.bytes <= a.E;
  __shared__ uint32_t s_pay[3];  // an LL send's payload (lane 0)
  TraceRec* const trace = TINY ? nullptr : a.trace;
  if (warp == 0) {
    // the free-mirror of my post slot, loaded alongside the ring scan (one
    // round trip instead of two in steady state, pseq >= R); an LL send's
    // payload loads are in flight with them too
    uint64_t pre = 0;
    uint32_t pay[3] = {0, 0, 0};
    // (relaxed: the slot's previous occupant is done with it once its mirror
    // moved; nothing read here depends on data the mirror publishes)
    if (lane == 0 && a.pseq >= (uint64_t)a.R) pre = M::ld_rlx(&a.post_mirror[ring_slot(a.pseq, a.R)]);
    if (lane == 0 && ll_send) ll_load(a.buf, a.bytes, pay);
    Snap sn;
    // An LL send posts first and scans after its fence (phase 2: the same
    // Dekker race, resolved by the CAS on its LL state word): its post
    // reaches the receiver one round trip earlier than scan-then-post.
    int j = ll_send ? -1 : warp_scan<SYS>(a.scan_ring, a.R, a.key, &sn);
    if (poll_recv && j < 0) j = poll_scan<SYS>(a, &sn);
    if (lane == 0) {
      trace_t(trace, 1);
      dc.wait_own = 0;
      dc.now = 0;
      dc.fin.clear();
      dc.action = ACT_NONE;
      dc.stage_ptr = a.staging;  // null: claim from the device arena if needed
      dc.stage_done = a.stage_done;
      dc.stage_gen = a.stage_gen;
      s_phase = 0;
      if (!a.is_recv) {
        if (j >= 0) {
          // receive already posted: push (my slot is skipped, but only after
          // its previous occupant retired, so its mirror stays monotonic)
          // (an LL send pushes the payload it already holds, s_pay below)
          if (wait_post_slot<SYS>(a, pre))
            send_win(a, dc, j, sn, false, ll_send ? reinterpret_cast<const uint8_t*>(s_pay) : a.buf);
        } else if (!TINY && a.mode == MODE_STAGED) {
          dc.action = ACT_STAGE;
          if (!dc.stage_ptr) s_phase = 3;
        } else if (wait_post_slot<SYS>(a, pre)) {
          if (ll_send) {
            // the Dekker fence and rescan follow the post (off the
            // receiver's critical path)
            ll_post<SYS>(a, pay);
            M::fence_sc();
            s_phase = 2;
          } else if (lle_send) {
            s_phase = 5;  // LL-eager post by the whole CTA, then the rescan
          } else if (a.mode == MODE_EAGER) {
            s_phase = 1;
          } else {  // MODE_ISEND: publish the user buffer
            post_desc<SYS>(a, (uint64_t)a.buf, a.bytes, (uint64_t)a.my_done, a.my_gen, false);
            s_phase = 2;
          }
        }
      } else {
        if (j >= 0) {
          // I have not posted, so no one else may take this descriptor (its
          // sender takes its own post only after finding my posted receive):
          // no CAS
          if (!wait_post_slot<SYS>(a, pre)) {
            // watchdog: leave the send descriptor for nobody
          } else if (sn.state & ST_LLE) {
            const uint64_t old = M::exch(&a.scan_ring[j].state, st_word(sn.state >> 8, ST_TAKEN));
            lle_take<SYS>(a, dc, j, sn, false, old);
          } else if (sn.state & ST_LL) {
            // TAKEN by an atomic exchange (no competitor: a plain store would
            // do, but it could land after the free-mirror below); its round
            // trip overlaps the payload and status stores
            const uint64_t old = M::exch(&a.scan_ring[j].state, st_word(sn.state >> 8, ST_TAKEN));
            LLMsg m;
            if (ll_read<SYS>(&a.scan_ring[j], sn, m, a)) ll_complete<SYS>(a, j, sn, m, false, old);
          } else {
            M::st_rlx(&a.scan_ring[j].state, st_word(sn.state >> 8, ST_TAKEN));
            recv_win(a, dc, j, sn, false);
          }
        } else if (!poll_recv && wait_post_slot<SYS>(a, pre)) {
          post_desc<SYS>(a, (uint64_t)a.buf, a.bytes, (uint64_t)a.my_done, a.my_gen, false);
          s_phase = 2;
        }
      }
      if (ll_send) {
        s_pay[0] = pay[0];
        s_pay[1] = pay[1];
        s_pay[2] = pay[2];
      }
    }
    __syncwarp();
    if (!TINY) {
      const int ph = s_phase;  // every lane reads before lane 0 may rewrite it
      __syncwarp();
      if (ph == 3 && !claim_stage_slot<SYS>(a, dc) && lane == 0) dc.action = ACT_NONE;
      __syncwarp();
      if (lane == 0 && ph == 3) s_phase = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_t(trace, 2);
  int phase = s_phase;
  if (phase == 5) {
    lle_post<SYS>(a);
    phase = 2;
  }
  if (phase == 1) {
    // Eager: payload into the receiver's eager slot (peer stores).
    const int slot = ring_slot(a.pseq, a.R);
    cta_copy(a.eager_ring + (uint64_t)slot * 2 * a.E, a.buf, a.bytes);
    __syncthreads();
    if (threadIdx.x == 0)
      post_desc<SYS>(a, (uint64_t)(a.eager_ring + (uint64_t)slot * 2 * a.E), a.bytes, 0, 0, true);
    phase = 2;
  }
  if (phase == 2 && warp == 0) {
    // Posted: rescan; if the other side's descriptor is there, race for the
    // send descriptor's state word (second arriver copies).
    Snap sn;
    int j = warp_scan<SYS>(a.scan_ring, a.R, a.key, &sn);
    if (lane == 0) {
     if (j >= 0) {
      if (!a.is_recv) {
        const int slot = ring_slot(a.pseq, a.R);
        uint64_t want = st_word(a.pseq, ll_send ? (ST_POSTED | ST_LL)
                                        : (lle_send ? (ST_POSTED | ST_LL | ST_LLE) : ST_POSTED));
        if (M::cas(&a.post_ring[slot].state, want, st_word(a.pseq, ST_TAKEN)) == want)
          send_win(a, dc, j, sn, true, ll_send ? reinterpret_cast<const uint8_t*>(s_pay) : a.buf);
      } else {
        const uint64_t want = sn.state;
        if (M::cas(&a.scan_ring[j].state, want, st_word(sn.state >> 8, ST_TAKEN)) == want) {
          if (sn.state & ST_LLE) {
            lle_take<SYS>(a, dc, j, sn, true, 0);
          } else if (sn.state & ST_LL) {
            LLMsg m;
            if (ll_read<SYS>(&a.scan_ring[j], sn, m, a)) ll_complete<SYS>(a, j, sn, m, true);
          } else {
            recv_win(a, dc, j, sn, true);
          }
        }
      }
     }
     // (lane 0 only: the other lanes never touch the shared decision)
     if (dc.action == ACT_NONE && a.is_recv && a.blocking) dc.wait_own = 1;
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_t(trace, 3);
}

// Publish a staged blocking send and race for its descriptor (whole CTA).
template <bool SYS>
__device__ void stage_publish(const P2PArgs& a, Decision& dc) {
  using M = Scope<SYS>;
  __shared__ int s_push;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      s_push = 0;
      dc.action = ACT_NONE;
      if (wait_post_slot<SYS>(a))
        post_desc<SYS>(a, (uint64_t)dc.stage_ptr, a.bytes, (uint64_t)dc.stage_done, dc.stage_gen, true);
      else
        s_push = -1;
    }
    __syncwarp();
    if (__shfl_sync(0xffffffffu, s_push, 0) == 0) {
      Snap sn;
      int j = warp_scan<SYS>(a.scan_ring, a.R, a.key, &sn);
      if (threadIdx.x == 0 && j >= 0) {
        const int slot = ring_slot(a.pseq, a.R);
        uint64_t want = st_word(a.pseq, ST_POSTED);
        if (M::cas(&a.post_ring[slot].state, want, st_word(a.pseq, ST_TAKEN)) == want) {
          send_win(a, dc, j, sn, true, dc.stage_ptr);
          s_push = 1;
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (s_push == 1) {
    cta_copy(reinterpret_cast<uint8_t*>(dc.dst), reinterpret_cast<const uint8_t*>(dc.src), dc.bytes);
    __syncthreads();
    if (threadIdx.x == 0) dc.fin.run<SYS>();
  }
}

// The whole handshake of one operation (one CTA). INLINE: the copy and the
// completion stores happen here too; otherwise the decision goes to the op
// record for k_copy / k_fin.
template <bool SYS, bool INLINE, bool TINY = false>
__device__ __forceinline__ void proto_body(const P2PArgs& a, Decision& s_dc) {
  static_assert(!TINY || INLINE, "tiny operations are inline");
  if (TINY) {  // static matching, inline, no staging, no graph counters, no trace
    decide<SYS, true>(a, s_dc);
    if (s_dc.action == ACT_LLE) {
      lle_finish<SYS>(a, s_dc);
    } else if (s_dc.action == ACT_COPY) {
      cta_copy(reinterpret_cast<uint8_t*>(s_dc.dst), reinterpret_cast<const uint8_t*>(s_dc.src),
               s_dc.bytes);
      __syncthreads();
      if (threadIdx.x == 0) s_dc.fin.run<SYS>();
    } else if (threadIdx.x == 0 && s_dc.wait_own) {
      spin_ge<SYS>(a.my_done, a.my_gen, a.err_word, a.spin_limit_ns, ERRW_WAIT_DONE);
    }
    return;
  }
  if (a.trace && threadIdx.x == 0) {
    // the record's head is written here, not by a host copy: a copy node
    // between two operation kernels would distort the gaps being measured
    a.trace->g0 = globaltimer();
    a.trace->t[0] = a.trace->g0;
    a.trace->seq = a.trace_seq;
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.trace->pad[0] = sm;
    a.trace->bytes = a.bytes;
    a.trace->key = a.key;
  }
  if (a.mate_skip) {  // a device-matched send: its receive copies and completes it
    if (!INLINE && threadIdx.x == 0) a.rec->action = ACT_NONE;
    __syncthreads();
    if (!INLINE) pdl_trigger();
    return;
  }
  if (a.greset) {  // captured blocking receive: its completion word is reused every replay
    if (threadIdx.x == 0) {
      *reinterpret_cast<volatile uint64_t*>(a.my_done) = 0;
      __threadfence();
    }
    __syncthreads();
  }
  if (a.paired) decide_paired<SYS>(a, s_dc);
  else if (a.dyn) decide_dyn<SYS>(a, s_dc);
  else decide<SYS>(a, s_dc);
  if (a.trace && threadIdx.x == 0)
    a.trace->info = (uint64_t)a.is_recv | ((uint64_t)a.mode << 4) | ((uint64_t)INLINE << 8) |
                    (s_dc.action << 12);
  if (!INLINE && s_dc.action == ACT_LLE) {
    lle_finish<SYS>(a, s_dc);
    if (threadIdx.x == 0) a.rec->action = ACT_NONE;  // nothing for the copy grid / k_fin
    __syncthreads();
    pdl_trigger();
    return;
  }
  if (!INLINE && s_dc.now) {
    cta_copy(reinterpret_cast<uint8_t*>(s_dc.dst), reinterpret_cast<const uint8_t*>(s_dc.src),
             s_dc.bytes);
    __syncthreads();
    if (threadIdx.x == 0) {
      s_dc.fin.run<SYS>();
      a.rec->action = ACT_NONE;  // nothing left for the copy grid / k_fin
    }
    __syncthreads();
    pdl_trigger();
    return;
  }
  if (!INLINE) {
    if (threadIdx.x == 0) {
      OpRecord* rec = a.rec;
      rec->action = s_dc.action;
      const bool stg = s_dc.action == ACT_STAGE;  // copy user buffer -> staging
      rec->src = stg ? (uint64_t)a.buf : s_dc.src;
      rec->dst = stg ? (uint64_t)s_dc.stage_ptr : s_dc.dst;
      rec->bytes = stg ? a.bytes : s_dc.bytes;
      rec->nfin = s_dc.fin.na | (s_dc.fin.nb << 8);
      rec->stage_ptr = (uint64_t)s_dc.stage_ptr;
      rec->stage_done = (uint64_t)s_dc.stage_done;
      rec->stage_gen = s_dc.stage_gen;
      rec->stat_addr = s_dc.fin.s_addr;
      rec->stat_bytes = s_dc.fin.s_bytes;
      rec->stat_srctag = s_dc.fin.s_srctag;
      for (uint32_t k = 0; k < s_dc.fin.na; ++k) {
        rec->fin_addr[k] = s_dc.fin.a_addr[k];
        rec->fin_val[k] = s_dc.fin.a_val[k];
      }
      for (uint32_t k = 0; k < s_dc.fin.nb; ++k) {
        rec->fin_addr[2 + k] = s_dc.fin.b_addr[k];
        rec->fin_val[2 + k] = s_dc.fin.b_val[k];
      }
    }
    // A blocking receive that posted and waits for the sender's push lets
    // its (then idle) copy grid launch only afterwards: a grid parked at
    // griddepcontrol.wait would occupy the SMs a sender on this GPU needs.
    if (a.early_trigger) pdl_trigger();
    if (threadIdx.x == 0 && s_dc.wait_own)
      spin_ge<SYS>(a.my_done, a.my_gen, a.err_word, a.spin_limit_ns, ERRW_WAIT_DONE);
    __syncthreads();
    pdl_trigger();
    return;
  }
  if (s_dc.action == ACT_LLE) {
    lle_finish<SYS>(a, s_dc);
    if (threadIdx.x == 0 && a.trace) a.trace->g1 = globaltimer();
  } else if (s_dc.action == ACT_COPY) {
    cta_copy(reinterpret_cast<uint8_t*>(s_dc.dst), reinterpret_cast<const uint8_t*>(s_dc.src),
             s_dc.bytes);
    __syncthreads();
    if (threadIdx.x == 0) {
      trace_t(a.trace, 4);
      s_dc.fin.run<SYS>();
      trace_t(a.trace, 5);
      if (a.trace) a.trace->g1 = globaltimer();
    }
  } else if (s_dc.action == ACT_STAGE) {
    cta_copy(s_dc.stage_ptr, a.buf, a.bytes);
    __syncthreads();
    if (a.dyn) stage_publish_dyn<SYS>(a, s_dc);
    else stage_publish<SYS>(a, s_dc);
  } else if (threadIdx.x == 0) {
    if (s_dc.wait_own) spin_ge<SYS>(a.my_done, a.my_gen, a.err_word, a.spin_limit_ns, ERRW_WAIT_DONE);
    if (a.trace) a.trace->g1 = globaltimer();
  }
}

template <bool SYS, bool INLINE>
__global__ void __launch_bounds__(kThreads) k_proto(const P2PArgs a) {
  __shared__ Decision s_dc;
  pdl_wait();                 // (launched early behind a previous operation)
  if (INLINE) pdl_trigger();  // the next small head kernel may park behind me
  proto_body<SYS, INLINE>(a, s_dc);
}

// Wide copy behind k_proto (PDL): never waits on anything but the stream.
__global__ void __launch_bounds__(kCopyThreads, 2) k_copy(const P2PArgs a) {
  pdl_wait();
  const OpRecord* rec = a.rec;
  const uint64_t action = rec->action;
  if (action == ACT_COPY || action == ACT_STAGE) {
    tile_copy(reinterpret_cast<uint8_t*>(rec->dst), reinterpret_cast<const uint8_t*>(rec->src),
              rec->bytes, blockIdx.x, gridDim.x);
  }
  pdl_trigger();
}

// Completion of a large operation after its copy grid retired: the
// completion stores, or the publication of a staged send.
template <bool SYS>
__device__ void fin_body(const P2PArgs& a, Decision& s_dc) {
  const OpRecord* rec = a.rec;
  const uint64_t action = rec->action;
  if (action == ACT_COPY) {
    if (threadIdx.x == 0) {
      Fin f;
      f.na = rec->nfin & 0xff;
      f.nb = rec->nfin >> 8;
      f.s_addr = rec->stat_addr;
      f.s_bytes = rec->stat_bytes;
      f.s_srctag = rec->stat_srctag;
      for (uint32_t k = 0; k < f.na; ++k) { f.a_addr[k] = rec->fin_addr[k]; f.a_val[k] = rec->fin_val[k]; }
      for (uint32_t k = 0; k < f.nb; ++k) { f.b_addr[k] = rec->fin_addr[2 + k]; f.b_val[k] = rec->fin_val[2 + k]; }
      f.run<SYS>();
    }
  } else if (action == ACT_STAGE) {
    if (threadIdx.x == 0) {
      s_dc.stage_ptr = reinterpret_cast<uint8_t*>(rec->stage_ptr);
      s_dc.stage_done = reinterpret_cast<uint64_t*>(rec->stage_done);
      s_dc.stage_gen = rec->stage_gen;
    }
    __syncthreads();
    if (a.dyn) stage_publish_dyn<SYS>(a, s_dc);
    else stage_publish<SYS>(a, s_dc);
  }
}

// Completion behind k_copy (PDL): the grid above has fully retired.
template <bool SYS>
__global__ void __launch_bounds__(kThreads) k_fin(const P2PArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ Decision s_dc;
  fin_body<SYS>(a, s_dc);
}

// ---------------------------------------------------------------------------
// Coalesced batches (host-side op batching). Operations of one
// batch are mutually unordered (non-blocking, plus at most one trailing
// blocking operation), so they run concurrently, one CTA each:
//   inline only:  k_batch (ops + the closing Wait/Waitall as CTA n)
//   with large:   k_batch (decisions) -> k_gcopy (one grouped copy grid over
//                 every large operation) -> k_gfin (completions + the wait)
// ---------------------------------------------------------------------------
__device__ void load_op(const BatchOp& o, uint64_t spin_limit_ns, P2PArgs& a) {
  a.is_recv = o.is_recv;
  a.mode = o.mode;
  a.blocking = o.blocking;
  a.R = o.R;
  a.key = o.key;
  a.pseq = o.pseq;
  a.greset = 0;
  if (o.gflags & G_ON) {  // graph-capturable comm: sequences relative to the device counters
    const volatile uint64_t* g = o.bases;
    a.pseq = g[o.gp] + o.pseq;
    const uint32_t t = (uint32_t)g[o.gt] + (uint32_t)o.key;
    a.key = (o.key & 0xffffffff00000000ull) | t;
    a.greset = (o.gflags & G_RESET) ? 1 : 0;
  }
  a.post_ring = o.post_ring;
  a.post_mirror = o.post_mirror;
  a.scan_ring = o.scan_ring;
  a.scan_mirror = o.scan_mirror;
  a.eager_ring = o.eager_ring;
  a.E = o.E;
  a.buf = o.buf;
  a.bytes = o.bytes;
  a.my_done = o.my_done;
  a.my_gen = o.my_gen;
  a.paired = o.paired;
  if (o.paired) {
    a.staging = nullptr;
    a.stage_done = nullptr;
    a.stage_gen = 0;
    a.arena = nullptr;
    a.arena_state = nullptr;
    a.arena_chunk = 0;
    a.pair_src = o.pr.src;
    a.pair_bytes = o.pr.bytes;
    a.pair_done = o.pr.done;
    a.pair_gen = o.pr.gen;
    a.pair_mirror = o.pr.mirror;
    a.pair_pseq = o.pr.pseq;
  } else {
    a.staging = o.st.staging;
    a.stage_done = o.st.stage_done;
    a.stage_gen = o.st.stage_gen;
    a.arena = o.st.arena;
    a.arena_state = o.st.arena_state;
    a.arena_chunk = o.st.arena_chunk;
  }
  a.arena_slots = o.arena_slots;
  a.rec = o.rec;
  a.opid = 0;
  a.err_word = o.err_word;
  a.spin_limit_ns = spin_limit_ns;
  a.trace = nullptr;
  a.early_trigger = o.early;
  a.ll = o.ll;
  a.mate_skip = 0;
  a.dyn = o.dyn;
  a.P = o.P;
  a.me = o.me;
  a.peer = o.peer;
  a.tag = o.tag;
  a.sidx = o.sidx;
  a.didx = o.didx;
  a.bases = o.bases;
}

// A graph-capturable self-message and its host-expected counterpart in the
// same launch (BatchOp::mate): both CTAs read the same device counters, so
// both reach the same verdict. Equal absolute keys: the receive takes the
// paired path (one copy, both completions, both ring slots consumed) and the
// send stands down; otherwise each runs the two-sided protocol.
__device__ void mate_match(const BatchOp& m, P2PArgs& a) {
  if (!(m.gflags & G_ON)) return;
  const volatile uint64_t* g = m.bases;
  const uint64_t mpseq = g[m.gp] + m.pseq;
  const uint32_t t = (uint32_t)g[m.gt] + (uint32_t)m.key;
  const uint64_t mkey = (m.key & 0xffffffff00000000ull) | t;
  if (mkey != a.key) return;
  if (a.is_recv) {
    a.paired = 1;
    a.pair_src = m.buf;
    a.pair_bytes = m.bytes;
    a.pair_done = m.my_done;
    a.pair_gen = m.my_gen;
    a.pair_mirror = m.post_mirror;
    a.pair_pseq = mpseq;
    a.staging = nullptr;
    a.stage_done = nullptr;
    a.stage_gen = 0;
  } else {
    a.mate_skip = 1;
  }
}

template <bool SYS>
__device__ void wait_all(const WaitEntry* w, int nwait, uint64_t* err_word, uint64_t spin_limit_ns) {
  for (int i = threadIdx.x; i < nwait; i += blockDim.x) {
    if (w[i].gen & kWaitConsume) {  // captured request: consume the completion (1 -> 0)
      if (!spin_ge<SYS>(w[i].flag, 1, err_word, spin_limit_ns, ERRW_WAIT_DONE)) break;
      Scope<SYS>::st_rlx(w[i].flag, 0);
    } else if (!spin_ge<SYS>(w[i].flag, w[i].gen, err_word, spin_limit_ns, ERRW_WAIT_DONE)) {
      break;
    }
  }
}

// Graph-capturable comms: the last CTA of a batch's final launch to finish
// advances the device sequence counters by the batch's per-counter counts
// (every CTA read them in load_op before, and the next launch of the stream
// reads them only after griddepcontrol.wait, i.e. after this grid).
template <int NOPS, int NWAIT>
__device__ void graph_advance(const BatchArgs<NOPS, NWAIT>& b) {
  if (!b.arrive || threadIdx.x != 0) return;
  __threadfence();  // my counter reads (load_op) before my arrival
  if (atomicAdd(b.arrive, 1u) != gridDim.x - 1) return;
  // Fire-and-forget reductions (no round trip each): the next reader is a
  // later launch of this stream, ordered behind this grid's completion.
  for (int i = 0; i < b.n; ++i) {
    const BatchOp& o = b.ops[i];
    if (!(o.gflags & G_ON)) continue;
    if (o.gflags & G_LASTP)
      atomicAdd(reinterpret_cast<unsigned long long*>(o.bases + o.gp), o.pseq + 1);
    if (o.gflags & G_LASTT)
      atomicAdd(reinterpret_cast<unsigned long long*>(o.bases + o.gt),
                (unsigned long long)(uint32_t)o.key + 1);
  }
  *reinterpret_cast<volatile uint32_t*>(b.arrive) = 0;
}

template <bool SYS, int NOPS, int NWAIT>
__global__ void __launch_bounds__(kThreads) k_batch(const BatchArgs<NOPS, NWAIT> b) {
  __shared__ Decision s_dc;
  pdl_wait();
  if (b.early) pdl_trigger();  // no grouped copy behind me: the next head kernel may park
  __shared__ P2PArgs a;
  if ((int)blockIdx.x < b.n_static) {
    const BatchOp& o = b.ops[blockIdx.x];
    if (threadIdx.x == 0) {
      load_op(o, b.spin_limit_ns, a);
      if (o.mate >= 0) mate_match(b.ops[o.mate], a);
    }
    __syncthreads();
    if (o.inl) proto_body<SYS, true>(a, s_dc);
    else proto_body<SYS, false>(a, s_dc);  // decision -> op record; triggers k_gcopy
  } else {
    // Dynamic-matching operations: the receives one after another in one
    // CTA, the sends in another, each in batch order. Matching serialises
    // them on the receiver's lock and tickets anyway, and receive tickets
    // (post order) and send tickets (per-destination order) only order ops
    // of one kind; one CTA per kind (instead of one spinning CTA per
    // operation) leaves the SMs to the other streams and ranks, and each
    // CTA holds at most one lock at a time.
    const int k = (int)blockIdx.x - b.n_static;
    const bool has_r = b.n_drecv > b.n_static, has_s = b.n > b.n_drecv;
    int lo = -1, hi = -1;
    if (has_r && k == 0) {
      lo = b.n_static;
      hi = b.n_drecv;
    } else if (has_s && k == (has_r ? 1 : 0)) {
      lo = b.n_drecv;
      hi = b.n;
    }
    if (lo >= 0) {
      for (int i = lo; i < hi; ++i) {
        const BatchOp& o = b.ops[i];
        if (threadIdx.x == 0) load_op(o, b.spin_limit_ns, a);
        __syncthreads();
        if (o.inl) proto_body<SYS, true>(a, s_dc);
        else proto_body<SYS, false>(a, s_dc);
        __syncthreads();
      }
    } else {
      wait_all<SYS>(b.w, b.nwait, b.err_word, b.spin_limit_ns);
    }
  }
  graph_advance(b);
}

// The lean k_batch: every operation inline, static matching,
// no staged send, no graph counters — the common small-message window. One
// CTA per operation plus the closing wait, as k_batch; its code is a fraction
// of k_batch's, so a launch on a cold SM fetches far fewer instructions.
template <bool SYS, int NOPS, int NWAIT>
__global__ void __launch_bounds__(kThreads) k_batch_tiny(const BatchArgs<NOPS, NWAIT> b) {
  __shared__ Decision s_dc;
  __shared__ P2PArgs a;
  pdl_wait();
  if (b.early) pdl_trigger();  // small grid, no grouped copy behind me: the next head kernel may park
  if ((int)blockIdx.x < b.n) {
    if (threadIdx.x == 0) load_op(b.ops[blockIdx.x], b.spin_limit_ns, a);
    __syncthreads();
    proto_body<SYS, true, true>(a, s_dc);
  } else {
    wait_all<SYS>(b.w, b.nwait, b.err_word, b.spin_limit_ns);
  }
}

// One operation, no wait (a blocking small send or receive: the ping-pong
// case): the operation is the kernel parameter itself, so its fields are
// read at compile-time offsets instead of through a run-time array index.
template <bool SYS>
__global__ void __launch_bounds__(kThreads) k_op1(const BatchOp o, const uint64_t spin_limit_ns) {
  __shared__ Decision s_dc;
  __shared__ P2PArgs a;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) load_op(o, spin_limit_ns, a);
  __syncthreads();
  proto_body<SYS, true, true>(a, s_dc);
}

// Grouped copy (PDL behind k_batch): CTA t finds its operation in the tile
// prefix table and streams one tile of it.
__global__ void __launch_bounds__(kCopyThreads, 2) k_gcopy(const GCopyArgs g) {
  if (!g.direct) pdl_wait();
  const uint32_t t = blockIdx.x;
  int lo = 0, hi = g.m - 1;
  while (lo < hi) {  // last j with tile_start[j] <= t
    const int mid = (lo + hi + 1) >> 1;
    if (g.tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  if (g.direct) {
    // launched once k_batch passed its own griddepcontrol.wait: everything
    // before k_batch in the stream is complete, so the sources are ready
    tile_copy(g.dst[lo], g.src[lo], g.nbytes[lo], t - g.tile_start[lo],
              g.tile_start[lo + 1] - g.tile_start[lo]);
    if (blockIdx.x == 0) pdl_wait();  // this grid completes after k_batch
    pdl_trigger();
    return;
  }
  const OpRecord* rec = g.rec[lo];
  const uint64_t action = rec->action;
  if (action == ACT_COPY || action == ACT_STAGE)
    tile_copy(reinterpret_cast<uint8_t*>(rec->dst), reinterpret_cast<const uint8_t*>(rec->src),
              rec->bytes, t - g.tile_start[lo], g.tile_start[lo + 1] - g.tile_start[lo]);
  pdl_trigger();
}

// Completions of the large operations (PDL behind k_gcopy), plus the wait
// that closed the batch (CTA n).
template <bool SYS, int NOPS, int NWAIT>
__global__ void __launch_bounds__(kThreads) k_gfin(const BatchArgs<NOPS, NWAIT> b) {
  pdl_wait();
  pdl_trigger();
  __shared__ Decision s_dc;
  if ((int)blockIdx.x < b.n) {
    const BatchOp& o = b.ops[blockIdx.x];
    if (!o.inl) {
      __shared__ P2PArgs a;
      if (threadIdx.x == 0) load_op(o, b.spin_limit_ns, a);
      __syncthreads();
      fin_body<SYS>(a, s_dc);
    }
  } else {
    wait_all<SYS>(b.w, b.nwait, b.err_word, b.spin_limit_ns);
  }
  graph_advance(b);
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

// Scalar element fold (unaligned buffers and tails): rank order 0..P-1.
template <int DT, int OP>
__device__ void reduce_elem(const uint64_t* sb, const uint64_t* outs, int nout, int P, uint64_t e) {
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

constexpr int kArThreads = 256;
constexpr int kArUnroll = 2;  // 8 KiB of every input per tile; kArGroup x 2 x 16 B in flight per thread
constexpr uint64_t kArTileVec = (uint64_t)kArThreads * kArUnroll;

// One tile [v0 + tile*kArTileVec, ...) of vectors within [v0, v1). Inputs
// are loaded kArGroup ranks at a time (all loads of a group in flight before
// any is folded) and folded strictly in rank order 0..P-1.
constexpr int kArGroup = 4;

template <int DT, int OP>
__device__ void reduce_tile(const uint64_t* sb, const uint64_t* outs, int nout, int P, uint64_t v0,
                            uint64_t v1, uint64_t tile) {
  const uint64_t base = v0 + tile * kArTileVec + threadIdx.x;
  Acc<DT> acc[kArUnroll];
  bool in[kArUnroll];
#pragma unroll
  for (int u = 0; u < kArUnroll; ++u) in[u] = base + u * kArThreads < v1;
  for (int q0 = 0; q0 < P; q0 += kArGroup) {
    uint4 x[kArGroup][kArUnroll];
#pragma unroll
    for (int g = 0; g < kArGroup; ++g) {
      if (q0 + g < P) {
        const uint4* sq = reinterpret_cast<const uint4*>(sb[q0 + g]);
#pragma unroll
        for (int u = 0; u < kArUnroll; ++u)
          if (in[u]) x[g][u] = sq[base + u * kArThreads];
      }
    }
#pragma unroll
    for (int g = 0; g < kArGroup; ++g) {
      if (q0 + g < P) {
#pragma unroll
        for (int u = 0; u < kArUnroll; ++u) {
          if (!in[u]) continue;
          if (q0 + g == 0) acc[u].init(x[g][u]);
          else acc[u].template add<OP>(x[g][u]);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kArUnroll; ++u) {
    if (!in[u]) continue;
    uint4 o = acc[u].out();
    for (int k = 0; k < nout; ++k) reinterpret_cast<uint4*>(outs[k])[base + u * kArThreads] = o;
  }
}

struct ArPlan {
  uint64_t v0, v1;  // my vector range
  uint64_t e0, e1;  // scalar element range handled here
  int nout;         // 1 (one-shot: my rbuf) or P (two-shot: every rbuf)
};

__device__ ArPlan ar_plan(const ARArgs& a, const uint64_t* sb, const uint64_t* rb, int algo) {
  ArPlan p;
  const int P = a.P;
  bool al = true;
  for (int q = 0; q < P; ++q) al &= ((sb[q] | rb[q]) & 15) == 0;
  const uint64_t nvec = al ? (a.count * (uint64_t)a.esize) >> 4 : 0;
  const uint64_t tail_e0 = (nvec << 4) / a.esize;
  if (algo == AR_TWOSHOT) {
    p.nout = P;
    uint64_t per = (nvec + P - 1) / P;
    p.v0 = umin(nvec, per * a.me);
    p.v1 = umin(nvec, p.v0 + per);
    if (al) {
      p.e0 = a.me == P - 1 ? tail_e0 : a.count;
      p.e1 = a.count;
    } else {
      uint64_t pe = (a.count + P - 1) / P;
      p.e0 = umin(a.count, pe * a.me);
      p.e1 = umin(a.count, p.e0 + pe);
    }
  } else {
    p.nout = 1;
    p.v0 = 0;
    p.v1 = nvec;
    p.e0 = tail_e0;
    p.e1 = a.count;
  }
  return p;
}

template <int DT, int OP>
__device__ void ar_tile(const ARArgs& a, const uint64_t* sb, const uint64_t* rb, int algo,
                        uint64_t tile, uint64_t ntiles) {
  ArPlan p = ar_plan(a, sb, rb, algo);
  const uint64_t* outs = p.nout == 1 ? rb + a.me : rb;  // shared-memory pointer table
  uint64_t nt_vec = (p.v1 - p.v0 + kArTileVec - 1) / kArTileVec;
  for (uint64_t t = tile; t < nt_vec; t += ntiles)
    reduce_tile<DT, OP>(sb, outs, p.nout, a.P, p.v0, p.v1, t);
  uint64_t gt = tile * blockDim.x + threadIdx.x, gn = ntiles * blockDim.x;
  for (uint64_t e = p.e0 + gt; e < p.e1; e += gn) reduce_elem<DT, OP>(sb, outs, p.nout, a.P, e);
}

// Collective epoch: host-assigned, or (graph-capturable comm) the device
// counter + 1, read after griddepcontrol.wait.
__device__ __forceinline__ uint64_t coll_epoch(const ARArgs& a) {
  return a.gseq ? *reinterpret_cast<volatile uint64_t*>(a.gseq) + 1 : a.epoch;
}
// ... advanced by the chain's last epoch reader (one thread, after the CTA
// has read it).
__device__ __forceinline__ void coll_advance(const ARArgs& a, int where) {
  __syncthreads();
  if (a.gseq && a.gbump == where && threadIdx.x == 0)  // read by a later launch only
    atomicAdd(reinterpret_cast<unsigned long long*>(a.gseq), 1ull);
}

// Entry: publish my buffers to every peer, wait for theirs, record them.
template <bool SYS>
__global__ void __launch_bounds__(32) k_ar_entry(const ARArgs a) {
  pdl_wait();
  const uint64_t epoch = coll_epoch(a);
  using M = Scope<SYS>;
  const int q = threadIdx.x;
  const int P = a.P;
  OpRecord* rec = a.rec;
  int ok = 1;
  uint64_t sb = 0, rb = 0;
  if (q < P) {
    CollSlot* dst = a.peer_in[q];
    M::st_rlx(&dst->sbuf, (uint64_t)a.sbuf);
    M::st_rlx(&dst->rbuf, (uint64_t)a.rbuf);
    M::st_rel(&dst->flag, epoch);
    ok = spin_ge<SYS>(&a.my_in[q].flag, epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL);
    sb = M::ld_rlx(&a.my_in[q].sbuf);
    rb = M::ld_rlx(&a.my_in[q].rbuf);
    switch (a.kind) {
      case CK_REDUCE_SCATTER:  // fold chunk `me` of every input into my buffer
        rec->coll[q] = sb + (uint64_t)a.me * a.chunk_bytes;
        if (q == a.me) rec->coll[kMaxCollRanks] = (uint64_t)a.rbuf;
        break;
      case CK_REDUCE:          // the root folds every input into its buffer
        rec->coll[q] = sb;
        if (q == a.me) rec->coll[kMaxCollRanks] = (uint64_t)a.rbuf;
        break;
      case CK_BCAST:           // one segment: the root's buffer -> mine
        if (q == a.root) rec->coll[0] = sb;
        if (q == a.me) rec->coll[kMaxCollRanks] = (uint64_t)a.rbuf;
        break;
      case CK_ALLGATHER:       // segment q: rank q's block -> my buffer at q
        rec->coll[q] = sb;
        rec->coll[kMaxCollRanks + q] = (uint64_t)a.rbuf + (uint64_t)q * a.chunk_bytes;
        break;
      case CK_ALLTOALL:        // segment q: block me of rank q's sendbuf -> my buffer at q
        rec->coll[q] = sb + (uint64_t)a.me * a.chunk_bytes;
        rec->coll[kMaxCollRanks + q] = (uint64_t)a.rbuf + (uint64_t)q * a.chunk_bytes;
        break;
      default:                 // allreduce: every member's buffers
        rec->coll[q] = sb;
        rec->coll[kMaxCollRanks + q] = rb;
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  // One-shot reads every peer's full buffer while peers write theirs: use
  // two-shot if any rank reduces in place.
  int inplace = __any_sync(0xffffffffu, q < P && sb == rb);
  if (q == 0) {
    uint64_t act = COLL_FAILED;
    if (ok) {
      switch (a.kind) {
        case CK_ALLREDUCE: act = (uint64_t)((inplace && P > 1) ? AR_TWOSHOT : a.algo) + 1; break;
        case CK_REDUCE: act = a.me == a.root ? COLL_FOLD : COLL_NOOP; rec->flags = P; break;
        case CK_REDUCE_SCATTER: act = COLL_FOLD; rec->flags = P; break;
        case CK_BCAST: act = a.me == a.root ? COLL_NOOP : COLL_COPY; rec->flags = 1; break;
        case CK_ALLGATHER: act = COLL_COPY; rec->flags = P; break;
        case CK_ALLTOALL: act = COLL_COPY; rec->flags = P; break;
        default: act = COLL_NOOP;
      }
    }
    rec->action = act;
  }
  coll_advance(a, GB_ENTRY);
  pdl_trigger();
}

// One instantiation per (dtype, op) so each gets its own register budget.
template <int DT, int OP>
__global__ void __launch_bounds__(kArThreads, (DT == AR_BF16 || DT == AR_F64) ? 3 : 4) k_ar_reduce(const ARArgs a) {
  pdl_wait();
  __shared__ uint64_t s_sb[kMaxCollRanks], s_rb[kMaxCollRanks];
  __shared__ uint64_t s_act;
  const OpRecord* rec = a.rec;
  if (threadIdx.x < a.P) {
    s_sb[threadIdx.x] = rec->coll[threadIdx.x];
    s_rb[threadIdx.x] = rec->coll[kMaxCollRanks + threadIdx.x];
  }
  if (threadIdx.x == 0) s_act = rec->action;
  __syncthreads();
  pdl_trigger();
  if (s_act == COLL_ONESHOT || s_act == COLL_TWOSHOT) {
    ar_tile<DT, OP>(a, s_sb, s_rb, (int)s_act - 1, blockIdx.x, gridDim.x);
  } else if (s_act == COLL_FOLD) {
    // Reduce / Reduce_scatter: a one-shot fold of rec->flags inputs (rank
    // order) into the single output coll[16]
    ARArgs f = a;
    f.P = (int)rec->flags;
    f.me = 0;
    if (threadIdx.x < f.P) {
      s_sb[threadIdx.x] = rec->coll[threadIdx.x];
      s_rb[threadIdx.x] = threadIdx.x == 0 ? rec->coll[kMaxCollRanks] : 0;
    }
    __syncthreads();
    ar_tile<DT, OP>(f, s_sb, s_rb, AR_ONESHOT, blockIdx.x, gridDim.x);
  }
}

// Bcast / Allgather (PDL behind k_ar_entry): rec->flags segments of
// a.chunk_bytes, coll[s] -> coll[16 + s]; CTA b copies tile b % tps of
// segment b / tps. In-place segments (src == dst) are skipped.
__global__ void __launch_bounds__(kCopyThreads, 2) k_coll_copy(const ARArgs a) {
  pdl_wait();
  const OpRecord* rec = a.rec;
  pdl_trigger();
  if (rec->action != COLL_COPY) return;
  const uint64_t tps = a.chunk_bytes ? (a.chunk_bytes + kTileVec * 16 - 1) / (kTileVec * 16) : 1;
  const uint64_t seg = blockIdx.x / tps, t = blockIdx.x % tps;
  if (seg >= rec->flags) return;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(rec->coll[seg]);
  uint8_t* dst = reinterpret_cast<uint8_t*>(rec->coll[kMaxCollRanks + seg]);
  tile_copy(dst, src, a.chunk_bytes, t, tps);
}

using ReduceKernel = void (*)(const ARArgs);

template <int DT>
static ReduceKernel reduce_kernel_op(int op) {
  if (op == AR_SUM) return k_ar_reduce<DT, AR_SUM>;
  if (op == AR_MAX) return k_ar_reduce<DT, AR_MAX>;
  return k_ar_reduce<DT, AR_MIN>;
}

static ReduceKernel reduce_kernel(int dtype, int op) {
  switch (dtype) {
    case AR_F32: return reduce_kernel_op<AR_F32>(op);
    case AR_BF16: return reduce_kernel_op<AR_BF16>(op);
    case AR_I32: return reduce_kernel_op<AR_I32>(op);
    default: return reduce_kernel_op<AR_F64>(op);
  }
}

// Small allreduce in ONE launch (bytes <= MPIX_ALLREDUCE_ONESHOT_MAX): one
// CTA runs the entry barrier, my two-shot chunk (read it from every input,
// fold in rank order, store it into every output — also correct in place),
// and the exit barrier. Replaces entry + reduce + exit for latency-bound
// sizes, where the host cost of three launches per rank dominated.
template <bool SYS>
__global__ void __launch_bounds__(kArThreads) k_ar_fused(const ARArgs a) {
  using M = Scope<SYS>;
  pdl_wait();
  pdl_trigger();
  const uint64_t epoch = coll_epoch(a);
  __shared__ uint64_t s_sb[kMaxCollRanks], s_rb[kMaxCollRanks];
  __shared__ int s_ok;
  const int q = threadIdx.x;
  const int P = a.P;
  if (q == 0) s_ok = 1;
  __syncthreads();
  if (q < P) {
    CollSlot* dst = a.peer_in[q];
    M::st_rlx(&dst->sbuf, (uint64_t)a.sbuf);
    M::st_rlx(&dst->rbuf, (uint64_t)a.rbuf);
    M::st_rel(&dst->flag, epoch);
    if (!spin_ge<SYS>(&a.my_in[q].flag, epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL))
      s_ok = 0;
    s_sb[q] = M::ld_rlx(&a.my_in[q].sbuf);
    s_rb[q] = M::ld_rlx(&a.my_in[q].rbuf);
  }
  __syncthreads();
  if (!s_ok) return;
  switch (a.dtype) {
    case AR_F32:
      if (a.op == AR_SUM) ar_tile<AR_F32, AR_SUM>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else if (a.op == AR_MAX) ar_tile<AR_F32, AR_MAX>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else ar_tile<AR_F32, AR_MIN>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      break;
    case AR_BF16:
      if (a.op == AR_SUM) ar_tile<AR_BF16, AR_SUM>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else if (a.op == AR_MAX) ar_tile<AR_BF16, AR_MAX>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else ar_tile<AR_BF16, AR_MIN>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      break;
    case AR_I32:
      if (a.op == AR_SUM) ar_tile<AR_I32, AR_SUM>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else if (a.op == AR_MAX) ar_tile<AR_I32, AR_MAX>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else ar_tile<AR_I32, AR_MIN>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      break;
    default:
      if (a.op == AR_SUM) ar_tile<AR_F64, AR_SUM>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else if (a.op == AR_MAX) ar_tile<AR_F64, AR_MAX>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      else ar_tile<AR_F64, AR_MIN>(a, s_sb, s_rb, AR_TWOSHOT, 0, 1);
      break;
  }
  __syncthreads();
  if (P > 1) {
    if (q == 0) M::fence_ar();
    __syncthreads();
    if (q < P) {
      M::st_rlx(a.peer_exit[q], epoch);
      spin_ge<SYS>(&a.my_exit[q], epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL);
    }
  }
  coll_advance(a, GB_EXIT);
}

// Exit: tell every peer I am done with its buffers; wait for all of them.
template <bool SYS>
__global__ void __launch_bounds__(32) k_ar_exit(const ARArgs a) {
  pdl_wait();
  pdl_trigger();
  using M = Scope<SYS>;
  const int q = threadIdx.x;
  if (a.rec->action == 0) return;
  const uint64_t epoch = coll_epoch(a);
  M::fence_ar();
  if (q < a.P) {
    M::st_rlx(a.peer_exit[q], epoch);
    spin_ge<SYS>(&a.my_exit[q], epoch, a.err_word, a.spin_limit_ns, ERRW_WAIT_COLL);
  }
  coll_advance(a, GB_EXIT);
}

// ---------------------------------------------------------------------------
// Host launchers (return the number of kernels launched, -1 on error)
// ---------------------------------------------------------------------------
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), int grid, int block, cudaStream_t s,
                              Args&&... args) {
  // MPIX_PDL=0: plain launches (A/B of programmatic dependent launch)
  static const bool pdl = [] {
    const char* v = std::getenv("MPIX_PDL");
    return !(v && v[0] == '0');
  }();
  if (!pdl) {
    k<<<grid, block, 0, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Operation head kernels (k_proto, k_batch, k_ar_entry) start with
// griddepcontrol.wait, so they may be launched programmatically behind the
// previous kernel of the stream and park there until it completes. Only
// small grids do so: parked CTAs hold SM slots, and at most kEarlyHeadCTAs
// per stream may wait behind a kernel that spins on a peer.
constexpr int kEarlyHeadCTAs = 4;

template <typename... KArgs, typename... Args>
static cudaError_t launch_head(void (*k)(KArgs...), int grid, int block, cudaStream_t s,
                               Args&&... args) {
  if (grid <= kEarlyHeadCTAs) return launch_pdl(k, grid, block, s, std::forward<Args>(args)...);
  k<<<grid, block, 0, s>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
}

uint64_t p2p_copy_grid(uint64_t bytes) {
  uint64_t tile = kTileVec * 16;
  uint64_t g = (bytes + tile - 1) / tile;
  if (g > (1ull << 30)) g = 1ull << 30;
  return g < 1 ? 1 : g;
}

int launch_p2p(const P2PArgs& a, bool sys, bool inl, uint64_t grid, cudaStream_t s,
               cudaEvent_t copy_ev0, cudaEvent_t copy_ev1) {
  if (inl) {
    cudaError_t e = sys ? launch_pdl(k_proto<true, true>, 1, kThreads, s, a)
                        : launch_pdl(k_proto<false, true>, 1, kThreads, s, a);
    return e == cudaSuccess ? 1 : -1;
  }
  {
    cudaError_t e = sys ? launch_pdl(k_proto<true, false>, 1, kThreads, s, a)
                        : launch_pdl(k_proto<false, false>, 1, kThreads, s, a);
    if (e != cudaSuccess) return -1;
  }
  if (copy_ev0) cudaEventRecord(copy_ev0, s);  // timing probe (bench roofline) only
  if (launch_pdl(k_copy, (int)grid, kCopyThreads, s, a) != cudaSuccess) return -1;
  if (copy_ev1) cudaEventRecord(copy_ev1, s);
  cudaError_t e = sys ? launch_pdl(k_fin<true>, 1, kThreads, s, a)
                      : launch_pdl(k_fin<false>, 1, kThreads, s, a);
  return e == cudaSuccess ? 3 : -1;
}

template <int NOPS, int NWAIT>
static int launch_batch_t(const BatchOp* ops, int n, const WaitEntry* w, int nwait,
                          uint64_t* err_word, uint64_t spin_limit_ns, bool sys, cudaStream_t s,
                          cudaEvent_t ev0, cudaEvent_t ev1, uint32_t* arrive) {
  BatchArgs<NOPS, NWAIT> b;
  b.arrive = arrive;  // graph counters: advanced by the final launch
  b.n = n;
  b.nwait = nwait;
  b.spin_limit_ns = spin_limit_ns;
  b.err_word = err_word;
  // static-matching operations first (one CTA each), then the dynamic ones
  // (one sequential CTA), keeping batch order within each group
  int k = 0;
  int newidx[NOPS];
  for (int i = 0; i < n; ++i) {
    newidx[i] = -1;
    if (!ops[i].dyn) {
      newidx[i] = k;
      b.ops[k++] = ops[i];
    }
  }
  b.n_static = k;
  for (int i = 0; i < k; ++i)  // mates refer to positions in this launch
    if (b.ops[i].mate >= 0) b.ops[i].mate = (int16_t)newidx[b.ops[i].mate];
  // Dynamic receives, then dynamic sends, batch order in each — unless a
  // blocking receive closes the batch: it may wait in k_batch for a push
  // that its send, had it run second in the other CTA, would leave to the
  // k_gcopy behind it; in batch order in one CTA the earlier sends run
  // first and the receive pulls instead.
  bool blocking_recv = false;
  for (int i = 0; i < n; ++i) blocking_recv |= ops[i].dyn && ops[i].is_recv && ops[i].blocking;
  for (int i = 0; i < n; ++i)
    if (ops[i].dyn && (blocking_recv || ops[i].is_recv)) b.ops[k++] = ops[i];
  b.n_drecv = k;
  for (int i = 0; i < n; ++i)
    if (ops[i].dyn && !blocking_recv && !ops[i].is_recv) b.ops[k++] = ops[i];
  const int head_ctas = b.n_static + (b.n_drecv > b.n_static ? 1 : 0) + (n > b.n_drecv ? 1 : 0);
  for (int i = 0; i < nwait; ++i) b.w[i] = w[i];
  GCopyArgs g;
  g.m = 0;
  g.direct = 1;
  uint64_t tiles = 0;
  for (int i = 0; i < n; ++i) {
    const BatchOp& o = b.ops[i];
    if (o.inl) continue;
    g.tile_start[g.m] = (uint32_t)tiles;
    g.rec[g.m] = o.rec;
    g.direct &= o.paired ? 1 : 0;
    g.src[g.m] = o.paired ? o.pr.src : nullptr;
    g.dst[g.m] = o.buf;
    g.nbytes[g.m] = o.paired ? (o.pr.bytes < o.bytes ? o.pr.bytes : o.bytes) : 0;
    tiles += p2p_copy_grid(o.bytes);
    ++g.m;
  }
  g.tile_start[g.m] = (uint32_t)tiles;
  for (int i = 0; i < n; ++i) b.ops[i].early = tiles <= kEarlyTriggerTiles;
  if (g.m == 0) {  // inline operations only: one launch, the wait included
    const int grid = head_ctas + (nwait > 0 ? 1 : 0);
    // let the stream's next head kernel launch (and park at
    // griddepcontrol.wait) early only behind a small grid: a parked
    // window-sized grid would hold SMs the peers' operations need while this
    // one's wait spins
    b.early = grid <= kEarlyHeadCtas ? 1 : 0;
    bool tiny = !arrive && b.n_static == n;
    for (int i = 0; i < n && tiny; ++i) {
      const BatchOp& o = b.ops[i];
      tiny = !o.paired && !(o.gflags & G_ON) && !(!o.is_recv && o.mode == MODE_STAGED);
    }
    static const bool op1 = [] {
      const char* v = std::getenv("MPIX_OP1");
      return !(v && v[0] == '0');
    }();
    if (tiny && op1 && n == 1 && nwait == 0 && !arrive) {
      cudaError_t e = sys ? launch_head(k_op1<true>, 1, kThreads, s, b.ops[0], spin_limit_ns)
                          : launch_head(k_op1<false>, 1, kThreads, s, b.ops[0], spin_limit_ns);
      return e == cudaSuccess ? 1 : -1;
    }
    if (tiny) {
      cudaError_t e = sys ? launch_head(k_batch_tiny<true, NOPS, NWAIT>, grid, kThreads, s, b)
                          : launch_head(k_batch_tiny<false, NOPS, NWAIT>, grid, kThreads, s, b);
      return e == cudaSuccess ? 1 : -1;
    }
    cudaError_t e = sys ? launch_head(k_batch<true, NOPS, NWAIT>, grid, kThreads, s, b)
                        : launch_head(k_batch<false, NOPS, NWAIT>, grid, kThreads, s, b);
    return e == cudaSuccess ? 1 : -1;
  }
  // decisions (the wait moves to k_gfin) -> grouped copy -> completions + wait
  const int nw = b.nwait;
  b.nwait = 0;
  b.early = g.direct;  // a direct copy grid starts as soon as k_batch has waited
  b.arrive = nullptr;  // the counters advance in k_gfin
  {
    cudaError_t e = sys ? launch_head(k_batch<true, NOPS, NWAIT>, head_ctas, kThreads, s, b)
                        : launch_head(k_batch<false, NOPS, NWAIT>, head_ctas, kThreads, s, b);
    if (e != cudaSuccess) return -1;
  }
  b.nwait = nw;
  b.arrive = arrive;
  if (ev0) cudaEventRecord(ev0, s);  // timing probe (bench roofline) only
  if (launch_pdl(k_gcopy, (int)tiles, kCopyThreads, s, g) != cudaSuccess) return -1;
  if (ev1) cudaEventRecord(ev1, s);
  const int fgrid = n + (nw > 0 ? 1 : 0);
  cudaError_t e = sys ? launch_pdl(k_gfin<true, NOPS, NWAIT>, fgrid, kThreads, s, b)
                      : launch_pdl(k_gfin<false, NOPS, NWAIT>, fgrid, kThreads, s, b);
  return e == cudaSuccess ? 3 : -1;
}

// Parameter-size classes: the whole struct is copied into the launch, so
// small batches use the small instantiations.
int launch_batch(const BatchOp* ops, int n, const WaitEntry* w, int nwait, uint64_t* err_word,
                 uint64_t spin_limit_ns, bool sys, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                 uint32_t* arrive) {
  if (n <= 0 && nwait <= 0) return 0;
  if (n <= 4 && nwait <= 8)
    return launch_batch_t<4, 8>(ops, n, w, nwait, err_word, spin_limit_ns, sys, s, ev0, ev1, arrive);
  if (n <= 16 && nwait <= 32)
    return launch_batch_t<16, 32>(ops, n, w, nwait, err_word, spin_limit_ns, sys, s, ev0, ev1, arrive);
  if (n <= 64 && nwait <= kBatchWaits)
    return launch_batch_t<64, kBatchWaits>(ops, n, w, nwait, err_word, spin_limit_ns, sys, s, ev0,
                                           ev1, arrive);
  if (n <= kBatchOps && nwait <= kBatchWaits)
    return launch_batch_t<kBatchOps, kBatchWaits>(ops, n, w, nwait, err_word, spin_limit_ns, sys, s,
                                                  ev0, ev1, arrive);
  return -1;
}

// One CTA per tile when it moves enough bytes (P inputs + outputs of
// kArTileVec x 16 B each); with few ranks a CTA takes several tiles so CTA
// launch does not dominate (P = 1: 4 tiles = 32 KiB in + 32 KiB out).
int launch_collective(const ARArgs& a, bool sys, uint64_t work_grid, cudaStream_t s) {
  {
    cudaError_t e = sys ? launch_pdl(k_ar_entry<true>, 1, 32, s, a)
                        : launch_pdl(k_ar_entry<false>, 1, 32, s, a);
    if (e != cudaSuccess) return -1;
  }
  int nk = 1;
  if (a.kind == CK_BCAST || a.kind == CK_ALLGATHER || a.kind == CK_ALLTOALL) {
    if (launch_pdl(k_coll_copy, (int)work_grid, kCopyThreads, s, a) != cudaSuccess) return -1;
    ++nk;
  } else if (a.kind == CK_REDUCE || a.kind == CK_REDUCE_SCATTER) {
    if (launch_pdl(reduce_kernel(a.dtype, a.op), (int)work_grid, kArThreads, s, a) != cudaSuccess)
      return -1;
    ++nk;
  }
  if (a.P > 1) {
    cudaError_t e = sys ? launch_pdl(k_ar_exit<true>, 1, 32, s, a)
                        : launch_pdl(k_ar_exit<false>, 1, 32, s, a);
    if (e != cudaSuccess) return -1;
    ++nk;
  }
  return nk;
}

uint64_t ar_reduce_grid(uint64_t work_bytes, int P) {
  const uint64_t tile = kArTileVec * 16;
  const uint64_t tiles = (work_bytes + tile - 1) / tile;
  const uint64_t per = P >= 4 ? 1 : (4 + P - 1) / P;
  uint64_t g = (tiles + per - 1) / per;
  if (g > (1ull << 20)) g = 1ull << 20;
  return g < 1 ? 1 : g;
}

int launch_allreduce(const ARArgs& a, bool sys, uint64_t grid, cudaStream_t s, bool fused) {
  if (fused) {
    cudaError_t e = sys ? launch_pdl(k_ar_fused<true>, 1, kArThreads, s, a)
                        : launch_pdl(k_ar_fused<false>, 1, kArThreads, s, a);
    return e == cudaSuccess ? 1 : -1;
  }
  {
    cudaError_t e = sys ? launch_pdl(k_ar_entry<true>, 1, 32, s, a)
                        : launch_pdl(k_ar_entry<false>, 1, 32, s, a);
    if (e != cudaSuccess) return -1;
  }
  if (launch_pdl(reduce_kernel(a.dtype, a.op), (int)grid, kArThreads, s, a) != cudaSuccess) return -1;
  if (a.P > 1) {
    cudaError_t e = sys ? launch_pdl(k_ar_exit<true>, 1, 32, s, a)
                        : launch_pdl(k_ar_exit<false>, 1, 32, s, a);
    if (e != cudaSuccess) return -1;
    return 3;
  }
  return 2;
}

// The reduce stage alone (profiling / roofline probe): P input buffers and
// P output buffers on this GPU, as rank `me` of a P-rank allreduce would see
// them after the entry barrier. `rec` is a device OpRecord the caller owns.
int launch_reduce_only(const uint64_t* sb, const uint64_t* rb, int P, int me, uint64_t count,
                       int esize, int dtype, int op, int algo, OpRecord* rec, cudaStream_t s) {
  if (P < 1 || P > kMaxCollRanks) return -1;
  OpRecord h = {};
  for (int q = 0; q < P; ++q) {
    h.coll[q] = sb[q];
    h.coll[kMaxCollRanks + q] = rb[q];
  }
  h.action = (uint64_t)algo + 1;
  if (cudaMemcpyAsync(rec, &h, sizeof(h), cudaMemcpyHostToDevice, s) != cudaSuccess) return -1;
  ARArgs a = {};
  a.count = count;
  a.esize = esize;
  a.dtype = dtype;
  a.op = op;
  a.algo = algo;
  a.P = P;
  a.me = me;
  a.rec = rec;
  uint64_t bytes = count * (uint64_t)esize;
  uint64_t work = algo == AR_TWOSHOT ? (bytes + P - 1) / P : bytes;
  reduce_kernel(dtype, op)<<<(unsigned)ar_reduce_grid(work, P), kArThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// Co-residency probe: can two spinning single-CTA kernels of different
// streams of one device run at the same time? A waits (bounded) for a flag B
// sets; B is launched after A. Under kernel serialisation (ncu's launch
// capture, some sanitizer modes) A times out. Ranks sharing a GPU need
// co-residency for every cross-rank wait of their collectives.
__global__ void k_cores_wait(volatile uint64_t* f, uint64_t limit_ns) {
  const uint64_t t0 = globaltimer();
  while (f[0] == 0) {
    if (globaltimer() - t0 > limit_ns) {
      f[1] = 2;
      return;
    }
    __nanosleep(256);
  }
  f[1] = 1;
}
__global__ void k_cores_set(volatile uint64_t* f) {
  __threadfence();
  f[0] = 1;
}

int coresident_probe(int device, int* ok) {
  *ok = 0;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  uint64_t* h = nullptr;
  cudaStream_t a = nullptr, b = nullptr;
  int rc = -1;
  if (cudaHostAlloc((void**)&h, 64, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess &&
      cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking) == cudaSuccess &&
      cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking) == cudaSuccess) {
    h[0] = h[1] = 0;
    uint64_t* d = nullptr;
    cudaHostGetDevicePointer((void**)&d, h, 0);
    k_cores_wait<<<1, 1, 0, a>>>(d, 200ull * 1000 * 1000);
    k_cores_set<<<1, 1, 0, b>>>(d);
    if (cudaStreamSynchronize(a) == cudaSuccess && cudaStreamSynchronize(b) == cudaSuccess) {
      *ok = ((volatile uint64_t*)h)[1] == 1;
      rc = 0;
    }
  }
  if (a) cudaStreamDestroy(a);
  if (b) cudaStreamDestroy(b);
  if (h) cudaFreeHost(h);
  cudaGetLastError();
  cudaSetDevice(prev);
  return rc;
}

// Force-load every kernel of this module on the current device. Under CUDA
// lazy loading the first launch of a kernel waits for the device while a
// spinning handshake kernel may be waiting for exactly that launch (a peer's
// kernel), so everything is loaded up front.
int preload_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaSuccess;
  const void* ks[] = {
      (const void*)k_proto<true, true>, (const void*)k_proto<true, false>,
      (const void*)k_proto<false, true>, (const void*)k_proto<false, false>,
      (const void*)k_copy, (const void*)k_fin<true>, (const void*)k_fin<false>,
      (const void*)k_ar_entry<true>, (const void*)k_ar_entry<false>,
      (const void*)k_ar_exit<true>, (const void*)k_ar_exit<false>,
      (const void*)k_ar_fused<true>, (const void*)k_ar_fused<false>, (const void*)k_coll_copy,
      (const void*)k_batch<true, 4, 8>, (const void*)k_batch<false, 4, 8>,
      (const void*)k_batch<true, 16, 32>, (const void*)k_batch<false, 16, 32>,
      (const void*)k_batch<true, 64, kBatchWaits>, (const void*)k_batch<false, 64, kBatchWaits>,
      (const void*)k_gfin<true, 64, kBatchWaits>, (const void*)k_gfin<false, 64, kBatchWaits>,
      (const void*)k_batch<true, kBatchOps, kBatchWaits>,
      (const void*)k_batch<false, kBatchOps, kBatchWaits>,
      (const void*)k_gfin<true, 4, 8>, (const void*)k_gfin<false, 4, 8>,
      (const void*)k_gfin<true, 16, 32>, (const void*)k_gfin<false, 16, 32>,
      (const void*)k_gfin<true, kBatchOps, kBatchWaits>,
      (const void*)k_gfin<false, kBatchOps, kBatchWaits>, (const void*)k_gcopy,
      (const void*)k_cores_wait, (const void*)k_cores_set,
      (const void*)k_op1<true>, (const void*)k_op1<false>,
      (const void*)k_batch_tiny<true, 4, 8>, (const void*)k_batch_tiny<false, 4, 8>,
      (const void*)k_batch_tiny<true, 16, 32>, (const void*)k_batch_tiny<false, 16, 32>,
      (const void*)k_batch_tiny<true, 64, kBatchWaits>, (const void*)k_batch_tiny<false, 64, kBatchWaits>,
      (const void*)k_batch_tiny<true, kBatchOps, kBatchWaits>,
      (const void*)k_batch_tiny<false, kBatchOps, kBatchWaits>};
  for (const void* k : ks) {
    cudaError_t r = cudaFuncGetAttributes(&fa, k);
    if (r != cudaSuccess) e = r;
  }
  for (int dt : {AR_I32, AR_F32, AR_BF16, AR_F64})
    for (int op : {AR_SUM, AR_MAX, AR_MIN}) {
      cudaError_t r = cudaFuncGetAttributes(&fa, (const void*)reduce_kernel(dt, op));
      if (r != cudaSuccess) e = r;
    }
  return e == cudaSuccess ? 0 : -1;
}

}  // namespace mpix
