// mpix_internal.h — structures shared by the host runtime (mpix_runtime.cpp)
// and the sm_100a kernels (mpix_kernels.cu).
//
// The reference moves a message through a loopback byte channel and a host
// matching engine (proj/src/wire.cpp:53-73, proj/src/endpoint.cpp:15-69).
// Here every rank owns, per communicator, one "region" of device memory on
// its GPU. Peers reach it over NVLink (or directly when they share the GPU).
// A message s->d meets its receive through two descriptor rings:
//
//   SR(s->d)  in d's region, written by s   send descriptors   (d scans it)
//   RR(s->d)  in s's region, written by d   receive descriptors (s scans it)
//
// Both sides scan first, then post their own descriptor, fence, and rescan
// (store-buffering / Dekker). The arbitration word is the send descriptor's
// state: whoever moves it POSTED->TAKEN with a system-scope CAS is the
// "second arriver" and performs the copy inside its own in-stream kernel —
// push (sender) or pull (receiver). No host thread and no progress engine.
#pragma once

#include <stdint.h>
#include <cuda_runtime.h>

namespace mpix {

constexpr int kThreads = 512;          // threads per CTA for every op kernel
constexpr int kMaxCollRanks = 16;      // max communicator size for Allreduce
constexpr uint64_t kOpRecords = 65536; // op-record ring entries per rank (32 MiB; bounds in-flight large ops)
// Completion pool of a rank: kReqSlots reusable request words, then
// kGraphReqs words of captured requests (never reused), then two status
// planes at a fixed byte offset from any completion word w: w + kStatusOff =
// delivered bytes | truncated << 63, w + 2 * kStatusOff = source << 32 | tag,
// written by whoever completes a receive (the reference's Status,
// request.hpp:13-19, filled by deliver, endpoint.cpp:17-24).
constexpr uint64_t kReqSlots = 1ull << 20;
constexpr uint64_t kGraphReqs = 1ull << 16;
constexpr uint64_t kDoneWords = kReqSlots + kGraphReqs;
constexpr uint64_t kStatusOff = kDoneWords * 8;
constexpr uint64_t kTruncBit = 1ull << 63;

enum : uint64_t { ST_FREE = 0, ST_POSTED = 1, ST_TAKEN = 2 };
// State bit of a posted send descriptor whose payload travels inside it as
// flag-in-data words (sends of <= kLLBytes). Scans match
// (state & ~ST_LL) == ST_POSTED.
constexpr uint64_t ST_LL = 0x10;
// With ST_LL: the payload is in the sender's eager slot as LL words (4
// bytes + the post's flag each) — an eager send of 13 B .. E.
constexpr uint64_t ST_LLE = 0x20;
constexpr uint64_t kLLBytes = 12;
// An LL word: 4 payload bytes | flag << 32, flag = 0x80000000 | (pseq &
// 0x7fffffff). A reader that sees the flag of the post's own pseq in every
// word holds that post's payload, whatever order the words landed in; no
// stale word carries it (the slot's previous occupant was pseq - R, and
// descriptor fields of other posts never have bit 63 set). The sender's
// completion word and value (< 2^48) travel with a 16-bit check of the same
// kind in their top bits (ll_chk).
__host__ __device__ inline uint32_t ll_flag(uint64_t pseq) {
  return 0x80000000u | (uint32_t)(pseq & 0x7fffffffu);
}
__host__ __device__ inline uint64_t ll_word(uint32_t data, uint32_t flag) {
  return ((uint64_t)flag << 32) | data;
}
__host__ __device__ inline uint64_t ll_chk(uint64_t pseq) { return (0x8000ull | (pseq & 0x7fffull)) << 48; }
constexpr uint64_t kLLPtrMask = (1ull << 48) - 1;
// Codes a kernel stores in the rank's watchdog word before giving up
// (the host turns any of them into the sticky MPIX_ERR_TIMEOUT / _DEVICE).
enum : uint64_t { ERRW_WAIT_SLOT = 1, ERRW_WAIT_DONE = 2, ERRW_WAIT_COLL = 3, ERRW_PROTOCOL = 4 };

__host__ __device__ inline uint64_t st_word(uint64_t pseq, uint64_t st) {
  return (pseq << 8) | st;
}

// One ring slot. Mirrors the fields of the reference's Envelope/RecvDesc
// (wire.hpp:13-21, endpoint.hpp:35-40) that matching needs: the (tag, seq)
// key replaces (context, source, tag) because the ring is per (comm, pair).
struct alignas(64) SlotDesc {
  uint64_t state;      // (pair_seq << 8) | ST_*
  uint64_t key;        // ((uint32)tag << 32) | per-(pair,tag) sequence
  uint64_t addr;       // send: payload address; recv: destination buffer
  uint64_t bytes;      // send: payload length; recv: capacity
  uint64_t done_addr;  // poster's completion word (0 = none)
  uint64_t done_val;   // value to store there
  uint64_t pad[2];
};
static_assert(sizeof(SlotDesc) == 64, "slot is one 64-B line");

struct alignas(32) CollSlot {
  uint64_t flag;  // allreduce epoch this peer has entered
  uint64_t sbuf;  // its send buffer
  uint64_t rbuf;  // its receive buffer
  uint64_t pad;
};

// Layout of one rank's per-communicator region.
// Per-(direction, peer, tag) match-sequence counters a graph-capturable
// communicator may use (distinct (peer, tag) keys over its lifetime).
constexpr uint32_t kGraphTagCounters = 1024;

struct RegionLayout {
  int P;       // communicator size
  int R;       // ring slots per ordered pair
  uint64_t E;  // eager bytes per slot

  __host__ __device__ uint64_t ring_bytes() const {
    return (uint64_t)R * sizeof(SlotDesc);
  }
  // send descriptors posted by peer q (messages q -> me)
  __host__ __device__ uint64_t sr(int q) const { return (uint64_t)q * ring_bytes(); }
  // receive descriptors posted by peer q (messages me -> q)
  __host__ __device__ uint64_t rr(int q) const {
    return (uint64_t)P * ring_bytes() + (uint64_t)q * ring_bytes();
  }
  // free-mirror of MY send slots inside q's SR(me->q) ring
  __host__ __device__ uint64_t sr_free(int q) const {
    return 2ull * P * ring_bytes() + (uint64_t)q * R * 8;
  }
  // free-mirror of MY receive slots inside q's RR(q->me) ring
  __host__ __device__ uint64_t rr_free(int q) const {
    return 2ull * P * ring_bytes() + (uint64_t)P * R * 8 + (uint64_t)q * R * 8;
  }
  __host__ __device__ uint64_t coll_in(int q) const {
    return 2ull * P * ring_bytes() + 2ull * P * R * 8 + (uint64_t)q * sizeof(CollSlot);
  }
  __host__ __device__ uint64_t coll_exit(int q) const {
    return coll_in(P) + (uint64_t)q * 8;
  }
  // Dynamic matching (MPIX_MATCHING=dynamic, wildcard receives): the
  // region bases of every member, then my matching domain (lock, receive
  // ticket, arrival counter, per-source send tickets) and my posted-receive
  // queue of R entries.
  __host__ __device__ uint64_t bases() const { return (coll_exit(P) + 63) & ~63ull; }
  __host__ __device__ uint64_t dom() const { return (bases() + 8ull * P + 63) & ~63ull; }
  __host__ __device__ uint64_t dom_lock() const { return dom(); }
  __host__ __device__ uint64_t dom_next_rpost() const { return dom() + 8; }
  __host__ __device__ uint64_t dom_arrival() const { return dom() + 16; }
  __host__ __device__ uint64_t dom_next_spost(int q) const { return dom() + 64 + 8ull * q; }
  __host__ __device__ uint64_t pq() const { return (dom_next_spost(P) + 63) & ~63ull; }
  // Device sequence counters (graph-capturable communicators, DESIGN.md
  // §3b): [0,P) send pair sequences, [P,2P) receive pair sequences, 2P the
  // collective epoch, then kGraphTagCounters per-(direction, peer, tag)
  // match sequences. Only my own kernels touch them.
  __host__ __device__ uint64_t gseq() const { return (pq() + ring_bytes() + 63) & ~63ull; }
  __host__ __device__ uint64_t eager_base() const {
    return (gseq() + 8ull * (2ull * P + 1 + kGraphTagCounters) + 255) & ~255ull;
  }
  // eager payload ring of messages q -> me
  // an eager slot holds E payload bytes, or E bytes as LL words (2E)
  __host__ __device__ uint64_t eager(int q) const {
    return eager_base() + (uint64_t)q * R * 2 * E;
  }
  __host__ __device__ uint64_t total() const { return eager(P); }
};

// Grid-wide decision record for multi-CTA operations (CTA 0 decides, the
// others follow). One per launched multi-CTA op, in a per-rank ring.
struct alignas(64) OpRecord {
  uint64_t opid;     // published last (release) by CTA 0
  uint64_t action;   // ACT_*
  uint64_t src;
  uint64_t dst;
  uint64_t bytes;
  uint32_t counter;  // CTAs finished copying
  uint32_t nfin;
  uint64_t fin_addr[8];  // completion stores (k_fin): [0,2) slot frees,
  uint64_t fin_val[8];   // [2,8) mirrors and done words
  uint64_t coll[2 * kMaxCollRanks];  // allreduce: peers' sbuf / rbuf
  uint64_t flags;
  uint64_t stage_ptr, stage_done, stage_gen;  // staged send: buffer + release
  uint64_t stat_addr, stat_bytes, stat_srctag; // status of the completed receive (kStatusOff)
};

enum : uint64_t { ACT_NONE = 0, ACT_COPY = 1, ACT_STAGE = 2, ACT_LLE = 3 };

// Per-op trace record (MPIX_TRACE=1), written by the op's kernels.
// t[]: clock64 stamps of k_proto phases: 0 start, 1 first scan done,
// 2 posted (or decided without posting), 3 final decision, 4 copy done,
// 5 completion stores done. g0/g1: globaltimer at k_proto start/end.
struct TraceRec {
  uint64_t seq;     // host op sequence (0 = unused)
  uint64_t info;    // is_recv | mode << 4 | inline << 8 | action << 12
  uint64_t bytes;
  uint64_t key;
  uint64_t t[6];
  uint64_t g0, g1;
  uint64_t pad[4];
};
static_assert(sizeof(TraceRec) == 128, "trace record is 128 B");
constexpr uint64_t kTraceRecs = 4096;

enum SendMode : int { MODE_ISEND = 0, MODE_EAGER = 1, MODE_STAGED = 2 };

struct P2PArgs {
  int is_recv;
  int mode;       // SendMode (send side)
  int blocking;   // recv: the kernel waits for its own completion
  int R;
  uint64_t key;
  uint64_t pseq;       // my pair sequence -> post slot pseq % R
  SlotDesc* post_ring; // ring I post into (peer memory)
  uint64_t* post_mirror;  // my free-mirror for that ring (local)
  SlotDesc* scan_ring;    // ring I scan (local)
  uint64_t* scan_mirror;  // peer's free-mirror for the scanned ring (peer)
  uint8_t* eager_ring;    // send: SR's eager payload ring (peer memory)
  uint64_t E;
  uint8_t* buf;
  uint64_t bytes;         // send: length; recv: capacity
  uint8_t* staging;       // MODE_STAGED
  uint64_t* my_done;      // my request's completion word (local)
  uint64_t my_gen;
  uint64_t* stage_done;   // MODE_STAGED: released by the consumer of staging
  uint64_t stage_gen;
  // MODE_STAGED with staging == null: claim a slot of the rank's device
  // staging arena in the kernel, only if the receive is not posted yet
  uint8_t* arena;
  uint64_t* arena_state;  // arena_slots words: even = free
  uint32_t arena_slots;
  uint64_t arena_chunk;
  OpRecord* rec;
  uint64_t opid;
  uint64_t* err_word;     // per-rank error word (watchdog)
  uint64_t spin_limit_ns; // 0 = wait forever
  TraceRec* trace;        // MPIX_TRACE: this op's trace record, else null
  uint64_t trace_seq;     // its host sequence number (the record's head)
  int ll;                 // MPIX_LL: LL sends (<= kLLBytes) + polling blocking receives
  int early_trigger;      // large blocking receive: let the copy grid launch before
                          // waiting for the sender (only when the grid is small)
  // dynamic matching (dyn = 1): pseq is the receive ticket on the receive
  // side; peer / tag may be -1 (ANY_SOURCE / ANY_TAG) on receives
  int dyn, P, me, peer, tag;
  int sidx, didx;         // multiplex stream indices (-2 none, -1 ANY source index)
  uint64_t* bases;        // region bases of the comm's members (in my region)
  // paired self-message (host-matched in a batch): this receive also carries
  // its send; no descriptors, only both ring slots' retirement and the copy
  int paired;
  const uint8_t* pair_src;
  uint64_t pair_bytes;
  uint64_t* pair_done;
  uint64_t pair_gen;
  uint64_t* pair_mirror;
  uint64_t pair_pseq;
  int greset;             // captured blocking receive: zero my_done before posting
  int mate_skip;          // a device-matched send: its receive does the paired copy
};

// Copy grids up to this many CTAs may be launched (and park at
// griddepcontrol.wait) while a blocking receive waits for its sender; larger
// ones launch after it, so a parked grid never fills the GPU.
constexpr uint64_t kEarlyTriggerTiles = 64;
// A head kernel (k_batch) of at most this many CTAs lets the stream's next
// head kernel launch early (programmatic dependent launch); larger ones
// trigger at exit.
constexpr int kEarlyHeadCtas = 8;

struct WaitEntry {
  uint64_t* flag;
  uint64_t gen;  // kWaitConsume: captured request, wait for 1 then reset to 0
};
constexpr uint64_t kWaitConsume = 1ull << 63;
enum : uint8_t { G_ON = 1, G_LASTP = 2, G_LASTT = 4, G_RESET = 8 };

// One operation of a coalesced batch (k_batch): the P2PArgs fields of an
// operation, packed (200 B) because the batch travels as kernel parameters.
// Large operations (inl == 0) decide in k_batch, copy in one grouped grid
// (k_gcopy) and complete in k_gfin.
struct BatchOp {
  SlotDesc* post_ring;
  uint64_t* post_mirror;
  SlotDesc* scan_ring;
  uint64_t* scan_mirror;
  uint8_t* eager_ring;
  uint8_t* buf;
  uint64_t bytes;
  uint64_t key;
  uint64_t pseq;
  uint64_t* my_done;
  uint64_t my_gen;
  uint64_t* err_word;
  OpRecord* rec;          // large operations: decision record
  union {
    struct {                // staged send
      uint8_t* staging;     // host staging buffer (or null: device arena)
      uint64_t* stage_done;
      uint64_t stage_gen;
      uint8_t* arena;
      uint64_t* arena_state;
      uint64_t arena_chunk;
    } st;
    struct {                // paired self-message (a receive carrying its send)
      uint8_t* src;
      uint64_t bytes;
      uint64_t* done;
      uint64_t gen;
      uint64_t* mirror;     // the send's SR-slot free-mirror
      uint64_t pseq;
    } pr;
  };
  uint64_t* bases;        // dynamic matching
  uint32_t arena_slots;
  uint32_t E;
  int32_t peer, tag;      // dynamic matching (-1 = ANY on receives)
  uint16_t R, P, me;
  uint8_t is_recv, mode, blocking, inl, early, dyn, paired;
  int8_t sidx, didx;      // multiplex stream indices (-2 none, -1 ANY)
  // Graph-capturable communicator (G_ON): pseq and the key's match sequence
  // are relative to the device counters bases[gp] / bases[gt] (`bases`
  // points at the counter block; dynamic matching is excluded), which the
  // last CTA of the launch chain advances (G_LASTP / G_LASTT: this is the
  // batch's last operation on that counter). G_RESET: a captured blocking
  // receive zeroes its completion word before posting.
  uint8_t gflags;
  uint16_t gp, gt;
  uint8_t ll;             // P2PArgs::ll
  // graph-capturable comm: the index in this launch of the operation the
  // host expects to match this self-message (-1 none); the kernels compare
  // both absolute keys (device counters) and, if equal, the receive does
  // the paired copy and the send stands down
  int16_t mate;
};
static_assert(sizeof(BatchOp) <= 216, "BatchOp packing");

constexpr int kBatchOps = 128;    // operations per coalesced launch (27.7 KB of parameters)
constexpr int kBatchWaits = 128;  // wait entries carried by the closing launch

template <int NOPS, int NWAIT>
struct BatchArgs {
  int n, nwait;
  uint32_t* arrive;  // graph counters: CTAs of this (final) launch that have finished; null = none
  int n_static;  // ops[0, n_static): one CTA each; then dynamic ops, in order:
  int n_drecv;   // receives [n_static, n_drecv) in one CTA, sends [n_drecv, n) in another
                 // (a batch closed by a blocking receive: all of them in one CTA, in order)
  int early;  // no grouped copy follows: trigger the next (head) kernel at start
  uint64_t spin_limit_ns;
  uint64_t* err_word;
  WaitEntry w[NWAIT];
  BatchOp ops[NOPS];
};

// The grouped copy grid of a batch's large operations: tiles
// [tile_start[j], tile_start[j+1]) belong to large operation j.
struct GCopyArgs {
  int m;
  // direct: every large operation is a host-paired self-message, so its copy
  // (src, dst, bytes) is known at launch — the grid copies without waiting
  // for k_batch's decisions (k_batch triggers it at once; CTA 0 waits for
  // k_batch after its tile, so k_gfin still runs after both)
  int direct;
  uint32_t tile_start[kBatchOps + 1];
  OpRecord* rec[kBatchOps];
  const uint8_t* src[kBatchOps];
  uint8_t* dst[kBatchOps];
  uint64_t nbytes[kBatchOps];
};

enum ARDtype : int { AR_I32 = 0, AR_F32 = 1, AR_BF16 = 2, AR_F64 = 3 };
enum AROp : int { AR_SUM = 0, AR_MAX = 1, AR_MIN = 2 };
enum ARAlgo : int { AR_ONESHOT = 0, AR_TWOSHOT = 1 };
// Enqueued collectives sharing the entry/exit barrier of Allreduce_enqueue.
enum CollKind : int {
  CK_ALLREDUCE = 0,
  CK_REDUCE = 1,          // fold at the root
  CK_REDUCE_SCATTER = 2,  // block: rank r folds chunk r
  CK_BCAST = 3,
  CK_ALLGATHER = 4,
  CK_BARRIER = 5,
  CK_ALLTOALL = 6,        // block q of my sendbuf -> rank q's recvbuf at block me
};
// OpRecord.action of a collective after its entry barrier.
enum : uint64_t {
  COLL_FAILED = 0,
  COLL_ONESHOT = 1,  // allreduce (AR_ONESHOT + 1)
  COLL_TWOSHOT = 2,  // allreduce (AR_TWOSHOT + 1)
  COLL_NOOP = 3,     // nothing to move on this rank (exit barrier only)
  COLL_FOLD = 4,     // fold OpRecord.flags inputs coll[0..) into coll[16]
  COLL_COPY = 5,     // OpRecord.flags segments coll[s] -> coll[16 + s]
};

struct ARArgs {
  const uint8_t* sbuf;
  uint8_t* rbuf;
  uint64_t count;   // elements
  int esize;
  int dtype;
  int op;
  int algo;
  int P;
  int me;
  uint64_t epoch;
  CollSlot* peer_in[kMaxCollRanks];   // region[q].coll_in[me]
  uint64_t* peer_exit[kMaxCollRanks]; // region[q].coll_exit[me]
  CollSlot* my_in;                    // region[me].coll_in[0..P)
  uint64_t* my_exit;                  // region[me].coll_exit[0..P)
  OpRecord* rec;
  uint64_t opid;
  uint64_t* err_word;
  uint64_t spin_limit_ns;
  int kind;              // CollKind
  int root;              // REDUCE / BCAST
  uint64_t chunk_bytes;  // ALLGATHER: bytes per rank; REDUCE_SCATTER: bytes of my block
  // graph-capturable communicator: epoch = *gseq + 1, read after
  // griddepcontrol.wait; the kernel named by gbump advances *gseq at its end
  uint64_t* gseq;
  int gbump;             // GB_NONE / GB_ENTRY (P = 1) / GB_EXIT (exit or fused)
};
enum : int { GB_NONE = 0, GB_ENTRY = 1, GB_EXIT = 2 };

// Launchers implemented in mpix_kernels.cu (host side). Each returns the
// number of kernels launched, or -1 on a CUDA error. `sys` selects
// system-scope primitives (some peer lives on another GPU).
int launch_p2p(const P2PArgs& a, bool sys, bool inline_copy, uint64_t copy_grid, cudaStream_t s,
               cudaEvent_t copy_ev0 = nullptr, cudaEvent_t copy_ev1 = nullptr);
int launch_batch(const BatchOp* ops, int n, const WaitEntry* w, int nwait, uint64_t* err_word,
                 uint64_t spin_limit_ns, bool sys, cudaStream_t s, cudaEvent_t copy_ev0 = nullptr,
                 cudaEvent_t copy_ev1 = nullptr, uint32_t* arrive = nullptr);
int launch_allreduce(const ARArgs& a, bool sys, uint64_t reduce_grid, cudaStream_t s, bool fused);
// Reduce / Reduce_scatter / Bcast / Allgather / Barrier: entry -> work -> exit.
int launch_collective(const ARArgs& a, bool sys, uint64_t work_grid, cudaStream_t s);
uint64_t p2p_copy_grid(uint64_t bytes);
uint64_t ar_reduce_grid(uint64_t work_bytes, int P);
int preload_kernels();
// 1 in *ok when two spinning kernels of different streams of `device` run
// concurrently (mpix_kernels.cu); -1 on a CUDA error.
int coresident_probe(int device, int* ok);
// Registry of CUDA streams this library created (MPIXT_Stream_create) or saw
// destroyed through it (MPIXT_Stream_destroy): the analogue of the
// reference's live exec-queue registry (proj/src/exec_queue.cpp:82-103).
// state: 1 live (created here), 0 destroyed here, -1 unknown (foreign).
void stream_registry_note(void* stream, int live);
int stream_registry_state(void* stream);
int launch_reduce_only(const uint64_t* sb, const uint64_t* rb, int P, int me, uint64_t count,
                       int esize, int dtype, int op, int algo, OpRecord* rec, cudaStream_t s);

}  // namespace mpix
