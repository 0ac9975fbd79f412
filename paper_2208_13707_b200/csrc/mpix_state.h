// mpix_state.h — host-side state shared by the runtime translation units:
// mpix_runtime.cpp (world, info, streams, communicators, introspection),
// mpix_p2p.cpp (coalesced launches, point-to-point, waits) and
// mpix_coll.cpp (enqueued collectives). See mpix_runtime.cpp for the map to
// the reference's host layers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "mpix.h"
#include "mpix_internal.h"
#include "mpix_testing.h"

namespace mpix {

// ---------------------------------------------------------------------------
// Configuration (env knobs, SURVEY.md §5 "Config / flags")
// ---------------------------------------------------------------------------
struct Config {
  uint64_t eager_bytes = 4096;       // MPIX_EAGER_BYTES
  int ring_slots = 128;              // MPIX_RING_SLOTS
  uint64_t inline_bytes = 65536;     // MPIX_INLINE_BYTES: 1-kernel path limit
  uint64_t oneshot_max = 65536;      // MPIX_ALLREDUCE_ONESHOT_MAX (bytes)
  uint64_t spin_limit_ns = 60ull * 1000 * 1000 * 1000;  // MPIX_SPIN_TIMEOUT_MS
  bool trace = false;                // MPIX_TRACE=1: per-op device trace ring
  bool force_sys = false;            // MPIX_FORCE_SYS=1: system scope even on one GPU
  bool batch = true;                 // MPIX_BATCH=0: one launch per operation
  bool dyn_match = false;            // MPIX_MATCHING=dynamic: device matching engine, wildcards
  int stage_slots = 64;              // MPIX_STAGE_SLOTS: device staging arena slots per rank
  uint64_t stage_chunk = 4ull << 20; // MPIX_STAGE_CHUNK: bytes per arena slot
  bool graph = false;                // MPIX_GRAPH=1: every enqueue comm is graph-capturable
  bool ll = true;                    // MPIX_LL=0: no flag-in-data sends, blocking receives post
  bool conv_batch = true;            // MPIX_CONV_BATCH=0: conventional p2p launches at once
  // MPIX_HOST_EXCLUSION (the reference's lock regimes, bench.hpp:13-16,
  // fabric.hpp:17-61): 0 "global" — one process-wide lock around every p2p
  // call and one internal stream per rank for conventional operations;
  // 1 "comm" (default) — a lock per communicator, an internal stream per
  // communicator; 2 "serial" — a communicator bound to one MPIX stream is a
  // serial context: no lock on its path (MPIX_SERIAL_CHECK=1 traps
  // concurrent entry, as the reference's debug owner check does)
  int excl = 1;
  bool serial_check = false;
  uint64_t flush_ns = 100000;        // MPIX_FLUSH_US: a held batch older than this is launched by
                                     // the flusher thread (progress guarantee); 0 = no flusher

  static Config from_env() {
    Config c;
    auto geti = [](const char* n, uint64_t d) -> uint64_t {
      const char* v = std::getenv(n);
      if (!v || !*v) return d;
      return std::strtoull(v, nullptr, 10);
    };
    c.eager_bytes = geti("MPIX_EAGER_BYTES", c.eager_bytes);
    c.eager_bytes = (c.eager_bytes + 15) & ~15ull;
    c.ring_slots = (int)geti("MPIX_RING_SLOTS", c.ring_slots);
    if (c.ring_slots < 2) c.ring_slots = 2;
    if (c.ring_slots > 256) c.ring_slots = 256;  // warp_scan holds 8 slots per lane
    c.inline_bytes = geti("MPIX_INLINE_BYTES", c.inline_bytes);
    c.oneshot_max = geti("MPIX_ALLREDUCE_ONESHOT_MAX", c.oneshot_max);
    c.spin_limit_ns = geti("MPIX_SPIN_TIMEOUT_MS", 60000) * 1000000ull;
    c.trace = geti("MPIX_TRACE", 0) != 0;
    c.force_sys = geti("MPIX_FORCE_SYS", 0) != 0;
    c.batch = geti("MPIX_BATCH", 1) != 0;
    const char* m = std::getenv("MPIX_MATCHING");
    c.dyn_match = m && std::string(m) == "dynamic";
    c.stage_slots = (int)geti("MPIX_STAGE_SLOTS", c.stage_slots);
    if (c.stage_slots > 1024) c.stage_slots = 1024;
    c.stage_chunk = (geti("MPIX_STAGE_CHUNK", c.stage_chunk) + 255) & ~255ull;
    c.graph = geti("MPIX_GRAPH", 0) != 0;
    c.flush_ns = geti("MPIX_FLUSH_US", 100) * 1000ull;
    c.ll = geti("MPIX_LL", 1) != 0;
    c.conv_batch = geti("MPIX_CONV_BATCH", 1) != 0;
    if (const char* x = std::getenv("MPIX_HOST_EXCLUSION")) {
      const std::string v(x);
      c.excl = (v == "global" || v == "0") ? 0 : (v == "serial" || v == "stream" || v == "2") ? 2 : 1;
    }
    c.serial_check = geti("MPIX_SERIAL_CHECK", 0) != 0;
    return c;
  }
};

constexpr uint64_t kStageSlots = 4096;      // staging buffers per rank

extern std::atomic<uint64_t> g_launches;  // kernels launched (MPIX_Launch_count)

// Timing probe for the bench's roofline (MPIXT_Copy_timing): CUDA events
// around every copy grid (both sides of a message) while enabled, with the
// decision records of its operations: only a grid whose records say it
// copied (the second arriver's) is counted, with the bytes it moved.
struct CopyTiming {
  struct Entry {
    cudaEvent_t e0, e1;
    int device;
    std::vector<OpRecord*> recs;
  };
  std::mutex mu;
  std::atomic<bool> on{false};
  std::vector<Entry> ev;
};
extern CopyTiming g_copy_timing;

// ---------------------------------------------------------------------------
// Host rendezvous for collective calls (replaces ctrl_send/ctrl_recv over the
// collective wire context, proj/src/proc_comm.cpp:17-29).
// ---------------------------------------------------------------------------
struct CollMsg {
  int64_t i0 = 0, i1 = 0;
  uint64_t u0 = 0;
  void* p0 = nullptr;
  std::shared_ptr<void> sp;
};

class Rendezvous {
 public:
  std::vector<CollMsg> exchange(int P, int rank, uint64_t seq, CollMsg m) {
    std::unique_lock<std::mutex> lk(mu_);
    Round& r = rounds_[seq];
    if (r.vals.empty()) r.vals.resize(P);
    r.vals[rank] = std::move(m);
    if (++r.arrived == P) {
      cv_.notify_all();
    } else {
      // a member that never arrives (it failed before this collective step)
      // must not hang the others: they give up after MPIX_RENDEZVOUS_MS
      static const uint64_t limit_ms = [] {
        const char* v = std::getenv("MPIX_RENDEZVOUS_MS");
        return v && *v ? std::strtoull(v, nullptr, 10) : 120000ull;
      }();
      if (!cv_.wait_for(lk, std::chrono::milliseconds(limit_ms), [&] { return r.arrived == P; })) {
        --r.arrived;
        return {};
      }
    }
    std::vector<CollMsg> out = r.vals;
    if (++r.left == P) rounds_.erase(seq);
    return out;
  }

 private:
  struct Round {
    std::vector<CollMsg> vals;
    int arrived = 0;
    int left = 0;
  };
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<uint64_t, Round> rounds_;
};

struct RankState {
  int rank = 0;
  bool hosted = true;  // false: a stub for a rank of another process (multi-process mode)
  int device = 0;
  int sms = 148;
  int per_device = 1;  // ranks sharing this GPU
  // internal streams of freed communicators, reused by new ones (a stream
  // handle stays valid while its StreamBatch entry exists)
  std::vector<cudaStream_t> conv_pool;
  std::mutex conv_pool_mu;
  bool coresident = true;  // their spinning kernels can run concurrently (probed)
  uint64_t* d_done = nullptr;
  std::atomic<uint64_t> req_next{0};
  OpRecord* d_rec = nullptr;
  std::atomic<uint64_t> op_next{1};
  TraceRec* d_trace = nullptr;  // MPIX_TRACE ring
  std::atomic<uint64_t> trace_next{0};
  uint64_t* h_err = nullptr;  // host-mapped error word
  uint64_t* d_err = nullptr;
  cudaStream_t aux = nullptr;      // setup work
  cudaStream_t p2p = nullptr;      // conventional (host-thread) p2p of this rank
  cudaMemPool_t pool = nullptr;
  std::mutex mu;
  // Staging buffers for large blocking sends whose receive is not posted yet
  // (the eager contract, proj/src/proc_p2p.cpp:60-62). Buffer b is released
  // when the consumer of the staged copy writes h_stage[b] >= its gen; the
  // flags live in host-mapped memory so the host reclaims without syncing.
  struct StageBuf {
    uint8_t* p = nullptr;
    uint64_t size = 0;
    uint64_t gen = 0;  // last use; free when h_stage[b] >= gen
  };
  uint64_t* h_stage = nullptr;
  uint64_t* d_stage = nullptr;
  // Device staging arena: staged sends up to cfg.stage_chunk bytes claim a
  // slot inside their own kernel, only when the receive is not posted yet
  // (no host allocation on the enqueue path).
  uint8_t* d_arena = nullptr;
  uint64_t* d_arena_state = nullptr;
  std::vector<StageBuf> stage;
  std::mutex stage_mu;
  // request table: slot -> issuing stream, for STREAM_MISMATCH
  struct ReqInfo {
    uint64_t gen = 0;
    cudaStream_t stream = nullptr;
    int source = -1, tag = -1;
    bool remote = false;  // the peer lives on another GPU (system scope)
    bool conventional = false;  // MPI_Isend/Irecv or MPIX_Stream_isend/irecv (host-waited)
    bool consumed = false;      // completed by MPI_Wait/Waitall (proc_p2p.cpp:147)
    bool is_recv = false;
    int me = -1;                // the issuing comm rank (a send's status source)
    uint64_t bytes = 0;         // send: payload bytes (its status, proc_p2p.cpp:54-58)
    const void* comm = nullptr; // conventional receive: its comm (MPI_Comm_free PENDING_OPS)
  };
  std::vector<ReqInfo> reqs;
  // CUDA-Graph capture: requests created while a stream is
  // being captured get completion words of their own (zeroed, never reused:
  // a graph may be replayed at any time), as do their decision records;
  // each captured stream batch gets an arrival word.
  uint64_t* d_gdone = nullptr;
  std::atomic<uint64_t> gdone_next{0};
  std::vector<ReqInfo> greqs;
  OpRecord* d_grec = nullptr;
  std::atomic<uint64_t> grec_next{0};
  uint32_t* d_arrive = nullptr;
  std::atomic<uint32_t> arrive_next{0};
};
constexpr uint64_t kGraphRecs = 4096;         // captured large operations per rank (lifetime)
constexpr uint32_t kArriveWords = 4096;       // streams with graph-capturable batches per rank

struct CommShared {
  uint32_t ctx = 0;
  bool dyn = false;  // dynamic (wildcard-capable) matching, agreed at creation
  int P = 0;
  bool multiplex = false;
  bool is_world = false;
  RegionLayout L{};
  std::vector<uint8_t*> base;  // per-rank region
  std::vector<int> counts;     // per-rank stream count
  Rendezvous rv;
};

// Host-side op batching (DESIGN.md §3 "Coalesced launches"): inline-sized
// non-blocking operations enqueued on a CUDA stream are held here and
// launched together, as one k_batch, by the next call that orders that
// stream — a blocking operation (which joins the batch as its last member),
// a Wait/Waitall (whose wait joins it), a large operation, an allreduce,
// MPI_Comm_free, or the batch filling up. Non-blocking operations only have
// to start before the stream's next ordering point, so results are
// unchanged; the launch count drops from one per operation to one per window.
struct StreamBatch {
  std::mutex mu;
  int device = 0;
  bool sys = false;
  uint64_t* err_word = nullptr;
  std::vector<BatchOp> ops;
  // Intra-batch dependencies that force a flush before an operation joins:
  // - a large operation frees its ring slot only in k_gfin, after the whole
  //   k_batch grid: an operation needing that slot (same ring, pseq >= the
  //   large operation's pseq + R) must go to a later launch;
  std::unordered_map<const void*, uint64_t> first_large_pseq;  // ring (post mirror) -> pseq
  // - a self-message operation launched post-only relies on its
  //   counterpart running after it, not concurrently in the same grid; if
  //   the counterpart joins the same batch the host pairs the two instead.
  struct PostOnly {
    const void* comm;
    uint64_t key;
    size_t idx;  // in ops
    bool is_recv;
  };
  std::vector<PostOnly> post_only;
  // - graph-capturable comms: self-message operations whose counterpart may
  //   join this batch (matched on the device)
  std::vector<PostOnly> gmates;
  // graph-capturable comms: operations of this batch per device counter so
  // far (the next operation's relative sequence), and the arrival word of
  // the final launch, which advances the counters
  std::unordered_map<const uint64_t*, uint32_t> grel;
  uint32_t* d_arrive = nullptr;
  // steady-clock ns when the first held operation joined (0 = empty): the
  // flusher thread launches a batch nobody ordered within cfg.flush_ns
  uint64_t t_first = 0;
};

}  // namespace mpix

// Opaque handle types of mpix.h.
// Opaque handle types of mpix.h.
struct mpix_info_s {
  std::map<std::string, std::string> entries;
};

struct mpix_stream_s {
  enum Kind { serial = 0, cuda = 1 } kind = serial;
  cudaStream_t cu = nullptr;
  int device = -1;
  bool exclusive = true;
  int matching = -1;  // info "mpix_matching": 0 static, 1 dynamic, -1 default
  int graph = -1;     // info "mpix_graph": 1 graph-capturable comms, 0 not, -1 default
  std::atomic<int> refcount{0};
};

struct mpix_comm_s {
  std::shared_ptr<mpix::CommShared> sh;
  int rank = 0;
  std::vector<mpix_stream_s*> local_streams;
  bool enqueue_ok = false;
  cudaStream_t cu = nullptr;
  std::vector<uint64_t> send_pseq, recv_pseq;
  uint64_t recv_rseq = 0;  // dynamic matching: my receive ticket
  std::mutex mu;           // conventional / multiplex use may come from several threads
  std::unordered_map<uint64_t, uint32_t> idx_tagseq;  // multiplex: (dir, peer, tag, sidx, didx)
  mpix::StreamBatch* batch = nullptr;  // the StreamBatch of cu (looked up once)
  bool any_remote = false; // some member lives on another GPU
  std::unordered_map<uint64_t, uint32_t> send_tagseq, recv_tagseq;
  uint64_t coll_epoch = 0;
  uint64_t rv_seq = 0;
  // Graph-capturable: sequence numbers come from device
  // counters in my region (RegionLayout::gseq), so a captured operation is
  // correct on every replay; gtag maps (direction, peer, tag) to a counter.
  bool graph = false;
  uint64_t* d_gseq = nullptr;
  std::unordered_map<uint64_t, uint16_t> gtag;
  // Conventional receives not yet waited (completion word, generation):
  // MPI_Comm_free returns PENDING_OPS while one is incomplete
  // (proc_comm.cpp:184, c.pending counts receives until delivery).
  std::vector<std::pair<uint64_t*, uint64_t>> conv_recvs;
  // Streams other than cu this member launched on (conventional and
  // multiplex p2p): MPI_Comm_free orders the region release after them.
  std::vector<cudaStream_t> side_streams;
  // A single-stream communicator (MPIX_Stream_comm_create with a stream):
  // a serial context — lock-free under MPIX_HOST_EXCLUSION=serial.
  bool serial_ctx = false;
  // Its conventional operations' internal stream (host exclusion comm /
  // serial), created on first use; and the owner trap of the serial regime.
  cudaStream_t conv_cu = nullptr;
  mpix::StreamBatch* conv_batch = nullptr;  // its StreamBatch (looked up once)
  std::once_flag conv_once;
  std::atomic<uint64_t> owner{0};
};

namespace mpix {

struct World {
  Config cfg;
  // Multi-process mode (MPIX_World_init_mp): this process hosts rank
  // `local`; the other RankStates are stubs (device only); collective host
  // steps go through the caller's allgather; device memory peers touch lives
  // in the symmetric heap (mpix_heap.cpp), so raw pointers stay valid.
  bool mp = false;
  int local = 0;
  MPIX_Allgather_fn ag = nullptr;
  void* ag_ctx = nullptr;
  std::mutex batch_mu;
  std::unordered_map<cudaStream_t, std::unique_ptr<StreamBatch>> batches;
  int n = 0;
  std::vector<std::unique_ptr<RankState>> ranks;
  std::vector<mpix_comm_s*> world_comms;
  std::mutex ctx_mu;
  uint32_t next_ctx = 1;
  std::priority_queue<uint32_t, std::vector<uint32_t>, std::greater<>> retired;
  std::mutex comms_mu;
  std::mutex global_mu;  // MPIX_HOST_EXCLUSION=global: the one critical section
  std::vector<mpix_comm_s*> all_comms;
  // Flusher thread (progress guarantee for held batches, mpix_p2p.cpp)
  std::thread flusher;
  std::mutex fl_mu;
  std::condition_variable fl_cv;
  bool fl_stop = false;
  std::atomic<bool> fl_armed{false};

  uint32_t alloc_ctx() {  // world.cpp:43-51: retired ids recycled lowest-first
    std::lock_guard<std::mutex> lk(ctx_mu);
    if (!retired.empty()) {
      uint32_t c = retired.top();
      retired.pop();
      return c;
    }
    return next_ctx++;
  }
  void retire_ctx(uint32_t c) {
    std::lock_guard<std::mutex> lk(ctx_mu);
    retired.push(c);
  }
};

extern std::mutex g_world_mu;
extern World* g_world;
extern thread_local int t_bound_rank;

// Sticky watchdog state (MPIX_ERR_TIMEOUT / MPIX_ERR_DEVICE): a kernel of
// the rank gave up a flag wait and recorded why in the rank's host-mapped
// error word; from then on every call naming the rank reports it.
inline int rank_health(const RankState& rs) {
  if (!rs.h_err) return MPI_SUCCESS;  // a stub rank of another process
  const uint64_t v = *reinterpret_cast<volatile uint64_t*>(rs.h_err);
  if (!v) return MPI_SUCCESS;
  return v == ERRW_PROTOCOL ? MPIX_ERR_DEVICE : MPIX_ERR_TIMEOUT;
}

#define CK(call)                                 \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return MPIX_ERR_CUDA; \
  } while (0)

// mpix_runtime.cpp
int type_size(MPI_Datatype dt);
// Collective host exchange over the members of a communicator: the in-process
// rendezvous, or the allgather of multi-process mode.
std::vector<CollMsg> comm_exchange(CommShared& sh, int me, uint64_t& seq, const CollMsg& m);
// Device memory that peers read or write: the symmetric heap in
// multi-process mode, cudaMalloc otherwise.
int peer_visible_alloc(void** p, uint64_t bytes);
bool mp_mode();
bool heap_live();  // mpix_heap.cpp
// Multi-process mode: memory a peer dereferences must be in the heap.
inline bool peer_ok(const void* p, uint64_t bytes) {
  return !mp_mode() || bytes == 0 || MPIX_Heap_contains(p, bytes);
}
std::string hex_encode(const void* bytes, size_t len);
int hex_decode(const std::string& s, std::vector<uint8_t>& out);
int rank_init(RankState& r, const Config& cfg);
int rank_pool(World& w, RankState& r);
World* world();
RankState& rank_of(int r);
int create_comm(mpix_comm_s* par, const std::vector<mpix_stream_s*>& streams, bool multiplex,
                mpix_comm_s** out);

// mpix_p2p.cpp
StreamBatch& batch_of(cudaStream_t s, int device);
int flush_locked(StreamBatch& b, cudaStream_t s, const WaitEntry* w, int nwait, bool wsys,
                 uint64_t* w_err);
int flush_stream(cudaStream_t s);
void flusher_start(World& w);
void flusher_stop(World& w);
void batch_note_held(StreamBatch& b);  // caller holds b.mu, b.ops non-empty

// mpix_coll.cpp
int coll_enqueue(int kind, const void* sbuf, void* rbuf, int count, MPI_Datatype dt, MPI_Op op,
                 int root, mpix_comm_s* c);

}  // namespace mpix
