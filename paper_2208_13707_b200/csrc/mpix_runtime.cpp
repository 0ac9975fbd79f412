// mpix_runtime.cpp — host runtime behind include/mpix.h.
//
// Replaces the reference's L1-L3 host layers: World/Proc
// (proj/src/world.cpp), stream lifecycle (proj/src/proc_stream.cpp),
// communicator rendezvous (proj/src/proc_comm.cpp), the enqueue engine
// (proj/src/proc_enqueue.cpp) and the simulated GPU queue
// (proj/src/exec_queue.cpp). The queue worker thread is gone: every enqueue
// call validates, assigns matching sequence numbers, and launches one
// sm_100a kernel (mpix_kernels.cu) into the user's cudaStream_t.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
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
    return c;
  }
};

constexpr uint64_t kReqSlots = 1ull << 20;  // completion words per rank
constexpr uint64_t kStageSlots = 4096;      // staging buffers per rank

std::atomic<uint64_t> g_launches{0};

// Timing probe for the bench's roofline (MPIXT_Copy_timing): CUDA events
// around every receive-side copy grid while enabled.
struct CopyTiming {
  std::mutex mu;
  std::atomic<bool> on{false};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
} g_copy_timing;

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
    if (++r.arrived == P)
      cv_.notify_all();
    else
      cv_.wait(lk, [&] { return r.arrived == P; });
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
  int device = 0;
  int sms = 148;
  int per_device = 1;  // ranks sharing this GPU
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
  };
  std::vector<ReqInfo> reqs;
};

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

}  // namespace mpix

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
  void* batch = nullptr;   // the StreamBatch of cu (looked up once)
  bool any_remote = false; // some member lives on another GPU
  std::unordered_map<uint64_t, uint32_t> send_tagseq, recv_tagseq;
  uint64_t coll_epoch = 0;
  uint64_t rv_seq = 0;
};

namespace mpix {

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
};

struct World {
  Config cfg;
  std::mutex batch_mu;
  std::unordered_map<cudaStream_t, std::unique_ptr<StreamBatch>> batches;
  int n = 0;
  std::vector<std::unique_ptr<RankState>> ranks;
  std::vector<mpix_comm_s*> world_comms;
  std::mutex ctx_mu;
  uint32_t next_ctx = 1;
  std::priority_queue<uint32_t, std::vector<uint32_t>, std::greater<>> retired;
  std::mutex comms_mu;
  std::vector<mpix_comm_s*> all_comms;

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

std::mutex g_world_mu;
World* g_world = nullptr;
thread_local int t_bound_rank = -1;

#define CK(call)                                 \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return MPIX_ERR_CUDA; \
  } while (0)

int type_size(MPI_Datatype dt) {
  switch (dt) {
    case MPI_BYTE: return 1;
    case MPI_INT: return 4;
    case MPI_DOUBLE: return 8;
    case MPI_FLOAT: return 4;
    case MPIX_BFLOAT16: return 2;
    default: return 0;
  }
}

// ---------------------------------------------------------------------------
// Hex codec (info.cpp:37-59 semantics: lowercase, high nibble first).
// ---------------------------------------------------------------------------
std::string hex_encode(const void* bytes, size_t len) {
  static const char d[] = "0123456789abcdef";
  const uint8_t* p = static_cast<const uint8_t*>(bytes);
  std::string s;
  s.reserve(len * 2);
  for (size_t i = 0; i < len; ++i) {
    s.push_back(d[p[i] >> 4]);
    s.push_back(d[p[i] & 15]);
  }
  return s;
}

int nibble(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  return -1;
}

int hex_decode(const std::string& s, std::vector<uint8_t>& out) {
  if (s.size() % 2) return MPIX_ERR_BAD_ENCODING;
  out.clear();
  out.reserve(s.size() / 2);
  for (size_t i = 0; i < s.size(); i += 2) {
    int hi = nibble(s[i]), lo = nibble(s[i + 1]);
    if (hi < 0 || lo < 0) return MPIX_ERR_BAD_ENCODING;
    out.push_back((uint8_t)((hi << 4) | lo));
  }
  return MPI_SUCCESS;
}

// ---------------------------------------------------------------------------
// Rank setup
// ---------------------------------------------------------------------------
int rank_init(RankState& r, const Config& cfg) {
  CK(cudaSetDevice(r.device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, r.device));
  r.sms = prop.multiProcessorCount;
  CK(cudaMalloc(&r.d_done, kReqSlots * sizeof(uint64_t)));
  CK(cudaMemset(r.d_done, 0, kReqSlots * sizeof(uint64_t)));
  CK(cudaMalloc(&r.d_rec, kOpRecords * sizeof(OpRecord)));
  CK(cudaMemset(r.d_rec, 0, kOpRecords * sizeof(OpRecord)));
  if (cfg.trace) {
    CK(cudaMalloc(&r.d_trace, kTraceRecs * sizeof(TraceRec)));
    CK(cudaMemset(r.d_trace, 0, kTraceRecs * sizeof(TraceRec)));
  }
  CK(cudaHostAlloc(&r.h_err, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(r.h_err, 0, 64);
  CK(cudaHostGetDevicePointer(&r.d_err, r.h_err, 0));
  CK(cudaStreamCreateWithFlags(&r.aux, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&r.p2p, cudaStreamNonBlocking));
  CK(cudaHostAlloc(&r.h_stage, kStageSlots * sizeof(uint64_t), cudaHostAllocMapped | cudaHostAllocPortable));
  memset(r.h_stage, 0, kStageSlots * sizeof(uint64_t));
  CK(cudaHostGetDevicePointer(&r.d_stage, r.h_stage, 0));
  r.reqs.resize(kReqSlots);
  if (preload_kernels() != 0) return MPIX_ERR_CUDA;
  MPIXT_Preload();
  CK(cudaDeviceSynchronize());
  return MPI_SUCCESS;
}

int rank_pool(World& w, RankState& r) {
  CK(cudaSetDevice(r.device));
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = r.device;
  CK(cudaMemPoolCreate(&r.pool, &props));
  uint64_t thr = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(r.pool, cudaMemPoolAttrReleaseThreshold, &thr));
  // Peers read staging buffers and regions over NVLink.
  std::vector<int> seen;
  for (auto& o : w.ranks) {
    if (o->device == r.device) continue;
    if (std::find(seen.begin(), seen.end(), o->device) != seen.end()) continue;
    seen.push_back(o->device);
    cudaMemAccessDesc ad = {};
    ad.location.type = cudaMemLocationTypeDevice;
    ad.location.id = o->device;
    ad.flags = cudaMemAccessFlagsProtReadWrite;
    CK(cudaMemPoolSetAccess(r.pool, &ad, 1));
  }
  if (w.cfg.stage_slots > 0 && w.cfg.stage_chunk > 0) {
    CK(cudaMallocFromPoolAsync((void**)&r.d_arena, (uint64_t)w.cfg.stage_slots * w.cfg.stage_chunk,
                               r.pool, r.aux));
    CK(cudaMallocFromPoolAsync((void**)&r.d_arena_state, (uint64_t)w.cfg.stage_slots * 8, r.pool,
                               r.aux));
    CK(cudaMemsetAsync(r.d_arena_state, 0, (uint64_t)w.cfg.stage_slots * 8, r.aux));
    CK(cudaStreamSynchronize(r.aux));
  }
  return MPI_SUCCESS;
}

World* world() { return g_world; }

StreamBatch& batch_of(cudaStream_t s, int device) {
  World& w = *g_world;
  std::lock_guard<std::mutex> lk(w.batch_mu);
  auto& b = w.batches[s];
  if (!b) {
    b.reset(new StreamBatch());
    b->device = device;
  }
  return *b;
}

// Launch the held operations of `b` plus `nwait` wait entries (caller holds
// b.mu and has selected b's device). Returns the number of launches or -1.
int flush_locked(StreamBatch& b, cudaStream_t s, const WaitEntry* w, int nwait, bool wsys,
                 uint64_t* w_err) {
  const Config& cfg = g_world->cfg;
  int launches = 0;
  int n = (int)b.ops.size();
  int wi = 0;
  uint64_t* err = b.err_word ? b.err_word : w_err;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_copy_timing.on.load()) {
    bool large_recv = false;
    for (auto& o : b.ops) large_recv |= !o.inl && o.is_recv;
    if (large_recv) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      std::lock_guard<std::mutex> tl(g_copy_timing.mu);
      g_copy_timing.ev.emplace_back(e0, e1);
    }
  }
  do {
    int m = std::min(nwait - wi, kBatchWaits);
    int rc = launch_batch(b.ops.data(), n, w + wi, m, err, cfg.spin_limit_ns, b.sys || wsys, s,
                          e0, e1);
    e0 = e1 = nullptr;
    if (rc < 0) return -1;
    launches += rc;
    n = 0;
    b.ops.clear();
    b.first_large_pseq.clear();
    b.post_only.clear();
    wi += m;
  } while (wi < nwait);
  b.sys = false;
  b.err_word = nullptr;
  g_launches.fetch_add(launches);
  return launches;
}

int flush_stream(cudaStream_t s) {
  World& w = *g_world;
  StreamBatch* b = nullptr;
  {
    std::lock_guard<std::mutex> lk(w.batch_mu);
    auto it = w.batches.find(s);
    if (it == w.batches.end()) return 0;
    b = it->second.get();
  }
  std::lock_guard<std::mutex> lk(b->mu);
  if (b->ops.empty()) return 0;
  if (cudaSetDevice(b->device) != cudaSuccess) return -1;
  return flush_locked(*b, s, nullptr, 0, false, nullptr);
}

BatchOp pack_op(const P2PArgs& a, bool inl) {
  BatchOp o = {};
  o.post_ring = a.post_ring;
  o.post_mirror = a.post_mirror;
  o.scan_ring = a.scan_ring;
  o.scan_mirror = a.scan_mirror;
  o.eager_ring = a.eager_ring;
  o.buf = a.buf;
  o.bytes = a.bytes;
  o.key = a.key;
  o.pseq = a.pseq;
  o.my_done = a.my_done;
  o.my_gen = a.my_gen;
  o.err_word = a.err_word;
  o.rec = a.rec;
  o.st.staging = a.staging;
  o.st.stage_done = a.stage_done;
  o.st.stage_gen = a.stage_gen;
  o.st.arena = a.arena;
  o.st.arena_state = a.arena_state;
  o.st.arena_chunk = a.arena_chunk;
  o.arena_slots = a.arena_slots;
  o.E = (uint32_t)a.E;
  o.R = (uint16_t)a.R;
  o.bases = a.bases;
  o.peer = a.peer;
  o.tag = a.tag;
  o.P = (uint16_t)a.P;
  o.me = (uint16_t)a.me;
  o.dyn = (uint8_t)a.dyn;
  o.is_recv = (uint8_t)a.is_recv;
  o.mode = (uint8_t)a.mode;
  o.blocking = (uint8_t)a.blocking;
  o.inl = inl ? 1 : 0;
  return o;
}

RankState& rank_of(int r) { return *g_world->ranks[r]; }

// Build and publish the per-rank view of a communicator. Collective over the
// parent's members (proc_comm.cpp:60-176): root allocates the context id,
// everyone allocates its region, then region bases are exchanged.
int create_comm(mpix_comm_s* par, const std::vector<mpix_stream_s*>& streams, bool multiplex,
                mpix_comm_s** out) {
  World& w = *g_world;
  const int me = par->rank;
  const int P = par->sh->P;
  RankState& rs = rank_of(me);

  // Validate locally before the rendezvous (proc_comm.cpp:64-77).
  for (auto* s : streams) {
    if (s && s->kind == mpix_stream_s::cuda && s->device != rs.device)
      return MPIX_ERR_INVALID_STREAM;
  }

  // Phase 1: context id from the root + stream counts.
  CollMsg m1;
  m1.i0 = (int64_t)streams.size();
  // matching mode: the env default, or a member's "mpix_matching" stream hint
  // (dynamic wins, so every member agrees)
  int want = w.cfg.dyn_match ? 1 : 0;
  for (auto* s : streams)
    if (s && s->matching >= 0) want = s->matching;
  m1.i1 = want;
  if (me == 0) m1.u0 = w.alloc_ctx();
  auto v1 = par->sh->rv.exchange(P, me, par->rv_seq++, m1);
  uint32_t ctx = (uint32_t)v1[0].u0;
  bool dyn = false;
  for (int q = 0; q < P; ++q) dyn |= v1[q].i1 != 0;

  // Shared state is created by the root and handed out in phase 2.
  std::shared_ptr<CommShared> sh;
  if (me == 0) {
    sh = std::make_shared<CommShared>();
    sh->ctx = ctx;
    sh->dyn = dyn;
    sh->P = P;
    sh->multiplex = multiplex;
    sh->L = RegionLayout{P, w.cfg.ring_slots, w.cfg.eager_bytes};
    sh->base.assign(P, nullptr);
    sh->counts.resize(P);
    for (int q = 0; q < P; ++q) sh->counts[q] = (int)v1[q].i0;
  }

  // My region on my GPU, zeroed (all rings FREE, all epochs 0).
  RegionLayout L{P, w.cfg.ring_slots, w.cfg.eager_bytes};
  uint8_t* region = nullptr;
  {
    CK(cudaSetDevice(rs.device));
    CK(cudaMallocFromPoolAsync((void**)&region, L.total(), rs.pool, rs.aux));
    CK(cudaMemsetAsync(region, 0, L.total(), rs.aux));
    CK(cudaStreamSynchronize(rs.aux));
  }

  CollMsg m2;
  m2.p0 = region;
  if (me == 0) m2.sp = sh;
  auto v2 = par->sh->rv.exchange(P, me, par->rv_seq++, m2);
  sh = std::static_pointer_cast<CommShared>(v2[0].sp);
  {
    // every member writes the same values; guard with the rank mutex of root
    std::lock_guard<std::mutex> lk(rank_of(0).mu);
    for (int q = 0; q < P; ++q) sh->base[q] = static_cast<uint8_t*>(v2[q].p0);
  }
  // The member bases also go into my region (dynamic matching resolves
  // wildcard sources on the device).
  {
    std::vector<uint64_t> bases(P);
    for (int q = 0; q < P; ++q) bases[q] = (uint64_t)v2[q].p0;
    CK(cudaSetDevice(rs.device));
    CK(cudaMemcpyAsync(region + L.bases(), bases.data(), 8ull * P, cudaMemcpyHostToDevice, rs.aux));
    CK(cudaStreamSynchronize(rs.aux));
  }
  // Phase 3: nobody uses the comm until every member has filled the table.
  par->sh->rv.exchange(P, me, par->rv_seq++, CollMsg{});

  auto* c = new mpix_comm_s();
  c->sh = sh;
  c->rank = me;
  c->local_streams = streams;
  for (auto* s : streams)
    if (s) s->refcount.fetch_add(1);
  // proc_enqueue.cpp:23-28: only a single-stream comm whose local stream is
  // a GPU stream accepts enqueue operations.
  c->enqueue_ok = !multiplex && streams.size() == 1 && streams[0] &&
                  streams[0]->kind == mpix_stream_s::cuda;
  c->cu = c->enqueue_ok ? streams[0]->cu : nullptr;
  c->send_pseq.assign(P, 0);
  c->recv_pseq.assign(P, 0);
  for (int q = 0; q < P; ++q) c->any_remote |= rank_of(q).device != rs.device;
  {
    std::lock_guard<std::mutex> lk(w.comms_mu);
    w.all_comms.push_back(c);
  }
  *out = c;
  return MPI_SUCCESS;
}

uint64_t tagseq_key(int peer, int tag) { return ((uint64_t)(uint32_t)peer << 32) | (uint32_t)tag; }
uint64_t idx_key(int dir, int peer, int tag, int sidx, int didx) {
  return ((uint64_t)dir << 63) | ((uint64_t)(peer & 0x7fff) << 48) | ((uint64_t)(sidx & 0xff) << 40) |
         ((uint64_t)(didx & 0xff) << 32) | (uint32_t)tag;
}

// check_args of proc_enqueue.cpp:8-20 (enqueue precedence: rank, tag, count).
int check_args(const mpix_comm_s* c, int count, int peer, int tag, bool recv_side) {
  const int P = c->sh->P;
  if (recv_side) {
    if (peer != MPI_ANY_SOURCE && (peer < 0 || peer >= P)) return MPIX_ERR_INVALID_RANK;
    if (tag != MPI_ANY_TAG && tag < 0) return MPIX_ERR_INVALID_TAG;
  } else {
    if (peer < 0 || peer >= P) return MPIX_ERR_INVALID_RANK;
    if (tag < 0) return MPIX_ERR_INVALID_TAG;
  }
  if (count < 0) return MPIX_ERR_INVALID_COUNT;
  return MPI_SUCCESS;
}

struct Ticket {
  uint64_t handle;
  uint64_t* flag;
  uint64_t gen;
};

Ticket new_ticket(RankState& rs, cudaStream_t s, int source, int tag, bool remote,
                  bool conventional) {
  uint64_t n = rs.req_next.fetch_add(1);
  uint64_t slot = n % kReqSlots;
  uint64_t gen = n / kReqSlots + 1;
  auto& ri = rs.reqs[slot];
  ri.gen = gen;
  ri.stream = s;
  ri.source = source;
  ri.tag = tag;
  ri.remote = remote;
  ri.conventional = conventional;
  ri.consumed = false;
  Ticket t;
  t.handle = ((uint64_t)(rs.rank + 1) << 48) | (n + 1);
  t.flag = rs.d_done + slot;
  t.gen = gen;
  return t;
}

bool decode_ticket(uint64_t h, int* rank, uint64_t* n) {
  if (h == 0) return false;
  int r = (int)(h >> 48) - 1;
  if (r < 0 || !g_world || r >= g_world->n) return false;
  uint64_t v = h & ((1ull << 48) - 1);
  if (v == 0) return false;
  *rank = r;
  *n = v - 1;
  return true;
}

// A staging buffer of >= bytes for a staged blocking send (stream-ordered
// allocation on first use, cached afterwards).
int acquire_staging(RankState& rs, uint64_t bytes, cudaStream_t s, uint8_t** p, uint64_t** flag,
                    uint64_t* gen) {
  std::lock_guard<std::mutex> lk(rs.stage_mu);
  int best = -1;
  for (size_t b = 0; b < rs.stage.size(); ++b) {
    auto& sb = rs.stage[b];
    bool free = *reinterpret_cast<volatile uint64_t*>(&rs.h_stage[b]) >= sb.gen;
    if (free && sb.size >= bytes && (best < 0 || sb.size < rs.stage[best].size)) best = (int)b;
  }
  if (best < 0) {
    if (rs.stage.size() >= kStageSlots) return MPIX_ERR_NO_MEM;
    uint64_t size = 1ull << 20;
    while (size < bytes) size <<= 1;
    RankState::StageBuf sb;
    if (cudaMallocFromPoolAsync((void**)&sb.p, size, rs.pool, s) != cudaSuccess) return MPIX_ERR_NO_MEM;
    sb.size = size;
    rs.stage.push_back(sb);
    best = (int)rs.stage.size() - 1;
  }
  auto& sb = rs.stage[best];
  sb.gen += 1;
  *p = sb.p;
  *flag = rs.d_stage + best;
  *gen = sb.gen;
  return MPI_SUCCESS;
}

// Point-to-point enqueue (send side and receive side).
// How an operation reaches p2p_post: the enqueue family (the comm's stream),
// conventional host-thread p2p (the rank's internal stream), or multiplex
// stream p2p (the stream of local index sidx / didx).
struct PostHow {
  cudaStream_t stream = nullptr;
  bool conventional = false;
  int sidx = -2, didx = -2;  // IDX_NONE unless multiplex (types.hpp:14)
};

int p2p_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
             bool is_recv, bool blocking, MPI_Request* req, const PostHow& how);

int p2p_enqueue(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
                bool is_recv, bool blocking, MPI_Request* req) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (!c->enqueue_ok) return MPIX_ERR_NOT_ENQUEUE_COMM;  // proc_enqueue.cpp:33-34
  int rc = check_args(c, count, peer, tag, is_recv);
  if (rc) return rc;
  PostHow how;
  how.stream = c->cu;
  return p2p_post(c, buf, count, dt, peer, tag, is_recv, blocking, req, how);
}

// check_send_args / check_recv_args of proc_p2p.cpp:9-23 (conventional
// precedence: rank, count, tag).
int check_p2p_args(const mpix_comm_s* c, int count, int peer, int tag, bool recv_side) {
  const int P = c->sh->P;
  if (recv_side) {
    if (peer != MPI_ANY_SOURCE && (peer < 0 || peer >= P)) return MPIX_ERR_INVALID_RANK;
    if (count < 0) return MPIX_ERR_INVALID_COUNT;
    if (tag != MPI_ANY_TAG && tag < 0) return MPIX_ERR_INVALID_TAG;
  } else {
    if (peer < 0 || peer >= P) return MPIX_ERR_INVALID_RANK;
    if (count < 0) return MPIX_ERR_INVALID_COUNT;
    if (tag < 0) return MPIX_ERR_INVALID_TAG;
  }
  return MPI_SUCCESS;
}

// Conventional p2p (Proc::isend/irecv, proc_p2p.cpp:96-113) on GPU buffers:
// executed on the rank's internal stream, launched at once (no batching:
// a posted conventional send must progress without a later MPI call).
int conv_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
              bool is_recv, bool blocking, MPI_Request* req) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (c->sh->multiplex) return MPIX_ERR_MULTIPLEX_COMM;
  int rc = check_p2p_args(c, count, peer, tag, is_recv);
  if (rc) return rc;
  PostHow how;
  how.stream = rank_of(c->rank).p2p;
  how.conventional = true;
  return p2p_post(c, buf, count, dt, peer, tag, is_recv, blocking, req, how);
}

// Multiplex stream p2p (Proc::stream_isend/irecv, proc_p2p.cpp:115-144):
// runs on the CUDA stream of local stream src_idx (send) / dst_idx (recv),
// or on the rank's internal stream when that MPIX stream is not a GPU stream.
int stream_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
                int src_idx, int dst_idx, bool is_recv, bool blocking, MPI_Request* req) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (!c->sh->multiplex) return MPIX_ERR_NOT_MULTIPLEX;
  int rc = check_p2p_args(c, count, peer, tag, is_recv);
  if (rc) return rc;
  const auto& counts = c->sh->counts;
  const int me = c->rank;
  if (!is_recv) {
    if (src_idx < 0 || src_idx >= counts[me]) return MPIX_ERR_INVALID_INDEX;
    if (dst_idx < 0 || dst_idx >= counts[peer]) return MPIX_ERR_INVALID_INDEX;
  } else {
    if (dst_idx == MPIX_ANY_INDEX) return MPIX_ERR_WILDCARD_DST;
    if (dst_idx < 0 || dst_idx >= counts[me]) return MPIX_ERR_INVALID_INDEX;
    if (src_idx != MPIX_ANY_INDEX) {
      if (src_idx < 0) return MPIX_ERR_INVALID_INDEX;
      if (peer != MPI_ANY_SOURCE && src_idx >= counts[peer]) return MPIX_ERR_INVALID_INDEX;
    }
    // the index travels in the static key; a wildcard index would need the
    // dynamic engine to filter on it (not implemented)
    if (src_idx == MPIX_ANY_INDEX || c->sh->dyn) return MPIX_ERR_UNSUPPORTED;
  }
  if (!is_recv && c->sh->dyn) return MPIX_ERR_UNSUPPORTED;
  const int local = is_recv ? dst_idx : src_idx;
  mpix_stream_s* ls = c->local_streams[local];
  PostHow how;
  how.stream = ls && ls->kind == mpix_stream_s::cuda ? ls->cu : rank_of(me).p2p;
  how.conventional = true;
  how.sidx = src_idx;
  how.didx = dst_idx;
  return p2p_post(c, buf, count, dt, peer, tag, is_recv, blocking, req, how);
}

int p2p_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
             bool is_recv, bool blocking, MPI_Request* req, const PostHow& how) {
  int esz = type_size(dt);
  if (!esz) return MPIX_ERR_TYPE;
  const bool dyn = c->sh->dyn;
  // Wildcards need the device matching engine (MPIX_MATCHING=dynamic).
  if (is_recv && !dyn && (peer == MPI_ANY_SOURCE || tag == MPI_ANY_TAG)) return MPIX_ERR_UNSUPPORTED;
  if (!blocking && !req) return MPIX_ERR_INVALID_ARG;

  World& w = *g_world;
  CommShared& sh = *c->sh;
  const RegionLayout& L = sh.L;
  const int me = c->rank;
  RankState& rs = rank_of(me);
  const uint64_t bytes = (uint64_t)count * (uint64_t)esz;
  const bool indexed = how.sidx >= 0;
  std::lock_guard<std::mutex> clk(c->mu);

  P2PArgs a = {};
  a.is_recv = is_recv;
  a.blocking = blocking;
  a.R = L.R;
  a.E = L.E;
  a.buf = static_cast<uint8_t*>(buf);
  a.bytes = bytes;
  a.err_word = rs.d_err;
  a.spin_limit_ns = w.cfg.spin_limit_ns;
  uint32_t tseq;
  if (!is_recv) {
    const int d = peer;
    tseq = indexed ? c->idx_tagseq[idx_key(0, d, tag, how.sidx, how.didx)]++
                   : c->send_tagseq[tagseq_key(d, tag)]++;
    a.pseq = c->send_pseq[d]++;
    a.post_ring = reinterpret_cast<SlotDesc*>(sh.base[d] + L.sr(me));
    a.post_mirror = reinterpret_cast<uint64_t*>(sh.base[me] + L.sr_free(d));
    a.scan_ring = reinterpret_cast<SlotDesc*>(sh.base[me] + L.rr(d));
    a.scan_mirror = reinterpret_cast<uint64_t*>(sh.base[d] + L.rr_free(me));
    a.eager_ring = sh.base[d] + L.eager(me);
    a.mode = !blocking ? MODE_ISEND : (bytes <= L.E ? MODE_EAGER : MODE_STAGED);
  } else if (dyn) {
    tseq = 0;
    a.pseq = c->recv_rseq++;  // receive ticket (post order)
    a.mode = 0;
  } else {
    const int s = peer;
    tseq = indexed ? c->idx_tagseq[idx_key(1, s, tag, how.sidx, how.didx)]++
                   : c->recv_tagseq[tagseq_key(s, tag)]++;
    a.pseq = c->recv_pseq[s]++;
    a.post_ring = reinterpret_cast<SlotDesc*>(sh.base[s] + L.rr(me));
    a.post_mirror = reinterpret_cast<uint64_t*>(sh.base[me] + L.rr_free(s));
    a.scan_ring = reinterpret_cast<SlotDesc*>(sh.base[me] + L.sr(s));
    a.scan_mirror = reinterpret_cast<uint64_t*>(sh.base[s] + L.sr_free(me));
    a.mode = 0;
  }
  a.key = ((uint64_t)(uint32_t)tag << 32) | tseq;
  if (indexed)  // multiplex: the stream indices are part of the match key (endpoint.hpp:26-32)
    a.key = ((uint64_t)(uint32_t)tag << 32) | ((uint64_t)(how.sidx & 0xff) << 24) |
            ((uint64_t)(how.didx & 0xff) << 16) | (tseq & 0xffff);
  if (dyn) {
    a.dyn = 1;
    a.P = sh.P;
    a.me = me;
    a.peer = peer;  // -1 = ANY_SOURCE (receives)
    a.tag = tag;    // -1 = ANY_TAG (receives)
    a.bases = reinterpret_cast<uint64_t*>(sh.base[me] + L.bases());
  }

  const bool sys = w.cfg.force_sys ||
                   (dyn ? c->any_remote : rank_of(peer).device != rs.device);
  CK(cudaSetDevice(rs.device));
  cudaStream_t s = how.stream;
  Ticket t{};
  if (!blocking || is_recv) {
    t = new_ticket(rs, s, is_recv ? peer : me, tag, sys, how.conventional);
    a.my_done = t.flag;
    a.my_gen = t.gen;
  }
  if (a.mode == MODE_STAGED && !is_recv) {
    if (rs.d_arena && bytes <= w.cfg.stage_chunk) {
      a.arena = rs.d_arena;
      a.arena_state = rs.d_arena_state;
      a.arena_slots = (uint32_t)w.cfg.stage_slots;
      a.arena_chunk = w.cfg.stage_chunk;
    } else {
      int rc2 = acquire_staging(rs, bytes, s, &a.staging, &a.stage_done, &a.stage_gen);
      if (rc2) return rc2;
    }
  }
  if (rs.d_trace) {
    uint64_t n = rs.trace_next.fetch_add(1);
    a.trace = rs.d_trace + (n % kTraceRecs);
    TraceRec head = {};
    head.seq = n + 1;
    head.bytes = bytes;
    head.key = a.key;
    CK(cudaMemcpyAsync(a.trace, &head, 32, cudaMemcpyHostToDevice, s));
  }
  bool inl = bytes <= w.cfg.inline_bytes || (!is_recv && a.mode == MODE_EAGER);
  bool post_only = false;
  if (!inl && !blocking && peer == me && !dyn && !how.conventional) {
    // Self-message whose counterpart has not been enqueued yet: it can only
    // be enqueued later on this same stream (an enqueue comm has one stream),
    // so it runs after this operation, which therefore only posts and never
    // copies: one small launch instead of proto + copy grid + fin.
    const auto& other = is_recv ? c->send_tagseq : c->recv_tagseq;
    auto it = other.find(tagseq_key(me, tag));
    if (it == other.end() || it->second <= tseq) inl = post_only = true;
  }
  if (!inl) {
    uint64_t op = rs.op_next.fetch_add(1);
    a.rec = rs.d_rec + (op % kOpRecords);
    a.opid = op;
  }
  if (!c->batch && !how.conventional) c->batch = &batch_of(s, rs.device);
  StreamBatch& b = how.conventional ? batch_of(s, rs.device) : *static_cast<StreamBatch*>(c->batch);
  std::lock_guard<std::mutex> lk(b.mu);
  if (w.cfg.batch && !a.trace) {
    // Join the stream's batch; a blocking operation closes it (it must have
    // completed before anything behind it in the stream runs).
    // A self-message whose counterpart is held post-only in this batch: the
    // host has matched them (same comm, same key, static matching), so the
    // two become one paired operation — no descriptors, one copy.
    int pk = -1;
    if (!dyn && peer == me && (!blocking || is_recv) && a.mode != MODE_STAGED) {
      for (size_t k = 0; k < b.post_only.size(); ++k) {
        const auto& po = b.post_only[k];
        if (po.comm == c && po.key == a.key && po.is_recv != is_recv) pk = (int)k;
      }
      // my ring slot must not wait on a large operation of this batch
      auto fl = b.first_large_pseq.find(a.post_mirror);
      if (fl != b.first_large_pseq.end() && a.pseq >= fl->second + (uint64_t)a.R) pk = -1;
    }
    if (pk >= 0) {
      const size_t j = b.post_only[pk].idx;
      b.post_only.erase(b.post_only.begin() + pk);
      const BatchOp held = b.ops[j];
      BatchOp m = is_recv ? pack_op(a, true) : held;  // the receive carries the pair
      const BatchOp snd = is_recv ? held : pack_op(a, true);
      m.paired = 1;
      m.pr.src = snd.buf;
      m.pr.bytes = snd.bytes;
      m.pr.done = snd.my_done;
      m.pr.gen = snd.my_gen;
      m.pr.mirror = snd.post_mirror;
      m.pr.pseq = snd.pseq;
      const uint64_t nb = std::min(snd.bytes, m.bytes);
      m.inl = nb <= w.cfg.inline_bytes ? 1 : 0;
      if (!m.inl) {
        if (!m.rec) m.rec = rs.d_rec + (rs.op_next.fetch_add(1) % kOpRecords);
        b.first_large_pseq.emplace(m.post_mirror, m.pseq);
        b.first_large_pseq.emplace(m.pr.mirror, m.pr.pseq);
      }
      m.blocking = blocking ? 1 : held.blocking;
      b.ops[j] = m;
      b.sys |= sys;
    } else {
      bool flush_first = (int)b.ops.size() >= kBatchOps;
      auto fl = b.first_large_pseq.find(a.post_mirror);
      flush_first |= fl != b.first_large_pseq.end() && a.pseq >= fl->second + (uint64_t)a.R;
      for (auto& po : b.post_only) flush_first |= po.comm == c && po.key == a.key;
      if (flush_first && flush_locked(b, s, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
      if (b.ops.empty()) b.err_word = rs.d_err;
      if (!inl && a.post_mirror) b.first_large_pseq.emplace(a.post_mirror, a.pseq);
      if (post_only) b.post_only.push_back({c, a.key, b.ops.size(), (bool)is_recv});
      b.ops.push_back(pack_op(a, inl));
      b.sys |= sys;
    }
    // a blocking operation closes the batch; conventional operations are
    // launched at once
    if ((blocking || how.conventional) && flush_locked(b, s, nullptr, 0, false, nullptr) < 0)
      return MPIX_ERR_CUDA;
  } else {
    if (!b.ops.empty() && flush_locked(b, s, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (!inl && is_recv && g_copy_timing.on.load()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      std::lock_guard<std::mutex> tl(g_copy_timing.mu);
      g_copy_timing.ev.emplace_back(e0, e1);
    }
    a.early_trigger = p2p_copy_grid(bytes) <= kEarlyTriggerTiles;
    int nk = launch_p2p(a, sys, inl, inl ? 1 : p2p_copy_grid(bytes), s, e0, e1);
    if (nk < 0) return MPIX_ERR_CUDA;
    g_launches.fetch_add(nk);
  }
  if (req) *req = (!blocking) ? t.handle : MPI_REQUEST_NULL;
  return MPI_SUCCESS;
}

int waitall_enqueue(int n, MPI_Request* reqs, MPI_Status* statuses) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (n < 0) return MPIX_ERR_INVALID_ARG;
  if (n == 0) return MPI_SUCCESS;  // proc_enqueue.cpp:121
  if (!reqs) return MPIX_ERR_INVALID_REQUEST;
  struct Item {
    int rank;
    uint64_t n;
  };
  std::vector<Item> items(n);
  for (int i = 0; i < n; ++i) {  // proc_enqueue.cpp:122-123
    if (!decode_ticket(reqs[i], &items[i].rank, &items[i].n)) return MPIX_ERR_INVALID_REQUEST;
  }
  cudaStream_t s0 = nullptr;
  int dev0 = -1;
  bool sys = false;
  for (int i = 0; i < n; ++i) {  // proc_enqueue.cpp:124-126
    RankState& rs = rank_of(items[i].rank);
    auto& ri = rs.reqs[items[i].n % kReqSlots];
    cudaStream_t s = ri.gen == items[i].n / kReqSlots + 1 ? ri.stream : nullptr;
    // a conventional request has no queue (proc_enqueue.cpp:124-126, Appendix A6)
    if (ri.conventional) return MPIX_ERR_STREAM_MISMATCH;
    if (i == 0) {
      s0 = s;
      dev0 = rs.device;
    }
    if (s != s0 || rs.device != dev0) return MPIX_ERR_STREAM_MISMATCH;
    sys |= ri.remote;
  }
  if (statuses) {
    for (int i = 0; i < n; ++i) {
      RankState& rs = rank_of(items[i].rank);
      auto& ri = rs.reqs[items[i].n % kReqSlots];
      statuses[i].MPI_SOURCE = ri.source;
      statuses[i].MPI_TAG = ri.tag;
      statuses[i].MPI_ERROR = MPI_SUCCESS;
      statuses[i].source_index = -2;
      statuses[i].count_bytes = UINT64_MAX;
      statuses[i].truncated = 0;
    }
  }
  CK(cudaSetDevice(dev0));
  std::vector<WaitEntry> we(n);
  for (int k = 0; k < n; ++k) {
    RankState& rs = rank_of(items[k].rank);
    uint64_t nn = items[k].n;
    we[k].flag = rs.d_done + (nn % kReqSlots);
    we[k].gen = nn / kReqSlots + 1;
  }
  // The wait closes the stream's batch: one launch for the window.
  StreamBatch& b = batch_of(s0, dev0);
  std::lock_guard<std::mutex> lk(b.mu);
  if (flush_locked(b, s0, we.data(), n, sys, rank_of(items[0].rank).d_err) < 0) return MPIX_ERR_CUDA;
  return MPI_SUCCESS;
}

int reduce_dtype(MPI_Datatype dt) {
  switch (dt) {
    case MPI_INT: return AR_I32;
    case MPI_FLOAT: return AR_F32;
    case MPIX_BFLOAT16: return AR_BF16;
    case MPI_DOUBLE: return AR_F64;
    default: return -1;
  }
}

int reduce_op(MPI_Op op) {
  switch (op) {
    case MPI_SUM: return AR_SUM;
    case MPI_MAX: return AR_MAX;
    case MPI_MIN: return AR_MIN;
    default: return -1;
  }
}

// Every enqueued collective: validate, fill the entry-barrier arguments,
// order the stream's held operations first, launch.
// MPI_Wait / MPI_Waitall on the host (Proc::wait/waitall, proc_p2p.cpp:
// 146-181): a request may be waited once (consumed); the wait is a device
// wait launched on the request's stream, then the host synchronises it.
int host_waitall(int n, MPI_Request* reqs, MPI_Status* statuses) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (n < 0) return MPIX_ERR_INVALID_ARG;
  if (n == 0) return MPI_SUCCESS;
  if (!reqs) return MPIX_ERR_INVALID_REQUEST;
  struct Item {
    int rank;
    uint64_t n;
  };
  std::vector<Item> items(n);
  for (int i = 0; i < n; ++i) {
    if (!decode_ticket(reqs[i], &items[i].rank, &items[i].n)) return MPIX_ERR_INVALID_REQUEST;
    auto& ri = rank_of(items[i].rank).reqs[items[i].n % kReqSlots];
    if (ri.gen != items[i].n / kReqSlots + 1 || ri.consumed) return MPIX_ERR_INVALID_REQUEST;
  }
  // group by stream: one device wait (and one synchronisation) per stream
  std::map<cudaStream_t, std::vector<int>> by;
  for (int i = 0; i < n; ++i) by[rank_of(items[i].rank).reqs[items[i].n % kReqSlots].stream].push_back(i);
  for (auto& kv : by) {
    cudaStream_t s = kv.first;
    const int r0 = items[kv.second[0]].rank;
    RankState& rs0 = rank_of(r0);
    std::vector<WaitEntry> we;
    bool sys = false;
    for (int i : kv.second) {
      RankState& rs = rank_of(items[i].rank);
      uint64_t nn = items[i].n;
      we.push_back({rs.d_done + (nn % kReqSlots), nn / kReqSlots + 1});
      sys |= rs.reqs[nn % kReqSlots].remote;
    }
    CK(cudaSetDevice(rs0.device));
    StreamBatch& b = batch_of(s, rs0.device);
    {
      std::lock_guard<std::mutex> lk(b.mu);
      if (flush_locked(b, s, we.data(), (int)we.size(), sys, rs0.d_err) < 0) return MPIX_ERR_CUDA;
    }
    CK(cudaStreamSynchronize(s));
  }
  for (int i = 0; i < n; ++i) {
    auto& ri = rank_of(items[i].rank).reqs[items[i].n % kReqSlots];
    ri.consumed = true;
    if (statuses) {
      statuses[i].MPI_SOURCE = ri.source;
      statuses[i].MPI_TAG = ri.tag;
      statuses[i].MPI_ERROR = MPI_SUCCESS;
      statuses[i].source_index = -2;
      statuses[i].count_bytes = UINT64_MAX;
      statuses[i].truncated = 0;
    }
    reqs[i] = MPI_REQUEST_NULL;
  }
  return MPI_SUCCESS;
}

// Blocking conventional / multiplex operation: post as a blocking device
// operation (eager or staged send, waiting receive), then synchronise.
int host_blocking(int rc, mpix_comm_s* c, cudaStream_t s, MPI_Status* status, int source, int tag) {
  if (rc) return rc;
  CK(cudaSetDevice(rank_of(c->rank).device));
  CK(cudaStreamSynchronize(s));
  if (status) {
    status->MPI_SOURCE = source;
    status->MPI_TAG = tag;
    status->MPI_ERROR = MPI_SUCCESS;
    status->source_index = -2;
    status->count_bytes = UINT64_MAX;
    status->truncated = 0;
  }
  return MPI_SUCCESS;
}

int coll_enqueue(int kind, const void* sbuf, void* rbuf, int count, MPI_Datatype dt, MPI_Op op,
                 int root, mpix_comm_s* c) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (!c->enqueue_ok) return MPIX_ERR_NOT_ENQUEUE_COMM;
  if (count < 0) return MPIX_ERR_INVALID_COUNT;
  CommShared& sh = *c->sh;
  const int P = sh.P;
  if (P > kMaxCollRanks) return MPIX_ERR_UNSUPPORTED;
  const bool folds = kind == CK_ALLREDUCE || kind == CK_REDUCE || kind == CK_REDUCE_SCATTER;
  int dtype = 0, aop = 0;
  if (kind != CK_BARRIER) {
    if (folds) {
      dtype = reduce_dtype(dt);
      if (dtype < 0) return MPIX_ERR_TYPE;
      aop = reduce_op(op);
      if (aop < 0) return MPIX_ERR_OP;
    } else if (!type_size(dt)) {
      return MPIX_ERR_TYPE;
    }
  }
  if ((kind == CK_REDUCE || kind == CK_BCAST) && (root < 0 || root >= P)) return MPIX_ERR_INVALID_RANK;
  const int me = c->rank;
  const int esz = kind == CK_BARRIER ? 1 : type_size(dt);
  const uint64_t bytes = (uint64_t)count * esz;
  switch (kind) {
    case CK_ALLREDUCE:
      if (!rbuf) return MPIX_ERR_INVALID_ARG;
      if (sbuf == MPI_IN_PLACE) sbuf = rbuf;
      break;
    case CK_REDUCE:
      if (me == root && !rbuf) return MPIX_ERR_INVALID_ARG;
      if (sbuf == MPI_IN_PLACE) {
        if (me != root) return MPIX_ERR_INVALID_ARG;
        sbuf = rbuf;
      }
      break;
    case CK_REDUCE_SCATTER:
      // in place would fold chunk me of my buffer while writing its start
      if (sbuf == MPI_IN_PLACE) return MPIX_ERR_UNSUPPORTED;
      if (!rbuf) return MPIX_ERR_INVALID_ARG;
      break;
    case CK_BCAST:
      sbuf = rbuf;  // one buffer: the root's is the source
      break;
    case CK_ALLGATHER:
      if (!rbuf) return MPIX_ERR_INVALID_ARG;
      if (sbuf == MPI_IN_PLACE) sbuf = static_cast<uint8_t*>(rbuf) + (uint64_t)me * bytes;
      break;
    default:
      break;
  }
  RankState& rs = rank_of(me);

  ARArgs a = {};
  a.kind = kind;
  a.root = root;
  a.sbuf = static_cast<const uint8_t*>(sbuf);
  a.rbuf = static_cast<uint8_t*>(rbuf);
  a.count = (uint64_t)count;
  a.esize = esz;
  a.dtype = dtype;
  a.op = aop;
  a.P = P;
  a.me = me;
  a.epoch = ++c->coll_epoch;
  a.algo = (bytes <= g_world->cfg.oneshot_max || P <= 2) ? AR_ONESHOT : AR_TWOSHOT;
  a.chunk_bytes = bytes;  // ALLGATHER: per rank; REDUCE_SCATTER: my block; BCAST: the buffer
  const RegionLayout& L = sh.L;
  for (int q = 0; q < P; ++q) {
    a.peer_in[q] = reinterpret_cast<CollSlot*>(sh.base[q] + L.coll_in(me));
    a.peer_exit[q] = reinterpret_cast<uint64_t*>(sh.base[q] + L.coll_exit(me));
  }
  a.my_in = reinterpret_cast<CollSlot*>(sh.base[me] + L.coll_in(0));
  a.my_exit = reinterpret_cast<uint64_t*>(sh.base[me] + L.coll_exit(0));
  a.err_word = rs.d_err;
  a.spin_limit_ns = g_world->cfg.spin_limit_ns;
  {
    uint64_t opid = rs.op_next.fetch_add(1);
    a.rec = rs.d_rec + (opid % kOpRecords);
    a.opid = opid;
  }
  bool sys = g_world->cfg.force_sys;
  for (int q = 0; q < P; ++q) sys |= rank_of(q).device != rs.device;
  CK(cudaSetDevice(rs.device));
  if (!c->batch) c->batch = &batch_of(c->cu, rs.device);
  StreamBatch& b = *static_cast<StreamBatch*>(c->batch);
  std::lock_guard<std::mutex> lk(b.mu);
  if (!b.ops.empty() && flush_locked(b, c->cu, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
  int nk;
  if (kind == CK_ALLREDUCE) {
    uint64_t work = a.algo == AR_TWOSHOT ? (bytes + P - 1) / P : bytes;
    // latency-bound sizes: entry + reduce + exit in one single-CTA launch
    const bool fused = bytes <= g_world->cfg.oneshot_max;
    nk = launch_allreduce(a, sys, ar_reduce_grid(work, P), c->cu, fused);
  } else {
    uint64_t grid = 1;  // ranks with nothing to move exit at once
    if ((kind == CK_REDUCE && me == root) || kind == CK_REDUCE_SCATTER)
      grid = ar_reduce_grid(bytes, P);
    else if (kind == CK_BCAST && me != root)
      grid = p2p_copy_grid(bytes);
    else if (kind == CK_ALLGATHER)
      grid = (uint64_t)P * p2p_copy_grid(bytes);
    nk = launch_collective(a, sys, grid, c->cu);
  }
  if (nk < 0) return MPIX_ERR_CUDA;
  g_launches.fetch_add(nk);
  return MPI_SUCCESS;
}

}  // namespace mpix

using namespace mpix;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* MPIX_Error_string(int code) {
  switch (code) {  // result.cpp:5-32
    case MPI_SUCCESS: return "OK";
    case MPIX_ERR_POOL_EXHAUSTED: return "POOL_EXHAUSTED";
    case MPIX_ERR_NO_EXPLICIT_POOL: return "NO_EXPLICIT_POOL";
    case MPIX_ERR_PENDING_OPS: return "PENDING_OPS";
    case MPIX_ERR_IN_USE: return "IN_USE";
    case MPIX_ERR_BAD_HINT: return "BAD_HINT";
    case MPIX_ERR_INVALID_STREAM: return "INVALID_STREAM";
    case MPIX_ERR_INVALID_COMM: return "INVALID_COMM";
    case MPIX_ERR_INVALID_RANK: return "INVALID_RANK";
    case MPIX_ERR_INVALID_COUNT: return "INVALID_COUNT";
    case MPIX_ERR_INVALID_TAG: return "INVALID_TAG";
    case MPIX_ERR_INVALID_REQUEST: return "INVALID_REQUEST";
    case MPIX_ERR_INVALID_INDEX: return "INVALID_INDEX";
    case MPIX_ERR_MULTIPLEX_COMM: return "MULTIPLEX_COMM";
    case MPIX_ERR_NOT_MULTIPLEX: return "NOT_MULTIPLEX";
    case MPIX_ERR_WILDCARD_DST: return "WILDCARD_DST";
    case MPIX_ERR_EMPTY_LIST: return "EMPTY_LIST";
    case MPIX_ERR_NOT_ENQUEUE_COMM: return "NOT_ENQUEUE_COMM";
    case MPIX_ERR_STREAM_MISMATCH: return "STREAM_MISMATCH";
    case MPIX_ERR_QUEUE_BUSY: return "QUEUE_BUSY";
    case MPIX_ERR_CONFIG_INVALID: return "CONFIG_INVALID";
    case MPIX_ERR_NOT_FOUND: return "NOT_FOUND";
    case MPIX_ERR_BAD_ENCODING: return "BAD_ENCODING";
    case MPIX_ERR_CUDA: return "CUDA_ERROR";
    case MPIX_ERR_NOT_INITIALIZED: return "NOT_INITIALIZED";
    case MPIX_ERR_UNSUPPORTED: return "UNSUPPORTED";
    case MPIX_ERR_INVALID_ARG: return "INVALID_ARG";
    case MPIX_ERR_TYPE: return "INVALID_TYPE";
    case MPIX_ERR_OP: return "INVALID_OP";
    case MPIX_ERR_NO_MEM: return "NO_MEM";
    default: return "UNKNOWN";
  }
}

// --------------------------------------------------------------------------
// World
// --------------------------------------------------------------------------
int MPIX_World_init(int nranks, const int* devices) {
  std::lock_guard<std::mutex> lk(g_world_mu);
  if (g_world) return MPIX_ERR_IN_USE;
  if (nranks < 1) return MPIX_ERR_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return MPIX_ERR_CUDA;
  std::unique_ptr<World> w(new World());
  w->cfg = Config::from_env();
  w->n = nranks;
  for (int r = 0; r < nranks; ++r) {
    auto rs = std::make_unique<RankState>();
    rs->rank = r;
    rs->device = devices ? devices[r] : r % ndev;
    if (rs->device < 0 || rs->device >= ndev) return MPIX_ERR_INVALID_ARG;
    w->ranks.push_back(std::move(rs));
  }
  for (auto& rs : w->ranks) {
    int per = 0;
    for (auto& o : w->ranks) per += o->device == rs->device;
    rs->per_device = per;
  }
  // Peer access between every pair of distinct devices (NVLink / NVSwitch).
  std::vector<int> devs;
  for (auto& rs : w->ranks)
    if (std::find(devs.begin(), devs.end(), rs->device) == devs.end()) devs.push_back(rs->device);
  for (int i : devs) {
    for (int j : devs) {
      if (i == j) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, i, j);
      if (!can) return MPIX_ERR_UNSUPPORTED;
      cudaSetDevice(i);
      cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        return MPIX_ERR_CUDA;
    }
  }
  for (auto& rs : w->ranks) {
    int rc = rank_init(*rs, w->cfg);
    if (rc) return rc;
  }
  for (auto& rs : w->ranks) {
    int rc = rank_pool(*w, *rs);
    if (rc) return rc;
  }
  // Bootstrap world communicator, ctx 0 (world.cpp:61-76). It carries no
  // stream, so enqueue on it is NOT_ENQUEUE_COMM; it has no region.
  auto sh = std::make_shared<CommShared>();
  sh->ctx = 0;
  sh->P = nranks;
  sh->is_world = true;
  sh->counts.assign(nranks, 1);
  sh->L = RegionLayout{nranks, w->cfg.ring_slots, w->cfg.eager_bytes};
  sh->base.assign(nranks, nullptr);
  sh->dyn = w->cfg.dyn_match;
  // The world comm carries conventional p2p (and the mixed mode of
  // Appendix A7): every rank gets a region for it too.
  for (int r = 0; r < nranks; ++r) {
    RankState& rs = *w->ranks[r];
    if (cudaSetDevice(rs.device) != cudaSuccess) return MPIX_ERR_CUDA;
    uint8_t* region = nullptr;
    if (cudaMallocFromPoolAsync((void**)&region, sh->L.total(), rs.pool, rs.aux) != cudaSuccess ||
        cudaMemsetAsync(region, 0, sh->L.total(), rs.aux) != cudaSuccess)
      return MPIX_ERR_CUDA;
    sh->base[r] = region;
  }
  {
    std::vector<uint64_t> bases(nranks);
    for (int r = 0; r < nranks; ++r) bases[r] = (uint64_t)sh->base[r];
    for (int r = 0; r < nranks; ++r) {
      RankState& rs = *w->ranks[r];
      cudaSetDevice(rs.device);
      if (cudaMemcpyAsync(sh->base[r] + sh->L.bases(), bases.data(), 8ull * nranks,
                          cudaMemcpyHostToDevice, rs.aux) != cudaSuccess ||
          cudaStreamSynchronize(rs.aux) != cudaSuccess)
        return MPIX_ERR_CUDA;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    auto* c = new mpix_comm_s();
    c->sh = sh;
    c->rank = r;
    c->send_pseq.assign(nranks, 0);
    c->recv_pseq.assign(nranks, 0);
    for (int q = 0; q < nranks; ++q) c->any_remote |= w->ranks[q]->device != w->ranks[r]->device;
    w->world_comms.push_back(c);
  }
  g_world = w.release();
  return MPI_SUCCESS;
}

int MPIX_World_finalize(void) {
  std::lock_guard<std::mutex> lk(g_world_mu);
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  World* w = g_world;
  std::vector<cudaStream_t> held;
  for (auto& kv : w->batches) held.push_back(kv.first);
  for (cudaStream_t s : held) flush_stream(s);
  for (auto& rs : w->ranks) {
    cudaSetDevice(rs->device);
    cudaDeviceSynchronize();
  }
  for (auto* c : w->all_comms) {
    RankState& rs = *w->ranks[c->rank];
    cudaSetDevice(rs.device);
    if (c->sh && c->sh->base[c->rank]) {
      cudaFreeAsync(c->sh->base[c->rank], rs.aux);
      c->sh->base[c->rank] = nullptr;
    }
    delete c;
  }
  for (auto* c : w->world_comms) {
    RankState& rs = *w->ranks[c->rank];
    cudaSetDevice(rs.device);
    if (c->sh->base[c->rank]) cudaFreeAsync(c->sh->base[c->rank], rs.aux);
    c->sh->base[c->rank] = nullptr;
    delete c;
  }
  for (auto& rs : w->ranks) {
    cudaSetDevice(rs->device);
    for (auto& sb : rs->stage) cudaFreeAsync(sb.p, rs->aux);
    if (rs->d_arena) cudaFreeAsync(rs->d_arena, rs->aux);
    if (rs->d_arena_state) cudaFreeAsync(rs->d_arena_state, rs->aux);
    cudaStreamSynchronize(rs->aux);
    cudaFree(rs->d_done);
    cudaFree(rs->d_rec);
    if (rs->d_trace) cudaFree(rs->d_trace);
    cudaFreeHost(rs->h_err);
    cudaStreamDestroy(rs->aux);
    cudaStreamDestroy(rs->p2p);
    cudaFreeHost(rs->h_stage);
    if (rs->pool) cudaMemPoolDestroy(rs->pool);
  }
  delete w;
  g_world = nullptr;
  return MPI_SUCCESS;
}

int MPIX_World_size(int* n) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  *n = g_world->n;
  return MPI_SUCCESS;
}

int MPIX_World_comm(int rank, MPI_Comm* comm) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (rank < 0 || rank >= g_world->n) return MPIX_ERR_INVALID_RANK;
  *comm = g_world->world_comms[rank];
  return MPI_SUCCESS;
}

int MPIX_Rank_bind(int rank) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (rank < 0 || rank >= g_world->n) return MPIX_ERR_INVALID_RANK;
  t_bound_rank = rank;
  return MPI_SUCCESS;
}

int MPIX_Comm_world_self(MPI_Comm* comm) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (t_bound_rank < 0) return MPIX_ERR_INVALID_RANK;
  *comm = g_world->world_comms[t_bound_rank];
  return MPI_SUCCESS;
}

int MPI_Comm_rank(MPI_Comm comm, int* rank) {
  if (!comm) return MPIX_ERR_INVALID_COMM;
  *rank = comm->rank;
  return MPI_SUCCESS;
}

int MPI_Comm_size(MPI_Comm comm, int* size) {
  if (!comm) return MPIX_ERR_INVALID_COMM;
  *size = comm->sh->P;
  return MPI_SUCCESS;
}

int MPI_Barrier(MPI_Comm comm) {  // proc_comm.cpp:31-46 (host-side)
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!comm) return MPIX_ERR_INVALID_COMM;
  comm->sh->rv.exchange(comm->sh->P, comm->rank, comm->rv_seq++, CollMsg{});
  return MPI_SUCCESS;
}

int MPI_Comm_free(MPI_Comm* comm) {  // proc_comm.cpp:178-194
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!comm || !*comm) return MPIX_ERR_INVALID_COMM;
  mpix_comm_s* c = *comm;
  if (c->sh->is_world) return MPIX_ERR_INVALID_COMM;
  World& w = *g_world;
  RankState& rs = rank_of(c->rank);
  const int P = c->sh->P;
  // Every member's outstanding work on this comm must retire before any
  // region is released: exchange one event per member and make each aux
  // stream wait on all of them.
  cudaEvent_t ev = nullptr;
  if (c->cu && flush_stream(c->cu) < 0) return MPIX_ERR_CUDA;
  CK(cudaSetDevice(rs.device));
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, c->cu ? c->cu : rs.aux));
  CollMsg m;
  m.p0 = ev;
  auto v = c->sh->rv.exchange(P, c->rank, c->rv_seq++, m);
  for (int q = 0; q < P; ++q) CK(cudaStreamWaitEvent(rs.aux, (cudaEvent_t)v[q].p0, 0));
  // Nobody destroys an event before all members have enqueued their waits.
  c->sh->rv.exchange(P, c->rank, c->rv_seq++, CollMsg{});
  CK(cudaEventDestroy(ev));
  uint8_t* region = c->sh->base[c->rank];
  if (region) CK(cudaFreeAsync(region, rs.aux));
  c->sh->base[c->rank] = nullptr;
  for (auto* s : c->local_streams)
    if (s) s->refcount.fetch_sub(1);
  if (c->rank == 0) w.retire_ctx(c->sh->ctx);
  {
    std::lock_guard<std::mutex> lk(w.comms_mu);
    w.all_comms.erase(std::remove(w.all_comms.begin(), w.all_comms.end(), c), w.all_comms.end());
  }
  delete c;
  *comm = MPI_COMM_NULL;
  return MPI_SUCCESS;
}

// --------------------------------------------------------------------------
// Info
// --------------------------------------------------------------------------
int MPI_Info_create(MPI_Info* info) {
  if (!info) return MPIX_ERR_INVALID_ARG;
  *info = new mpix_info_s();
  return MPI_SUCCESS;
}

int MPI_Info_free(MPI_Info* info) {
  if (!info || !*info) return MPIX_ERR_INVALID_ARG;
  delete *info;
  *info = MPI_INFO_NULL;
  return MPI_SUCCESS;
}

int MPI_Info_set(MPI_Info info, const char* key, const char* value) {
  if (!info || !key || !value) return MPIX_ERR_INVALID_ARG;
  info->entries[key] = value;
  return MPI_SUCCESS;
}

int MPI_Info_get(MPI_Info info, const char* key, int valuelen, char* value, int* flag) {
  if (!info || !key || !flag) return MPIX_ERR_INVALID_ARG;
  auto it = info->entries.find(key);
  if (it == info->entries.end()) {
    *flag = 0;
    return MPI_SUCCESS;
  }
  *flag = 1;
  if (value && valuelen > 0) {
    size_t n = std::min((size_t)valuelen - 1, it->second.size());
    memcpy(value, it->second.data(), n);
    value[n] = 0;
  }
  return MPI_SUCCESS;
}

int MPIX_Info_set_hex(MPI_Info info, const char* key, const void* value, int vallen) {
  if (!info || !key || vallen < 0 || (vallen > 0 && !value)) return MPIX_ERR_INVALID_ARG;
  info->entries[key] = hex_encode(value, (size_t)vallen);
  return MPI_SUCCESS;
}

int MPIX_Info_get_hex(MPI_Info info, const char* key, void* value, int maxlen, int* outlen) {
  if (!info || !key) return MPIX_ERR_INVALID_ARG;
  auto it = info->entries.find(key);
  if (it == info->entries.end()) return MPIX_ERR_NOT_FOUND;
  std::vector<uint8_t> out;
  int rc = hex_decode(it->second, out);
  if (rc) return rc;
  if (outlen) *outlen = (int)out.size();
  if (value && maxlen > 0) memcpy(value, out.data(), std::min((size_t)maxlen, out.size()));
  return MPI_SUCCESS;
}

// --------------------------------------------------------------------------
// Streams
// --------------------------------------------------------------------------
int MPIX_Stream_create(MPI_Info info, MPIX_Stream* stream) {
  if (!stream) return MPIX_ERR_INVALID_ARG;
  auto s = std::make_unique<mpix_stream_s>();
  s->kind = mpix_stream_s::serial;
  s->exclusive = true;
  if (info) {
    auto it = info->entries.find("type");
    if (it != info->entries.end()) {  // proc_stream.cpp:11-17
      if (it->second != "cudaStream_t") return MPIX_ERR_BAD_HINT;
      auto v = info->entries.find("value");
      if (v == info->entries.end()) return MPIX_ERR_BAD_HINT;
      std::vector<uint8_t> bytes;
      if (hex_decode(v->second, bytes) != MPI_SUCCESS) return MPIX_ERR_BAD_HINT;
      if (bytes.size() != sizeof(cudaStream_t)) return MPIX_ERR_BAD_HINT;
      cudaStream_t cs;
      memcpy(&cs, bytes.data(), sizeof(cs));
      int dev = -1;
      if (cudaStreamGetDevice(cs, &dev) != cudaSuccess) {
        cudaGetLastError();
        return MPIX_ERR_BAD_HINT;  // not a live stream
      }
      s->kind = mpix_stream_s::cuda;
      s->cu = cs;
      s->device = dev;
      s->exclusive = false;  // proc_stream.cpp:23-24
    }
    auto mm = info->entries.find("mpix_matching");  // this library's hint
    if (mm != info->entries.end()) {
      if (mm->second == "dynamic")
        s->matching = 1;
      else if (mm->second == "static")
        s->matching = 0;
      else
        return MPIX_ERR_BAD_HINT;
    }
    auto p = info->entries.find("endpoint_policy");  // proc_stream.cpp:27-33
    if (p != info->entries.end()) {
      if (p->second == "shared")
        s->exclusive = false;
      else if (p->second == "exclusive")
        s->exclusive = true;
      else
        return MPIX_ERR_BAD_HINT;
    }
  }
  *stream = s.release();
  return MPI_SUCCESS;
}

int MPIX_Stream_free(MPIX_Stream* stream) {  // proc_stream.cpp:49-60
  if (!stream || !*stream) return MPIX_ERR_INVALID_STREAM;
  if ((*stream)->refcount.load() > 0) return MPIX_ERR_IN_USE;
  delete *stream;
  *stream = MPIX_STREAM_NULL;
  return MPI_SUCCESS;
}

int MPIX_Stream_get_cuda(MPIX_Stream stream, void** cuda_stream) {
  if (!stream || !cuda_stream) return MPIX_ERR_INVALID_STREAM;
  *cuda_stream = stream->kind == mpix_stream_s::cuda ? (void*)stream->cu : nullptr;
  return MPI_SUCCESS;
}

// --------------------------------------------------------------------------
// Communicators
// --------------------------------------------------------------------------
int MPIX_Stream_comm_create(MPI_Comm parent, MPIX_Stream stream, MPI_Comm* newcomm) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!parent) return MPIX_ERR_INVALID_COMM;
  if (!newcomm) return MPIX_ERR_INVALID_ARG;
  return create_comm(parent, {stream}, false, newcomm);
}

int MPIX_Stream_comm_create_multiplex(MPI_Comm parent, int count, MPIX_Stream streams[],
                                      MPI_Comm* newcomm) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!parent) return MPIX_ERR_INVALID_COMM;
  if (!newcomm) return MPIX_ERR_INVALID_ARG;
  if (count <= 0 || !streams) return MPIX_ERR_EMPTY_LIST;  // proc_comm.cpp:55
  std::vector<mpix_stream_s*> v(streams, streams + count);
  return create_comm(parent, v, true, newcomm);
}

int MPIX_Stream_comm_create_multiple(MPI_Comm parent, int count, MPIX_Stream streams[],
                                     MPI_Comm* newcomm) {
  return MPIX_Stream_comm_create_multiplex(parent, count, streams, newcomm);
}

// --------------------------------------------------------------------------
// Enqueue
// --------------------------------------------------------------------------
int MPIX_Send_enqueue(const void* buf, int count, MPI_Datatype datatype, int dest, int tag,
                      MPI_Comm comm) {
  return p2p_enqueue(comm, const_cast<void*>(buf), count, datatype, dest, tag, false, true,
                     nullptr);
}

int MPIX_Recv_enqueue(void* buf, int count, MPI_Datatype datatype, int source, int tag,
                      MPI_Comm comm, MPI_Status* status) {
  int rc = p2p_enqueue(comm, buf, count, datatype, source, tag, true, true, nullptr);
  if (rc == MPI_SUCCESS && status) {
    status->MPI_SOURCE = source;
    status->MPI_TAG = tag;
    status->MPI_ERROR = MPI_SUCCESS;
    status->source_index = -2;
    status->count_bytes = UINT64_MAX;
    status->truncated = 0;
  }
  return rc;
}

int MPIX_Isend_enqueue(const void* buf, int count, MPI_Datatype datatype, int dest, int tag,
                       MPI_Comm comm, MPI_Request* request) {
  return p2p_enqueue(comm, const_cast<void*>(buf), count, datatype, dest, tag, false, false,
                     request);
}

int MPIX_Irecv_enqueue(void* buf, int count, MPI_Datatype datatype, int source, int tag,
                       MPI_Comm comm, MPI_Request* request) {
  return p2p_enqueue(comm, buf, count, datatype, source, tag, true, false, request);
}

int MPIX_Wait_enqueue(MPI_Request* request, MPI_Status* status) {
  if (!request) return MPIX_ERR_INVALID_REQUEST;
  return waitall_enqueue(1, request, status);
}

int MPIX_Waitall_enqueue(int count, MPI_Request requests[], MPI_Status statuses[]) {
  return waitall_enqueue(count, requests, statuses);
}

// --------------------------------------------------------------------------
// Conventional p2p and multiplex stream p2p (host-thread semantics)
// --------------------------------------------------------------------------
int MPI_Isend(const void* buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
              MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_ARG;
  return conv_post(comm, const_cast<void*>(buf), count, datatype, dest, tag, false, false, request);
}

int MPI_Irecv(void* buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_ARG;
  return conv_post(comm, buf, count, datatype, source, tag, true, false, request);
}

int MPI_Send(const void* buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm) {
  int rc = conv_post(comm, const_cast<void*>(buf), count, datatype, dest, tag, false, true, nullptr);
  return rc ? rc : host_blocking(rc, comm, rank_of(comm->rank).p2p, nullptr, dest, tag);
}

int MPI_Recv(void* buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
             MPI_Status* status) {
  int rc = conv_post(comm, buf, count, datatype, source, tag, true, true, nullptr);
  return rc ? rc : host_blocking(rc, comm, rank_of(comm->rank).p2p, status, source, tag);
}

int MPI_Wait(MPI_Request* request, MPI_Status* status) {
  if (!request) return MPIX_ERR_INVALID_REQUEST;
  return host_waitall(1, request, status);
}

int MPI_Waitall(int count, MPI_Request requests[], MPI_Status statuses[]) {
  return host_waitall(count, requests, statuses);
}

static cudaStream_t local_stream_of(MPI_Comm comm, int idx) {
  mpix_stream_s* ls = comm->local_streams[idx];
  return ls && ls->kind == mpix_stream_s::cuda ? ls->cu : rank_of(comm->rank).p2p;
}

int MPIX_Stream_isend(const void* buf, int count, MPI_Datatype datatype, int dest, int tag,
                      MPI_Comm comm, int src_idx, int dst_idx, MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_ARG;
  return stream_post(comm, const_cast<void*>(buf), count, datatype, dest, tag, src_idx, dst_idx,
                     false, false, request);
}

int MPIX_Stream_irecv(void* buf, int count, MPI_Datatype datatype, int source, int tag,
                      MPI_Comm comm, int src_idx, int dst_idx, MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_ARG;
  return stream_post(comm, buf, count, datatype, source, tag, src_idx, dst_idx, true, false, request);
}

int MPIX_Stream_send(const void* buf, int count, MPI_Datatype datatype, int dest, int tag,
                     MPI_Comm comm, int src_idx, int dst_idx) {
  int rc = stream_post(comm, const_cast<void*>(buf), count, datatype, dest, tag, src_idx, dst_idx,
                       false, true, nullptr);
  return rc ? rc : host_blocking(rc, comm, local_stream_of(comm, src_idx), nullptr, dest, tag);
}

int MPIX_Stream_recv(void* buf, int count, MPI_Datatype datatype, int source, int tag,
                     MPI_Comm comm, int src_idx, int dst_idx, MPI_Status* status) {
  int rc = stream_post(comm, buf, count, datatype, source, tag, src_idx, dst_idx, true, true,
                       nullptr);
  return rc ? rc : host_blocking(rc, comm, local_stream_of(comm, dst_idx), status, source, tag);
}

int MPIX_Request_free(MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_REQUEST;
  *request = MPI_REQUEST_NULL;
  return MPI_SUCCESS;
}

int MPIX_Allreduce_enqueue(const void* sendbuf, void* recvbuf, int count, MPI_Datatype datatype,
                           MPI_Op op, MPI_Comm comm) {
  return coll_enqueue(CK_ALLREDUCE, sendbuf, recvbuf, count, datatype, op, 0, comm);
}

int MPIX_Reduce_enqueue(const void* sendbuf, void* recvbuf, int count, MPI_Datatype datatype,
                        MPI_Op op, int root, MPI_Comm comm) {
  return coll_enqueue(CK_REDUCE, sendbuf, recvbuf, count, datatype, op, root, comm);
}

int MPIX_Reduce_scatter_block_enqueue(const void* sendbuf, void* recvbuf, int recvcount,
                                      MPI_Datatype datatype, MPI_Op op, MPI_Comm comm) {
  return coll_enqueue(CK_REDUCE_SCATTER, sendbuf, recvbuf, recvcount, datatype, op, 0, comm);
}

int MPIX_Bcast_enqueue(void* buffer, int count, MPI_Datatype datatype, int root, MPI_Comm comm) {
  return coll_enqueue(CK_BCAST, buffer, buffer, count, datatype, MPI_SUM, root, comm);
}

int MPIX_Allgather_enqueue(const void* sendbuf, int sendcount, MPI_Datatype sendtype, void* recvbuf,
                           int recvcount, MPI_Datatype recvtype, MPI_Comm comm) {
  if (sendbuf != MPI_IN_PLACE &&
      (uint64_t)sendcount * type_size(sendtype) != (uint64_t)recvcount * type_size(recvtype))
    return MPIX_ERR_INVALID_COUNT;
  return coll_enqueue(CK_ALLGATHER, sendbuf, recvbuf, recvcount, recvtype, MPI_SUM, 0, comm);
}

int MPIX_Barrier_enqueue(MPI_Comm comm) {
  return coll_enqueue(CK_BARRIER, nullptr, nullptr, 0, MPI_BYTE, MPI_SUM, 0, comm);
}

// --------------------------------------------------------------------------
// Introspection
// --------------------------------------------------------------------------
uint64_t MPIX_Launch_count(void) { return g_launches.load(); }

int MPIX_Config_get(uint64_t* eager_bytes, int* ring_slots, int* max_ctas,
                    uint64_t* oneshot_max_bytes) {
  Config c = g_world ? g_world->cfg : Config::from_env();
  if (eager_bytes) *eager_bytes = c.eager_bytes;
  if (ring_slots) *ring_slots = c.ring_slots;
  if (max_ctas) *max_ctas = (int)c.inline_bytes;
  if (oneshot_max_bytes) *oneshot_max_bytes = c.oneshot_max;
  return MPI_SUCCESS;
}

int MPIX_Comm_get_ctx(MPI_Comm comm, uint32_t* ctx) {
  if (!comm) return MPIX_ERR_INVALID_COMM;
  *ctx = comm->sh->ctx;
  return MPI_SUCCESS;
}

int MPIX_Comm_is_enqueue(MPI_Comm comm, int* flag) {
  if (!comm) return MPIX_ERR_INVALID_COMM;
  *flag = comm->enqueue_ok ? 1 : 0;
  return MPI_SUCCESS;
}

int MPIX_Type_size(MPI_Datatype datatype) { return type_size(datatype); }

int MPIX_Rank_error(int rank, uint64_t* code) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (rank < 0 || rank >= g_world->n || !code) return MPIX_ERR_INVALID_RANK;
  *code = *reinterpret_cast<volatile uint64_t*>(g_world->ranks[rank]->h_err);
  return MPI_SUCCESS;
}

int MPIX_Trace_read(int rank, void* out, int max_records, int* n_records) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (rank < 0 || rank >= g_world->n) return MPIX_ERR_INVALID_RANK;
  RankState& rs = *g_world->ranks[rank];
  if (!rs.d_trace) {
    if (n_records) *n_records = 0;
    return MPI_SUCCESS;
  }
  int n = (int)std::min<uint64_t>({(uint64_t)max_records, rs.trace_next.load(), kTraceRecs});
  CK(cudaSetDevice(rs.device));
  CK(cudaDeviceSynchronize());
  if (n > 0) CK(cudaMemcpy(out, rs.d_trace, (size_t)n * sizeof(TraceRec), cudaMemcpyDeviceToHost));
  if (n_records) *n_records = n;
  return MPI_SUCCESS;
}

int MPIX_Comm_region(MPI_Comm comm, void** base, uint64_t* bytes) {
  if (!comm) return MPIX_ERR_INVALID_COMM;
  if (base) *base = comm->sh->base[comm->rank];
  if (bytes) *bytes = comm->sh->L.total();
  return MPI_SUCCESS;
}

int MPIXT_Reduce_only(int P, int me, void** sendbufs, void** recvbufs, int count,
                      MPI_Datatype datatype, MPI_Op op, int twoshot, void* stream) {
  int dtype, aop;
  switch (datatype) {
    case MPI_INT: dtype = AR_I32; break;
    case MPI_FLOAT: dtype = AR_F32; break;
    case MPIX_BFLOAT16: dtype = AR_BF16; break;
    case MPI_DOUBLE: dtype = AR_F64; break;
    default: return MPIX_ERR_TYPE;
  }
  switch (op) {
    case MPI_SUM: aop = AR_SUM; break;
    case MPI_MAX: aop = AR_MAX; break;
    case MPI_MIN: aop = AR_MIN; break;
    default: return MPIX_ERR_OP;
  }
  if (P < 1 || P > kMaxCollRanks || me < 0 || me >= P || count < 0) return MPIX_ERR_INVALID_ARG;
  static OpRecord* rec = nullptr;
  if (!rec && cudaMalloc(&rec, sizeof(OpRecord)) != cudaSuccess) return MPIX_ERR_CUDA;
  std::vector<uint64_t> sb(P), rb(P);
  for (int q = 0; q < P; ++q) {
    sb[q] = (uint64_t)sendbufs[q];
    rb[q] = (uint64_t)recvbufs[q];
  }
  int rc = launch_reduce_only(sb.data(), rb.data(), P, me, (uint64_t)count, type_size(datatype),
                              dtype, aop, twoshot ? AR_TWOSHOT : AR_ONESHOT, rec,
                              (cudaStream_t)stream);
  return rc < 0 ? MPIX_ERR_CUDA : MPI_SUCCESS;
}

int MPIXT_Copy_timing(int enable) {
  std::lock_guard<std::mutex> tl(g_copy_timing.mu);
  for (auto& p : g_copy_timing.ev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  g_copy_timing.ev.clear();
  g_copy_timing.on.store(enable != 0);
  return MPI_SUCCESS;
}

int MPIXT_Copy_timing_read(double* total_ms, int* n) {
  std::lock_guard<std::mutex> tl(g_copy_timing.mu);
  double tot = 0;
  for (auto& p : g_copy_timing.ev) {
    if (cudaEventSynchronize(p.second) != cudaSuccess) return MPIX_ERR_CUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, p.first, p.second);
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (n) *n = (int)g_copy_timing.ev.size();
  return MPI_SUCCESS;
}

const char* MPIX_Version(void) { return "mpix-b200 0.1 (sm_100a)"; }

}  // extern "C"
