// mpix_p2p.cpp — point-to-point behind include/mpix.h: coalesced launches
// (DESIGN.md §3), the enqueue family (Proc::*_enqueue,
// proj/src/proc_enqueue.cpp:8-141), conventional host-thread p2p and
// multiplex stream p2p (proj/src/proc_p2p.cpp:96-212), and the waits.
#include "mpix_state.h"

#include <chrono>
#include <cstdio>
#include <functional>
#include <thread>

namespace mpix {

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
  // graph-capturable comms: mark each device counter's last operation (the
  // final launch advances the counter past it)
  uint32_t* arrive = nullptr;
  if (!b.grel.empty()) {
    arrive = b.d_arrive;
    std::unordered_set<const uint64_t*> seen;
    for (int i = n - 1; i >= 0; --i) {
      BatchOp& o = b.ops[i];
      if (!(o.gflags & G_ON)) continue;
      if (seen.insert(o.bases + o.gp).second) o.gflags |= G_LASTP;
      if (seen.insert(o.bases + o.gt).second) o.gflags |= G_LASTT;
    }
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_copy_timing.on.load()) {
    std::vector<OpRecord*> recs;
    for (auto& o : b.ops)
      if (!o.inl) recs.push_back(o.rec);
    if (!recs.empty()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      std::lock_guard<std::mutex> tl(g_copy_timing.mu);
      g_copy_timing.ev.push_back({e0, e1, b.device, std::move(recs)});
    }
  }
  do {
    int m = std::min(nwait - wi, kBatchWaits);
    int rc = launch_batch(b.ops.data(), n, w + wi, m, err, cfg.spin_limit_ns, b.sys || wsys, s,
                          e0, e1, n ? arrive : nullptr);
    e0 = e1 = nullptr;
    if (rc < 0) return -1;
    launches += rc;
    n = 0;
    b.ops.clear();
    b.first_large_pseq.clear();
    b.post_only.clear();
    b.gmates.clear();
    b.grel.clear();
    wi += m;
  } while (wi < nwait);
  b.sys = false;
  b.err_word = nullptr;
  b.t_first = 0;
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

// ---------------------------------------------------------------------------
// Flusher thread: the progress guarantee of held batches. A non-blocking
// operation held in a stream's batch is normally launched by that stream's
// next ordering call; the reference instead registers I-operations at their
// own queue position (proc_enqueue.cpp:67-114), so a program that never
// makes such a call (e.g. Isend_enqueue on stream A, then a host wait on
// stream B for the matching receive) must still progress: any batch held
// longer than cfg.flush_ns is launched here.
// ---------------------------------------------------------------------------
static uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void batch_note_held(StreamBatch& b) {
  if (b.t_first) return;
  b.t_first = now_ns();
  World& w = *g_world;
  if (w.cfg.flush_ns && !w.fl_armed.exchange(true)) {
    std::lock_guard<std::mutex> lk(w.fl_mu);
    w.fl_cv.notify_one();
  }
}

// Launch every batch older than flush_ns; returns the ns until the next one
// is due (0: nothing held).
static uint64_t flush_due(World& w) {
  std::vector<std::pair<cudaStream_t, StreamBatch*>> v;
  {
    std::lock_guard<std::mutex> lk(w.batch_mu);
    v.reserve(w.batches.size());
    for (auto& kv : w.batches) v.emplace_back(kv.first, kv.second.get());
  }
  uint64_t next = 0;
  for (auto& e : v) {
    StreamBatch& b = *e.second;
    std::unique_lock<std::mutex> lk(b.mu, std::try_to_lock);
    if (!lk.owns_lock()) {  // its owner is working on it right now
      next = next ? std::min(next, w.cfg.flush_ns) : w.cfg.flush_ns;
      continue;
    }
    if (b.ops.empty()) continue;
    const uint64_t age = now_ns() - b.t_first;
    if (age < w.cfg.flush_ns) {
      const uint64_t d = w.cfg.flush_ns - age;
      next = next ? std::min(next, d) : d;
      continue;
    }
    // a batch of a stream being captured stays with its capture (its wait,
    // inside the capture, launches it)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(e.first, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      continue;
    }
    if (cudaSetDevice(b.device) == cudaSuccess) flush_locked(b, e.first, nullptr, 0, false, nullptr);
  }
  return next;
}

static void flusher_main(World* w) {
  std::unique_lock<std::mutex> lk(w->fl_mu);
  while (!w->fl_stop) {
    if (!w->fl_armed.load()) {
      w->fl_cv.wait(lk, [&] { return w->fl_stop || w->fl_armed.load(); });
      continue;
    }
    w->fl_armed.store(false);  // before the scan: a batch started after it re-arms
    lk.unlock();
    const uint64_t next = flush_due(*w);
    lk.lock();
    if (next) {
      w->fl_armed.store(true);
      w->fl_cv.wait_for(lk, std::chrono::nanoseconds(next), [&] { return w->fl_stop; });
    }
  }
}

void flusher_start(World& w) {
  if (!w.cfg.flush_ns || !w.cfg.batch) return;
  w.fl_stop = false;
  w.flusher = std::thread(flusher_main, &w);
}

void flusher_stop(World& w) {
  if (!w.flusher.joinable()) return;
  {
    std::lock_guard<std::mutex> lk(w.fl_mu);
    w.fl_stop = true;
  }
  w.fl_cv.notify_all();
  w.flusher.join();
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
  o.sidx = (int8_t)a.sidx;
  o.didx = (int8_t)a.didx;
  o.is_recv = (uint8_t)a.is_recv;
  o.mode = (uint8_t)a.mode;
  o.blocking = (uint8_t)a.blocking;
  o.inl = inl ? 1 : 0;
  o.ll = (uint8_t)a.ll;
  o.mate = -1;
  return o;
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
                  bool conventional, bool is_recv, int me, uint64_t bytes) {
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
  ri.is_recv = is_recv;
  ri.me = me;
  ri.bytes = bytes;
  ri.comm = nullptr;
  Ticket t;
  t.handle = ((uint64_t)(rs.rank + 1) << 48) | (n + 1);
  t.flag = rs.d_done + slot;
  t.gen = gen;
  return t;
}

// A request created while its stream is captured into a CUDA graph: a
// completion word of its own, set to 1 by the completion and consumed
// (reset to 0) by the captured wait, so every replay sees a fresh request.
constexpr uint64_t kGraphTicket = 1ull << 47;

int new_graph_ticket(RankState& rs, cudaStream_t s, int source, int tag, bool remote, bool is_recv,
                     int me, uint64_t bytes, Ticket* t) {
  uint64_t n = rs.gdone_next.fetch_add(1);
  if (n >= kGraphReqs) return MPIX_ERR_NO_MEM;
  auto& ri = rs.greqs[n];
  ri.gen = 1;
  ri.stream = s;
  ri.source = source;
  ri.tag = tag;
  ri.remote = remote;
  ri.conventional = false;
  ri.consumed = false;
  ri.is_recv = is_recv;
  ri.me = me;
  ri.bytes = bytes;
  ri.comm = nullptr;
  t->handle = ((uint64_t)(rs.rank + 1) << 48) | kGraphTicket | (n + 1);
  t->flag = rs.d_gdone + n;
  t->gen = 1;
  return MPI_SUCCESS;
}

bool decode_ticket(uint64_t h, int* rank, uint64_t* n, bool* graph = nullptr) {
  if (h == 0) return false;
  int r = (int)(h >> 48) - 1;
  if (r < 0 || !g_world || r >= g_world->n) return false;
  const bool g = (h & kGraphTicket) != 0;
  uint64_t v = h & (kGraphTicket - 1);
  if (v == 0 || (g && v > kGraphReqs)) return false;
  *rank = r;
  *n = v - 1;
  if (graph) *graph = g;
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
    uint64_t rel = 0;  // the buffer's release word
    if (mp_mode()) {   // in heap memory (a peer process releases it)
      if (cudaMemcpy(&rel, rs.d_stage + b, sizeof(rel), cudaMemcpyDeviceToHost) != cudaSuccess)
        return MPIX_ERR_CUDA;
    } else {
      rel = *reinterpret_cast<volatile uint64_t*>(&rs.h_stage[b]);
    }
    bool free = rel >= sb.gen;
    if (free && sb.size >= bytes && (best < 0 || sb.size < rs.stage[best].size)) best = (int)b;
  }
  if (best < 0) {
    if (rs.stage.size() >= kStageSlots) return MPIX_ERR_NO_MEM;
    uint64_t size = 1ull << 20;
    while (size < bytes) size <<= 1;
    RankState::StageBuf sb;
    if (mp_mode()) {  // the receiver (another process) pulls from it
      if (MPIX_Alloc_mem(size, (void**)&sb.p)) return MPIX_ERR_NO_MEM;
    } else if (cudaMallocFromPoolAsync((void**)&sb.p, size, rs.pool, s) != cudaSuccess) {
      return MPIX_ERR_NO_MEM;
    }
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
  uint64_t* ticket = nullptr; // out: the operation's ticket (blocking receives too)
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

// The stream conventional operations of comm c run on: the rank's internal
// stream, or — graph-capturable comm, whose device counters must be read
// and advanced in one stream order — the comm's own stream.
cudaStream_t conv_stream(mpix_comm_s* c) {
  if (c->graph && c->cu) return c->cu;
  RankState& rs = rank_of(c->rank);
  // One internal stream per communicator (every host exclusion regime: the
  // regimes differ in host locking only): threads on different comms never
  // queue behind each other's blocking operations — with one stream per
  // rank, a blocking MPI_Recv kernel of one thread would stall the operations
  // its peer is waiting for (a cross-rank deadlock the reference's global
  // progress does not have)
  std::call_once(c->conv_once, [&] {
    {
      std::lock_guard<std::mutex> pl(rs.conv_pool_mu);
      if (!rs.conv_pool.empty()) {
        c->conv_cu = rs.conv_pool.back();
        rs.conv_pool.pop_back();
        return;
      }
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(rs.device);
    if (cudaStreamCreateWithFlags(&c->conv_cu, cudaStreamNonBlocking) != cudaSuccess) c->conv_cu = nullptr;
    if (prev >= 0) cudaSetDevice(prev);
  });
  return c->conv_cu ? c->conv_cu : rs.p2p;
}

// The host exclusion of one p2p call (Config::excl; EndpointGuard,
// proj/include/streamix/fabric.hpp:17-61): the process-wide lock, the
// communicator's lock, or — a serial-context communicator under the serial
// regime — nothing (with the optional owner trap).
struct CommGuard {
  std::unique_lock<std::mutex> lk;
  std::atomic<uint64_t>* owner = nullptr;
  CommGuard(mpix_comm_s* c) {
    const Config& cfg = g_world->cfg;
    if (cfg.excl == 0) {
      lk = std::unique_lock<std::mutex>(g_world->global_mu);
    } else if (cfg.excl == 2 && c->serial_ctx) {
      if (cfg.serial_check) {
        const uint64_t me = (uint64_t)std::hash<std::thread::id>()(std::this_thread::get_id()) | 1;
        uint64_t prev = c->owner.exchange(me);
        if (prev != 0 && prev != me) {
          std::fprintf(stderr, "mpix: concurrent entry into a serial-context communicator "
                               "(MPIX_HOST_EXCLUSION=serial contract violated)\n");
          std::abort();
        }
        owner = &c->owner;
      }
    } else {
      lk = std::unique_lock<std::mutex>(c->mu);
    }
  }
  ~CommGuard() {
    if (owner) owner->store(0);
  }
};

// Conventional p2p (Proc::isend/irecv, proc_p2p.cpp:96-113) on GPU buffers:
// executed on the rank's internal stream, launched at once (no batching:
// a posted conventional send must progress without a later MPI call).
int conv_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
              bool is_recv, bool blocking, MPI_Request* req, uint64_t* ticket = nullptr) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (c->sh->multiplex) return MPIX_ERR_MULTIPLEX_COMM;
  int rc = check_p2p_args(c, count, peer, tag, is_recv);
  if (rc) return rc;
  PostHow how;
  how.stream = conv_stream(c);
  how.conventional = true;
  how.ticket = ticket;
  return p2p_post(c, buf, count, dt, peer, tag, is_recv, blocking, req, how);
}

// Multiplex stream p2p (Proc::stream_isend/irecv, proc_p2p.cpp:115-144):
// runs on the CUDA stream of local stream src_idx (send) / dst_idx (recv),
// or on the rank's internal stream when that MPIX stream is not a GPU stream.
int stream_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
                int src_idx, int dst_idx, bool is_recv, bool blocking, MPI_Request* req,
                uint64_t* ticket = nullptr) {
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
    // a wildcard index needs the dynamic engine (it filters on the indices);
    // the static key carries concrete ones
    if (src_idx == MPIX_ANY_INDEX && !c->sh->dyn) return MPIX_ERR_UNSUPPORTED;
  }
  const int local = is_recv ? dst_idx : src_idx;
  mpix_stream_s* ls = c->local_streams[local];
  PostHow how;
  how.stream = ls && ls->kind == mpix_stream_s::cuda ? ls->cu : rank_of(me).p2p;
  how.conventional = true;
  how.sidx = src_idx;
  how.didx = dst_idx;
  how.ticket = ticket;
  return p2p_post(c, buf, count, dt, peer, tag, is_recv, blocking, req, how);
}

int p2p_post(mpix_comm_s* c, void* buf, int count, MPI_Datatype dt, int peer, int tag,
             bool is_recv, bool blocking, MPI_Request* req, const PostHow& how) {
  if (int h = rank_health(rank_of(c->rank))) return h;  // sticky watchdog state
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
  const bool indexed = how.sidx != -2;  // IDX_NONE (types.hpp:14) outside multiplex
  // Multi-process mode: a receive buffer is pushed into by the sender and an
  // Isend buffer pulled by the receiver, so both must be heap memory; a
  // blocking send reads its own buffer (eager or staged copies).
  if ((is_recv || !blocking) && !peer_ok(buf, bytes)) return MPIX_ERR_INVALID_ARG;
  // CUDA-Graph capture: a graph-capturable comm takes its
  // sequence numbers from device counters; any other comm would replay
  // stale ones (checked here for blocking operations and at the wait, off
  // the non-blocking fast path).
  const bool gr = c->graph;
  bool capturing = false;
  if (gr || blocking) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(how.stream, &cs) != cudaSuccess) return MPIX_ERR_CUDA;
    capturing = cs != cudaStreamCaptureStatusNone;
    if (capturing && !gr) return MPIX_ERR_UNSUPPORTED;
  }
  if (capturing && !is_recv && blocking && bytes > L.E && bytes > w.cfg.stage_chunk)
    return MPIX_ERR_UNSUPPORTED;  // host staging buffers are reclaimed by the host
  CommGuard clk(c);

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
  a.me = me;      // the status source of a receive this operation completes
  a.peer = peer;  // -1 = ANY_SOURCE (receives, dynamic matching)
  a.tag = tag;    // -1 = ANY_TAG (receives, dynamic matching)
  a.sidx = how.sidx;  // multiplex stream indices (-2 none)
  a.didx = how.didx;
  // flag-in-data small sends and polling blocking receives (static matching)
  a.ll = w.cfg.ll && !dyn ? 1 : 0;
  if (dyn) {
    a.dyn = 1;
    a.P = sh.P;
    a.bases = reinterpret_cast<uint64_t*>(sh.base[me] + L.bases());
  }

  // graph-capturable: the pair-sequence counter and the (direction, peer,
  // tag) match-sequence counter of this operation
  uint16_t gp = 0, gt = 0;
  if (gr) {
    gp = (uint16_t)(is_recv ? sh.P + peer : peer);
    const uint64_t tk = ((uint64_t)is_recv << 63) | ((uint64_t)(uint32_t)peer << 32) | (uint32_t)tag;
    auto it = c->gtag.find(tk);
    if (it == c->gtag.end()) {
      if (c->gtag.size() >= kGraphTagCounters) return MPIX_ERR_UNSUPPORTED;
      it = c->gtag.emplace(tk, (uint16_t)(2 * sh.P + 1 + c->gtag.size())).first;
    }
    gt = it->second;
  }

  const bool sys = w.cfg.force_sys ||
                   (dyn ? c->any_remote : rank_of(peer).device != rs.device);
  // the rank's device is made current only before a CUDA call: a held
  // (batched) operation makes none, and cudaSetDevice is ~1/4 of its host cost
  bool dev_set = false;
  auto ensure_dev = [&]() -> bool {
    if (!dev_set) dev_set = cudaSetDevice(rs.device) == cudaSuccess;
    return dev_set;
  };
  cudaStream_t s = how.stream;
  Ticket t{};
  if (!blocking || is_recv) {
    if (capturing) {
      int rc2 = new_graph_ticket(rs, s, is_recv ? peer : me, tag, sys, is_recv, me, bytes, &t);
      if (rc2) return rc2;
    } else {
      t = new_ticket(rs, s, is_recv ? peer : me, tag, sys, how.conventional, is_recv, me, bytes);
      if (how.conventional && is_recv) {  // MPI_Comm_free's PENDING_OPS check
        auto& v = c->conv_recvs;
        if (v.size() >= 256) {  // drop the ones already waited
          v.erase(std::remove_if(v.begin(), v.end(),
                                 [&](const std::pair<uint64_t*, uint64_t>& e) {
                                   auto& r = rs.reqs[(uint64_t)(e.first - rs.d_done) % kReqSlots];
                                   return r.consumed || r.gen != e.second;
                                 }),
                  v.end());
        }
        v.emplace_back(t.flag, t.gen);
        rs.reqs[(uint64_t)(t.flag - rs.d_done)].comm = c;
      }
    }
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
      if (!ensure_dev()) return MPIX_ERR_CUDA;
      int rc2 = acquire_staging(rs, bytes, s, &a.staging, &a.stage_done, &a.stage_gen);
      if (rc2) return rc2;
    }
  }
  if (rs.d_trace && !gr) {
    uint64_t n = rs.trace_next.fetch_add(1);
    a.trace = rs.d_trace + (n % kTraceRecs);
    a.trace_seq = n + 1;
  }
  bool inl = bytes <= w.cfg.inline_bytes || (!is_recv && a.mode == MODE_EAGER);
  bool post_only = false;
  if (!blocking && peer == me && !dyn && !how.conventional && !gr) {
    // Self-message whose counterpart has not been enqueued yet: it can only
    // be enqueued later on this same stream (an enqueue comm has one stream),
    // so it runs after this operation, which therefore only posts and never
    // copies: one small launch instead of proto + copy grid + fin. Small
    // ones too: if the counterpart joins the same batch, the host pairs them
    // (one copy, no descriptors, no Dekker race between two CTAs).
    const auto& other = is_recv ? c->send_tagseq : c->recv_tagseq;
    auto it = other.find(tagseq_key(me, tag));
    if (it == other.end() || it->second <= tseq) inl = post_only = true;
  }
  if (!inl && capturing) {  // a decision record no later operation reuses
    uint64_t k = rs.grec_next.fetch_add(1);
    if (k >= kGraphRecs) return MPIX_ERR_NO_MEM;
    a.rec = rs.d_grec + k;
    a.opid = k;
  } else if (!inl) {
    uint64_t op = rs.op_next.fetch_add(1);
    a.rec = rs.d_rec + (op % kOpRecords);
    a.opid = op;
  }
  if (!c->batch && !how.conventional) c->batch = &batch_of(s, rs.device);
  // the batch of a conventional operation's stream: the comm's internal
  // stream's is looked up once (no process-wide lock per operation)
  StreamBatch* bp = c->batch;
  if (how.conventional) {
    if (s == c->conv_cu) {
      if (!c->conv_batch) c->conv_batch = &batch_of(s, rs.device);
      bp = c->conv_batch;
    } else {
      bp = &batch_of(s, rs.device);
    }
  }
  StreamBatch& b = *bp;
  std::lock_guard<std::mutex> lk(b.mu);
  if ((w.cfg.batch || gr) && !a.trace) {
    // Join the stream's batch; a blocking operation closes it (it must have
    // completed before anything behind it in the stream runs).
    // A self-message whose counterpart is held post-only in this batch: the
    // host has matched them (same comm, same key, static matching), so the
    // two become one paired operation — no descriptors, one copy.
    int pk = -1;
    if (!dyn && !gr && peer == me && (!blocking || is_recv) && a.mode != MODE_STAGED) {
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
      // graph-capturable: sequences relative to the batch's start (the
      // kernels add the device counters)
      const uint64_t* pc = c->d_gseq + gp;
      const uint64_t* tc = c->d_gseq + gt;
      auto relative = [&] {
        a.pseq = b.grel[pc];
        a.key = ((uint64_t)(uint32_t)tag << 32) | b.grel[tc];
      };
      if (gr) relative();
      bool flush_first = (int)b.ops.size() >= kBatchOps;
      auto fl = b.first_large_pseq.find(a.post_mirror);
      flush_first |= fl != b.first_large_pseq.end() && a.pseq >= fl->second + (uint64_t)a.R;
      for (auto& po : b.post_only) flush_first |= po.comm == c && po.key == a.key;
      // graph-capturable comm (no host pairing): a blocking self-receive
      // whose send is in this batch could wait in k_batch for the send's
      // push, which only the k_gcopy behind it performs — launch the send first
      flush_first |= gr && blocking && is_recv && peer == me && !b.ops.empty();
      // a blocking receive may wait inside k_batch for a peer's push; that
      // push can sit in the peer's own k_gcopy behind a k_batch whose blocking
      // receive waits for MY deferred copy (head-to-head large Isend + Recv,
      // found by tests/test_gpu_model_check.py): never let a blocking receive
      // share a launch with a copy-grid operation
      if (blocking && is_recv && !flush_first)
        for (const BatchOp& o : b.ops) flush_first |= !o.inl;
      if (gr && !b.d_arrive) {
        uint32_t k = rs.arrive_next.fetch_add(1);
        if (k >= kArriveWords) return MPIX_ERR_NO_MEM;
        b.d_arrive = rs.d_arrive + k;
      }
      if (flush_first) {
        if (!ensure_dev() || flush_locked(b, s, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
        if (gr) relative();
      }
      if (b.ops.empty()) b.err_word = rs.d_err;
      if (!inl && a.post_mirror) b.first_large_pseq.emplace(a.post_mirror, a.pseq);
      if (post_only) b.post_only.push_back({c, a.key, b.ops.size(), (bool)is_recv});
      // graph-capturable self-message: remember it, or mate it with the
      // opposite operation of the same (relative) key already in this batch
      int mate = -1;
      if (gr && peer == me && !blocking && inl) {
        for (size_t k = 0; k < b.gmates.size() && mate < 0; ++k) {
          const auto& gm = b.gmates[k];
          if (gm.comm == c && gm.key == a.key && gm.is_recv != is_recv) {
            mate = (int)gm.idx;
            b.gmates.erase(b.gmates.begin() + k);
          }
        }
        if (mate < 0) b.gmates.push_back({c, a.key, b.ops.size(), (bool)is_recv});
      }
      b.ops.push_back(pack_op(a, inl));
      if (mate >= 0) {
        b.ops.back().mate = (int16_t)mate;
        b.ops[mate].mate = (int16_t)(b.ops.size() - 1);
      }
      if (gr) {
        BatchOp& o = b.ops.back();
        o.bases = c->d_gseq;
        o.gp = gp;
        o.gt = gt;
        o.gflags = G_ON | ((capturing && blocking && is_recv) ? G_RESET : 0);
        b.grel[pc] += 1;
        b.grel[tc] += 1;
      }
      b.sys |= sys;
    }
    // a blocking operation closes the batch; conventional operations are
    // launched at once
    // conventional operations are held like enqueued ones (MPIX_CONV_BATCH,
    // default on): launched by the thread's next ordering call on that
    // stream (a blocking operation or a wait) or, failing one, by the flusher
    if (blocking || (how.conventional && !w.cfg.conv_batch) || !w.cfg.batch) {
      if (!ensure_dev() || flush_locked(b, s, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
    } else if (!b.ops.empty()) {
      batch_note_held(b);  // the flusher launches it if no ordering call comes
    }
  } else {
    if (!ensure_dev()) return MPIX_ERR_CUDA;
    if (!b.ops.empty() && flush_locked(b, s, nullptr, 0, false, nullptr) < 0) return MPIX_ERR_CUDA;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (!inl && g_copy_timing.on.load()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      std::lock_guard<std::mutex> tl(g_copy_timing.mu);
      g_copy_timing.ev.push_back({e0, e1, rs.device, {a.rec}});
    }
    a.early_trigger = p2p_copy_grid(bytes) <= kEarlyTriggerTiles;
    int nk = launch_p2p(a, sys, inl, inl ? 1 : p2p_copy_grid(bytes), s, e0, e1);
    if (nk < 0) return MPIX_ERR_CUDA;
    g_launches.fetch_add(nk);
  }
  if (s != c->cu &&
      std::find(c->side_streams.begin(), c->side_streams.end(), s) == c->side_streams.end())
    c->side_streams.push_back(s);
  if (req) *req = (!blocking) ? t.handle : MPI_REQUEST_NULL;
  if (how.ticket) *how.ticket = t.handle;
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
    bool graph;
  };
  std::vector<Item> items(n);
  int ngraph = 0;
  for (int i = 0; i < n; ++i) {  // proc_enqueue.cpp:122-123
    if (!decode_ticket(reqs[i], &items[i].rank, &items[i].n, &items[i].graph))
      return MPIX_ERR_INVALID_REQUEST;
    ngraph += items[i].graph;
  }
  if (int h = rank_health(rank_of(items[0].rank))) return h;  // sticky watchdog state
  auto info = [&](const Item& it) -> RankState::ReqInfo& {
    RankState& rs = rank_of(it.rank);
    return it.graph ? rs.greqs[it.n] : rs.reqs[it.n % kReqSlots];
  };
  cudaStream_t s0 = nullptr;
  int dev0 = -1;
  bool sys = false;
  for (int i = 0; i < n; ++i) {  // proc_enqueue.cpp:124-126
    RankState& rs = rank_of(items[i].rank);
    auto& ri = info(items[i]);
    cudaStream_t s = items[i].graph || ri.gen == items[i].n / kReqSlots + 1 ? ri.stream : nullptr;
    // a conventional request has no queue (proc_enqueue.cpp:124-126, Appendix A6)
    if (ri.conventional) return MPIX_ERR_STREAM_MISMATCH;
    if (i == 0) {
      s0 = s;
      dev0 = rs.device;
    }
    if (s != s0 || rs.device != dev0) return MPIX_ERR_STREAM_MISMATCH;
    sys |= ri.remote;
  }
  {  // captured requests are waited inside their capture, the others outside
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s0, &cs) != cudaSuccess) return MPIX_ERR_CUDA;
    const bool capturing = cs != cudaStreamCaptureStatusNone;
    if (capturing ? ngraph != n : ngraph != 0) return MPIX_ERR_UNSUPPORTED;
  }
  if (statuses) {
    for (int i = 0; i < n; ++i) {
      auto& ri = info(items[i]);
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
    if (items[k].graph) {
      we[k].flag = rs.d_gdone + nn;
      we[k].gen = kWaitConsume;
    } else {
      we[k].flag = rs.d_done + (nn % kReqSlots);
      we[k].gen = nn / kReqSlots + 1;
    }
  }
  // The wait closes the stream's batch: one launch for the window.
  std::unique_lock<std::mutex> glk;  // MPIX_HOST_EXCLUSION=global
  if (g_world->cfg.excl == 0) glk = std::unique_lock<std::mutex>(g_world->global_mu);
  StreamBatch& b = batch_of(s0, dev0);
  std::lock_guard<std::mutex> lk(b.mu);
  if (flush_locked(b, s0, we.data(), n, sys, rank_of(items[0].rank).d_err) < 0) return MPIX_ERR_CUDA;
  return MPI_SUCCESS;
}

// The status of a completed request (host side, after its stream was
// synchronised): a receive reads the status planes its completion wrote
// (source, tag, stream index, bytes, truncated: deliver, endpoint.cpp:17-24);
// a send reports (me, tag, bytes) as post_send does (proc_p2p.cpp:54-58).
int read_status(RankState& rs, uint64_t n, MPI_Status* st) {
  const auto& ri = rs.reqs[n % kReqSlots];
  st->MPI_ERROR = MPI_SUCCESS;
  if (!ri.is_recv) {
    st->MPI_SOURCE = ri.me;
    st->MPI_TAG = ri.tag;
    st->source_index = -2;
    st->count_bytes = ri.bytes;
    st->truncated = 0;
    return MPI_SUCCESS;
  }
  const uint64_t* w = rs.d_done + (n % kReqSlots);
  uint64_t v[2];
  CK(cudaMemcpy(&v[0], reinterpret_cast<const uint8_t*>(w) + kStatusOff, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&v[1], reinterpret_cast<const uint8_t*>(w) + 2 * kStatusOff, 8, cudaMemcpyDeviceToHost));
  st->count_bytes = v[0] & ~kTruncBit;
  st->truncated = (v[0] & kTruncBit) ? 1 : 0;
  st->MPI_SOURCE = (int)((v[1] >> 40) & 0xffffff);
  st->source_index = (int)((v[1] >> 32) & 0xff) - 2;
  st->MPI_TAG = (int)(uint32_t)v[1];
  return MPI_SUCCESS;
}

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
    bool graph = false;
    if (!decode_ticket(reqs[i], &items[i].rank, &items[i].n, &graph)) return MPIX_ERR_INVALID_REQUEST;
    if (graph) return MPIX_ERR_UNSUPPORTED;  // a captured request is waited in its graph
    auto& ri = rank_of(items[i].rank).reqs[items[i].n % kReqSlots];
    if (ri.gen != items[i].n / kReqSlots + 1 || ri.consumed) return MPIX_ERR_INVALID_REQUEST;
    if (int h = rank_health(rank_of(items[i].rank))) return h;
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
      // the global regime's lock covers the launch, not the synchronisation
      // below (another thread's send may be what this wait needs)
      std::unique_lock<std::mutex> glk;
      if (g_world->cfg.excl == 0) glk = std::unique_lock<std::mutex>(g_world->global_mu);
      std::lock_guard<std::mutex> lk(b.mu);
      if (flush_locked(b, s, we.data(), (int)we.size(), sys, rs0.d_err) < 0) return MPIX_ERR_CUDA;
    }
    CK(cudaStreamSynchronize(s));
  }
  // a watchdog expiry while waiting: the requests did not complete
  for (int i = 0; i < n; ++i)
    if (int h = rank_health(rank_of(items[i].rank))) return h;
  for (int i = 0; i < n; ++i) {
    RankState& rs = rank_of(items[i].rank);
    auto& ri = rs.reqs[items[i].n % kReqSlots];
    ri.consumed = true;
    if (statuses) {
      CK(cudaSetDevice(rs.device));
      if (int rc = read_status(rs, items[i].n, &statuses[i])) return rc;
    }
    reqs[i] = MPI_REQUEST_NULL;
  }
  return MPI_SUCCESS;
}

// Blocking conventional / multiplex operation: post as a blocking device
// operation (eager or staged send, waiting receive), then synchronise and
// report the operation's status (its ticket).
int host_blocking(int rc, mpix_comm_s* c, cudaStream_t s, MPI_Status* status, uint64_t ticket) {
  if (rc) return rc;
  RankState& rs = rank_of(c->rank);
  CK(cudaSetDevice(rs.device));
  CK(cudaStreamSynchronize(s));
  if (int h = rank_health(rs)) return h;
  int r = 0;
  uint64_t n = 0;
  if (ticket && decode_ticket(ticket, &r, &n)) {
    rs.reqs[n % kReqSlots].consumed = true;
    if (status) return read_status(rs, n, status);
  } else if (status) {  // a blocking send carries no completion word
    status->MPI_SOURCE = c->rank;
    status->MPI_TAG = -1;
    status->MPI_ERROR = MPI_SUCCESS;
    status->source_index = -2;
    status->count_bytes = UINT64_MAX;
    status->truncated = 0;
  }
  return MPI_SUCCESS;
}

}  // namespace mpix

using namespace mpix;

extern "C" {

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
  return rc ? rc : host_blocking(rc, comm, conv_stream(comm), nullptr, 0);
}

int MPI_Recv(void* buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
             MPI_Status* status) {
  uint64_t t = 0;
  int rc = conv_post(comm, buf, count, datatype, source, tag, true, true, nullptr, &t);
  return rc ? rc : host_blocking(rc, comm, conv_stream(comm), status, t);
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
  return rc ? rc : host_blocking(rc, comm, local_stream_of(comm, src_idx), nullptr, 0);
}

int MPIX_Stream_recv(void* buf, int count, MPI_Datatype datatype, int source, int tag,
                     MPI_Comm comm, int src_idx, int dst_idx, MPI_Status* status) {
  uint64_t t = 0;
  int rc = stream_post(comm, buf, count, datatype, source, tag, src_idx, dst_idx, true, true,
                       nullptr, &t);
  return rc ? rc : host_blocking(rc, comm, local_stream_of(comm, dst_idx), status, t);
}

int MPIX_Request_free(MPI_Request* request) {
  if (!request) return MPIX_ERR_INVALID_REQUEST;
  *request = MPI_REQUEST_NULL;
  return MPI_SUCCESS;
}

}  // extern "C"
