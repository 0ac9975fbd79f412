// mpix_runtime.cpp — host runtime behind include/mpix.h: world, info,
// streams, communicators and introspection.
//
// Replaces the reference's L1-L3 host layers: World/Proc
// (proj/src/world.cpp), stream lifecycle (proj/src/proc_stream.cpp) and
// communicator rendezvous (proj/src/proc_comm.cpp). The enqueue engine
// (proj/src/proc_enqueue.cpp) and the simulated GPU queue
// (proj/src/exec_queue.cpp) are replaced by mpix_p2p.cpp / mpix_coll.cpp: the
// queue worker thread is gone, every enqueue call validates, assigns
// matching sequence numbers, and launches sm_100a kernels (mpix_kernels.cu)
// into the user's cudaStream_t.
#include <cuda.h>
#include <dlfcn.h>
#include <stdio.h>

#include "mpix_state.h"

namespace mpix {

std::atomic<uint64_t> g_launches{0};
CopyTiming g_copy_timing;

bool mp_mode() { return g_world && g_world->mp; }

static std::mutex g_streams_mu;
static std::unordered_map<void*, int> g_streams;  // handle -> 1 live / 0 destroyed

void stream_registry_note(void* stream, int live) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  g_streams[stream] = live ? 1 : 0;
}

int stream_registry_state(void* stream) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  auto it = g_streams.find(stream);
  return it == g_streams.end() ? -1 : it->second;
}

// CUDA multiplexes streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware queues
// (default 8), read when a device's primary context is created. A stream
// whose head is a spinning wait blocks every later kernel of the streams
// sharing its queue, including the peers it waits for. Raise
// it to 32 while no context exists; warn when a context already does.
static void hw_queue_check() {
  const char* v = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  if (v && atoi(v) >= 32) return;
  // driver entry points through dlopen (the library does not link libcuda)
  int active_any = 0, ndev = 0;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
  if (h) {
    auto init = reinterpret_cast<decltype(&cuInit)>(dlsym(h, "cuInit"));
    auto count = reinterpret_cast<decltype(&cuDeviceGetCount)>(dlsym(h, "cuDeviceGetCount"));
    auto get = reinterpret_cast<decltype(&cuDeviceGet)>(dlsym(h, "cuDeviceGet"));
    auto state = reinterpret_cast<decltype(&cuDevicePrimaryCtxGetState)>(
        dlsym(h, "cuDevicePrimaryCtxGetState"));
    if (init && count && get && state && init(0) == CUDA_SUCCESS && count(&ndev) == CUDA_SUCCESS) {
      for (int d = 0; d < ndev; ++d) {
        CUdevice dev;
        unsigned flags = 0;
        int active = 0;
        if (get(&dev, d) == CUDA_SUCCESS && state(dev, &flags, &active) == CUDA_SUCCESS && active)
          active_any = 1;
      }
    }
  }
  if (!active_any) {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 1);
    return;
  }
  static std::atomic<bool> warned{false};
  if (!warned.exchange(true))
    fprintf(stderr,
            "mpix: warning: a CUDA context already exists with CUDA_DEVICE_MAX_CONNECTIONS=%s "
            "(< 32 hardware queues); more concurrently waiting MPIX streams per GPU than queues "
            "can stall until the watchdog (set it to 32 before the first CUDA call)\n",
            v ? v : "unset (8)");
}

int peer_visible_alloc(void** p, uint64_t bytes) {
  if (mp_mode()) return MPIX_Alloc_mem(bytes, p);
  return cudaMalloc(p, bytes) == cudaSuccess ? MPI_SUCCESS : MPIX_ERR_NO_MEM;
}

std::vector<CollMsg> comm_exchange(CommShared& sh, int me, uint64_t& seq, const CollMsg& m) {
  if (!mp_mode()) return sh.rv.exchange(sh.P, me, seq++, m);
  ++seq;
  struct Wire {
    int64_t i0, i1;
    uint64_t u0, p0;
  };
  Wire in{m.i0, m.i1, m.u0, (uint64_t)m.p0};
  std::vector<Wire> out(sh.P);
  std::vector<CollMsg> v(sh.P);
  if (g_world->ag(&in, sizeof(in), out.data(), g_world->ag_ctx) != 0) return {};
  for (int q = 0; q < sh.P; ++q) {
    v[q].i0 = out[q].i0;
    v[q].i1 = out[q].i1;
    v[q].u0 = out[q].u0;
    v[q].p0 = (void*)out[q].p0;
  }
  return v;
}
std::mutex g_world_mu;
World* g_world = nullptr;
thread_local int t_bound_rank = -1;

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
  {  // peers store into my completion words and status planes (kStatusOff)
    const uint64_t nb = 3 * kDoneWords * sizeof(uint64_t);
    int rc = mp_mode() ? MPIX_Alloc_mem(nb, (void**)&r.d_done)
                       : (cudaMalloc(&r.d_done, nb) == cudaSuccess ? MPI_SUCCESS : MPIX_ERR_NO_MEM);
    if (rc) return rc;
    CK(cudaMemset(r.d_done, 0, nb));
    r.d_gdone = r.d_done + kReqSlots;  // captured requests' words (never reused)
  }
  CK(cudaMalloc(&r.d_rec, kOpRecords * sizeof(OpRecord)));
  CK(cudaMemset(r.d_rec, 0, kOpRecords * sizeof(OpRecord)));
  CK(cudaMalloc(&r.d_grec, kGraphRecs * sizeof(OpRecord)));
  CK(cudaMemset(r.d_grec, 0, kGraphRecs * sizeof(OpRecord)));
  CK(cudaMalloc(&r.d_arrive, kArriveWords * sizeof(uint32_t)));
  CK(cudaMemset(r.d_arrive, 0, kArriveWords * sizeof(uint32_t)));
  r.greqs.resize(kGraphReqs);
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
  if (mp_mode()) {
    // a peer process releases my staging buffers: the flags must be heap
    // memory (host-mapped memory of this process is not visible to it)
    if (MPIX_Alloc_mem(kStageSlots * sizeof(uint64_t), (void**)&r.d_stage)) return MPIX_ERR_NO_MEM;
    CK(cudaMemset(r.d_stage, 0, kStageSlots * sizeof(uint64_t)));
  } else {
    CK(cudaHostGetDevicePointer(&r.d_stage, r.h_stage, 0));
  }
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
    if (w.mp) {  // peers pull from my arena and release its slots
      if (MPIX_Alloc_mem((uint64_t)w.cfg.stage_slots * w.cfg.stage_chunk, (void**)&r.d_arena) ||
          MPIX_Alloc_mem((uint64_t)w.cfg.stage_slots * 8, (void**)&r.d_arena_state))
        return MPIX_ERR_NO_MEM;
    } else {
      CK(cudaMallocFromPoolAsync((void**)&r.d_arena, (uint64_t)w.cfg.stage_slots * w.cfg.stage_chunk,
                                 r.pool, r.aux));
      CK(cudaMallocFromPoolAsync((void**)&r.d_arena_state, (uint64_t)w.cfg.stage_slots * 8, r.pool,
                                 r.aux));
    }
    CK(cudaMemsetAsync(r.d_arena_state, 0, (uint64_t)w.cfg.stage_slots * 8, r.aux));
    CK(cudaStreamSynchronize(r.aux));
  }
  return MPI_SUCCESS;
}

World* world() { return g_world; }

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
  auto v1 = comm_exchange(*par->sh, me, par->rv_seq, m1);
  if ((int)v1.size() != P) return MPIX_ERR_CUDA;
  uint32_t ctx = (uint32_t)v1[0].u0;
  bool dyn = false;
  for (int q = 0; q < P; ++q) dyn |= v1[q].i1 != 0;

  // Shared state is created by the root and handed out in phase 2.
  std::shared_ptr<CommShared> sh;
  if (me == 0 || w.mp) {  // multi-process: every member builds its own copy
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
    if (w.mp) {
      if (MPIX_Alloc_mem(L.total(), (void**)&region)) return MPIX_ERR_NO_MEM;
    } else {
      CK(cudaMallocFromPoolAsync((void**)&region, L.total(), rs.pool, rs.aux));
    }
    CK(cudaMemsetAsync(region, 0, L.total(), rs.aux));
    CK(cudaStreamSynchronize(rs.aux));
  }

  CollMsg m2;
  m2.p0 = region;
  if (me == 0) m2.sp = sh;
  auto v2 = comm_exchange(*par->sh, me, par->rv_seq, m2);
  if ((int)v2.size() != P) return MPIX_ERR_CUDA;
  if (!w.mp) sh = std::static_pointer_cast<CommShared>(v2[0].sp);
  {
    // every member writes the same values; guard with the rank mutex of root
    std::lock_guard<std::mutex> lk(rank_of(w.mp ? me : 0).mu);
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
  if ((int)comm_exchange(*par->sh, me, par->rv_seq, CollMsg{}).size() != P) return MPIX_ERR_CUDA;

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
  c->serial_ctx = !multiplex && streams.size() == 1 && streams[0];
  c->send_pseq.assign(P, 0);
  c->recv_pseq.assign(P, 0);
  // graph-capturable: this rank's choice alone (the device counters count
  // exactly what the host counters would), static matching only
  {
    int g = w.cfg.graph ? 1 : 0;
    for (auto* s : streams)
      if (s && s->graph >= 0) g = s->graph;
    c->graph = g && c->enqueue_ok && !sh->dyn;
    c->d_gseq = reinterpret_cast<uint64_t*>(region + L.gseq());
  }
  for (int q = 0; q < P; ++q) c->any_remote |= rank_of(q).device != rs.device;
  {
    std::lock_guard<std::mutex> lk(w.comms_mu);
    w.all_comms.push_back(c);
  }
  *out = c;
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
    case MPIX_ERR_TIMEOUT: return "TIMEOUT";
    case MPIX_ERR_DEVICE: return "DEVICE_PROTOCOL";
    case MPIX_ERR_NOT_CORESIDENT: return "NOT_CORESIDENT";
    default: return "UNKNOWN";
  }
}

// --------------------------------------------------------------------------
// World
// --------------------------------------------------------------------------
// Build the world: all ranks in this process (MPIX_World_init) or only
// rank `w->local` with stubs for the others (MPIX_World_init_mp).
static int world_build(World* w, int nranks, const int* devices, int ndev) {
  w->n = nranks;
  for (int r = 0; r < nranks; ++r) {
    auto rs = std::make_unique<RankState>();
    rs->rank = r;
    rs->device = devices ? devices[r] : r % ndev;
    rs->hosted = !w->mp || r == w->local;
    if (rs->hosted && (rs->device < 0 || rs->device >= ndev)) return MPIX_ERR_INVALID_ARG;
    w->ranks.push_back(std::move(rs));
  }
  for (auto& rs : w->ranks) {
    int per = 0;
    for (auto& o : w->ranks) per += o->device == rs->device;
    rs->per_device = per;
  }
  if (!w->mp) {
    // Peer access between every pair of distinct devices (NVLink / NVSwitch);
    // in multi-process mode the heap mappings grant access instead.
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
  }
  for (auto& rs : w->ranks) {
    if (!rs->hosted) continue;
    int rc = rank_init(*rs, w->cfg);
    if (rc) return rc;
  }
  for (auto& rs : w->ranks) {
    if (!rs->hosted) continue;
    int rc = rank_pool(*w, *rs);
    if (rc) return rc;
  }
  // Ranks of this process sharing a GPU: can their spinning kernels be
  // co-resident? (one probe per device; processes time-slice instead)
  if (!w->mp) {
    std::map<int, int> probed;
    for (auto& rs : w->ranks) {
      if (rs->per_device < 2) continue;
      auto it = probed.find(rs->device);
      if (it == probed.end()) {
        int ok = 0;
        if (coresident_probe(rs->device, &ok) != 0) return MPIX_ERR_CUDA;
        it = probed.emplace(rs->device, ok).first;
      }
      rs->coresident = it->second != 0;
    }
  }
  // Bootstrap world communicator, ctx 0 (world.cpp:61-76). It carries no
  // stream, so enqueue on it is NOT_ENQUEUE_COMM.
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
    if (!rs.hosted) continue;
    if (cudaSetDevice(rs.device) != cudaSuccess) return MPIX_ERR_CUDA;
    uint8_t* region = nullptr;
    if (w->mp) {
      if (MPIX_Alloc_mem(sh->L.total(), (void**)&region)) return MPIX_ERR_NO_MEM;
    } else if (cudaMallocFromPoolAsync((void**)&region, sh->L.total(), rs.pool, rs.aux) != cudaSuccess) {
      return MPIX_ERR_CUDA;
    }
    if (cudaMemsetAsync(region, 0, sh->L.total(), rs.aux) != cudaSuccess) return MPIX_ERR_CUDA;
    sh->base[r] = region;
  }
  if (w->mp) {  // the other ranks' world regions, from their processes
    CollMsg m;
    m.p0 = sh->base[w->local];
    uint64_t seq = 0;
    auto v = comm_exchange(*sh, w->local, seq, m);
    if ((int)v.size() != nranks) return MPIX_ERR_CUDA;
    for (int r = 0; r < nranks; ++r) sh->base[r] = static_cast<uint8_t*>(v[r].p0);
  }
  {
    std::vector<uint64_t> bases(nranks);
    for (int r = 0; r < nranks; ++r) bases[r] = (uint64_t)sh->base[r];
    for (int r = 0; r < nranks; ++r) {
      RankState& rs = *w->ranks[r];
      if (!rs.hosted) continue;
      cudaSetDevice(rs.device);
      if (cudaMemcpyAsync(sh->base[r] + sh->L.bases(), bases.data(), 8ull * nranks,
                          cudaMemcpyHostToDevice, rs.aux) != cudaSuccess ||
          cudaStreamSynchronize(rs.aux) != cudaSuccess)
        return MPIX_ERR_CUDA;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    if (!w->ranks[r]->hosted) {
      w->world_comms.push_back(nullptr);
      continue;
    }
    auto* c = new mpix_comm_s();
    c->sh = sh;
    c->rank = r;
    c->send_pseq.assign(nranks, 0);
    c->recv_pseq.assign(nranks, 0);
    for (int q = 0; q < nranks; ++q) c->any_remote |= w->ranks[q]->device != w->ranks[r]->device;
    c->any_remote |= w->mp && nranks > 1;
    w->world_comms.push_back(c);
  }
  return MPI_SUCCESS;
}

int MPIX_World_init(int nranks, const int* devices) {
  std::lock_guard<std::mutex> lk(g_world_mu);
  if (g_world) return MPIX_ERR_IN_USE;
  if (nranks < 1) return MPIX_ERR_INVALID_ARG;
  hw_queue_check();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return MPIX_ERR_CUDA;
  std::unique_ptr<World> w(new World());
  w->cfg = Config::from_env();
  int rc = world_build(w.get(), nranks, devices, ndev);
  if (rc) return rc;
  g_world = w.release();
  flusher_start(*g_world);
  return MPI_SUCCESS;
}

int MPIX_World_init_mp(int rank, int nranks, const int* devices, MPIX_Allgather_fn allgather,
                       void* ctx) {
  std::lock_guard<std::mutex> lk(g_world_mu);
  if (g_world) return MPIX_ERR_IN_USE;
  if (nranks < 1 || rank < 0 || rank >= nranks || !devices || !allgather) return MPIX_ERR_INVALID_ARG;
  if (nranks > 1 && !heap_live()) return MPIX_ERR_NOT_INITIALIZED;  // MPIX_Heap_create + attach first
  hw_queue_check();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return MPIX_ERR_CUDA;
  std::unique_ptr<World> w(new World());
  w->cfg = Config::from_env();
  w->mp = true;
  w->local = rank;
  w->ag = allgather;
  w->ag_ctx = ctx;
  w->cfg.force_sys = true;  // peers are other processes: system scope everywhere
  // Host staging buffers are not peer-visible: staged blocking sends use the
  // device arena only, so give it larger slots (1 GiB of heap by default).
  if (!std::getenv("MPIX_STAGE_CHUNK")) w->cfg.stage_chunk = 64ull << 20;
  if (!std::getenv("MPIX_STAGE_SLOTS")) w->cfg.stage_slots = 16;
  g_world = w.get();        // comm_exchange during the build reads g_world
  int rc = world_build(w.get(), nranks, devices, ndev);
  if (rc) {
    g_world = nullptr;
    return rc;
  }
  w.release();
  flusher_start(*g_world);
  return MPI_SUCCESS;
}

int MPIX_World_local_rank(int* rank) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!rank) return MPIX_ERR_INVALID_ARG;
  *rank = g_world->mp ? g_world->local : 0;
  return MPI_SUCCESS;
}

int MPIX_World_finalize(void) {
  std::lock_guard<std::mutex> lk(g_world_mu);
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  World* w = g_world;
  flusher_stop(*w);
  std::vector<cudaStream_t> held;
  for (auto& kv : w->batches) held.push_back(kv.first);
  for (cudaStream_t s : held) flush_stream(s);
  for (auto& rs : w->ranks) {
    if (!rs->hosted) continue;
    cudaSetDevice(rs->device);
    cudaDeviceSynchronize();
  }
  // heap memory (multi-process mode) is released with the heap
  for (auto* c : w->all_comms) {
    RankState& rs = *w->ranks[c->rank];
    cudaSetDevice(rs.device);
    if (c->sh && c->sh->base[c->rank] && !w->mp) cudaFreeAsync(c->sh->base[c->rank], rs.aux);
    if (c->sh) c->sh->base[c->rank] = nullptr;
    delete c;
  }
  for (auto* c : w->world_comms) {
    if (!c) continue;
    RankState& rs = *w->ranks[c->rank];
    cudaSetDevice(rs.device);
    if (c->sh->base[c->rank] && !w->mp) cudaFreeAsync(c->sh->base[c->rank], rs.aux);
    c->sh->base[c->rank] = nullptr;
    delete c;
  }
  for (auto& rs : w->ranks) {
    if (!rs->hosted) continue;
    cudaSetDevice(rs->device);
    if (!w->mp)  // multi-process: heap memory, released with the heap
      for (auto& sb : rs->stage) cudaFreeAsync(sb.p, rs->aux);
    if (!w->mp) {
      if (rs->d_arena) cudaFreeAsync(rs->d_arena, rs->aux);
      if (rs->d_arena_state) cudaFreeAsync(rs->d_arena_state, rs->aux);
    }
    cudaStreamSynchronize(rs->aux);
    if (!w->mp) cudaFree(rs->d_done);
    cudaFree(rs->d_rec);
    cudaFree(rs->d_grec);
    cudaFree(rs->d_arrive);
    if (rs->d_trace) cudaFree(rs->d_trace);
    cudaFreeHost(rs->h_err);
    cudaStreamDestroy(rs->aux);
    cudaStreamDestroy(rs->p2p);
    for (cudaStream_t cs : rs->conv_pool) cudaStreamDestroy(cs);
    rs->conv_pool.clear();
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
  if (rank < 0 || rank >= g_world->n || !g_world->world_comms[rank]) return MPIX_ERR_INVALID_RANK;
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
  if ((int)comm_exchange(*comm->sh, comm->rank, comm->rv_seq, CollMsg{}).size() != comm->sh->P)
    return MPIX_ERR_CUDA;
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
  // proc_comm.cpp:182-184: a receive posted on this comm and not yet
  // delivered keeps it alive (checked locally, before the rendezvous).
  // Conventional receives are host-waited, so they are checked here from
  // their completion words; enqueue operations are ordered by the streams.
  {
    std::lock_guard<std::mutex> clk(c->mu);
    for (auto& e : c->conv_recvs) {
      auto& ri = rs.reqs[(uint64_t)(e.first - rs.d_done) % kReqSlots];
      if (ri.consumed || ri.gen != e.second) continue;
      uint64_t v = 0;
      CK(cudaSetDevice(rs.device));
      CK(cudaMemcpy(&v, e.first, 8, cudaMemcpyDeviceToHost));
      if (v < e.second) return MPIX_ERR_PENDING_OPS;
    }
  }
  // Every member's outstanding work on this comm must retire before any
  // region is released: the member's release point follows its enqueue
  // stream and every other stream it launched on (conventional p2p on the
  // rank's internal stream, multiplex p2p on the local streams); members
  // exchange those events and each aux stream waits on all of them.
  cudaEvent_t ev = nullptr;
  if (c->cu && flush_stream(c->cu) < 0) return MPIX_ERR_CUDA;
  for (cudaStream_t s2 : c->side_streams)
    if (flush_stream(s2) < 0) return MPIX_ERR_CUDA;
  CK(cudaSetDevice(rs.device));
  if (w.mp) {
    // events do not cross processes: retire my work, then agree
    CK(cudaStreamSynchronize(c->cu ? c->cu : rs.aux));
    for (cudaStream_t s2 : c->side_streams) CK(cudaStreamSynchronize(s2));
    if ((int)comm_exchange(*c->sh, c->rank, c->rv_seq, CollMsg{}).size() != P) return MPIX_ERR_CUDA;
    c->sh->base[c->rank] = nullptr;  // heap memory is released with the heap
    for (auto* s : c->local_streams)
      if (s) s->refcount.fetch_sub(1);
    {
      std::lock_guard<std::mutex> lk(w.comms_mu);
      w.all_comms.erase(std::remove(w.all_comms.begin(), w.all_comms.end(), c), w.all_comms.end());
    }
    if (c->conv_cu) {
      std::lock_guard<std::mutex> pl(rs.conv_pool_mu);
      rs.conv_pool.push_back(c->conv_cu);
    }
    delete c;
    *comm = MPI_COMM_NULL;
    return MPI_SUCCESS;
  }
  {  // my side streams first: aux follows them, then my enqueue stream
    std::vector<cudaStream_t> mine = c->side_streams;
    if (c->cu) mine.push_back(c->cu);
    for (cudaStream_t s2 : mine) {
      cudaEvent_t e2 = nullptr;
      CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      CK(cudaEventRecord(e2, s2));
      CK(cudaStreamWaitEvent(rs.aux, e2, 0));
      CK(cudaEventDestroy(e2));
    }
  }
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, rs.aux));
  CollMsg m;
  m.p0 = ev;
  auto v = c->sh->rv.exchange(P, c->rank, c->rv_seq++, m);
  if ((int)v.size() != P) return MPIX_ERR_TIMEOUT;  // a member never arrived
  for (int q = 0; q < P; ++q) CK(cudaStreamWaitEvent(rs.aux, (cudaEvent_t)v[q].p0, 0));
  // Nobody destroys an event before all members have enqueued their waits.
  if ((int)c->sh->rv.exchange(P, c->rank, c->rv_seq++, CollMsg{}).size() != P) return MPIX_ERR_TIMEOUT;
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
  if (c->conv_cu) {  // after the region release was ordered behind it
    std::lock_guard<std::mutex> pl(rs.conv_pool_mu);
    rs.conv_pool.push_back(c->conv_cu);
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
      // exec_queue_is_live (proj/src/proc_stream.cpp:17): a stream this
      // library saw destroyed is rejected without touching the handle; a
      // foreign stream is probed (the runtime cannot know its lifetime).
      if (stream_registry_state((void*)cs) == 0) return MPIX_ERR_BAD_HINT;
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
    auto mg = info->entries.find("mpix_graph");  // this library's hint
    if (mg != info->entries.end()) {
      if (mg->second == "1" || mg->second == "true")
        s->graph = 1;
      else if (mg->second == "0" || mg->second == "false")
        s->graph = 0;
      else
        return MPIX_ERR_BAD_HINT;
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

int MPIXT_Set_exclusion(int regime, int* prev) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (regime < 0 || regime > 2) return MPIX_ERR_INVALID_ARG;
  if (prev) *prev = g_world->cfg.excl;
  g_world->cfg.excl = regime;
  return MPI_SUCCESS;
}

int MPIX_Device_coresident(int device, int* coresident) {
  if (!coresident) return MPIX_ERR_INVALID_ARG;
  int ok = 0;
  if (coresident_probe(device, &ok) != 0) return MPIX_ERR_CUDA;
  *coresident = ok;
  return MPI_SUCCESS;
}

int MPIX_Comm_check(MPI_Comm comm) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!comm) return MPIX_ERR_INVALID_COMM;
  return rank_health(rank_of(comm->rank));
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

int MPIXT_Copy_timing(int enable) {
  std::lock_guard<std::mutex> tl(g_copy_timing.mu);
  for (auto& p : g_copy_timing.ev) {
    cudaEventDestroy(p.e0);
    cudaEventDestroy(p.e1);
  }
  g_copy_timing.ev.clear();
  g_copy_timing.on.store(enable != 0);
  return MPI_SUCCESS;
}

int MPIXT_Copy_timing_read(double* total_ms, int* n, uint64_t* bytes) {
  std::lock_guard<std::mutex> tl(g_copy_timing.mu);
  double tot = 0;
  int cnt = 0;
  uint64_t moved = 0;
  for (auto& p : g_copy_timing.ev) {
    if (cudaEventSynchronize(p.e1) != cudaSuccess) return MPIX_ERR_CUDA;
    uint64_t b = 0;
    CK(cudaSetDevice(p.device));
    for (OpRecord* r : p.recs) {  // did this grid copy? (the second arriver's did)
      uint64_t f[5];
      CK(cudaMemcpy(f, &r->action, sizeof(f), cudaMemcpyDeviceToHost));  // action, src, dst, bytes
      if (f[0] == ACT_COPY || f[0] == ACT_STAGE) b += f[3];
    }
    if (!b) continue;
    float ms = 0;
    cudaEventElapsedTime(&ms, p.e0, p.e1);
    tot += ms;
    moved += b;
    ++cnt;
  }
  if (total_ms) *total_ms = tot;
  if (n) *n = cnt;
  if (bytes) *bytes = moved;
  return MPI_SUCCESS;
}

const char* MPIX_Version(void) { return "mpix-b200 0.1 (sm_100a)"; }

}  // extern "C"
