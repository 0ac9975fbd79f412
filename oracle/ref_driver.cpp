// ref_driver.cpp — C ABI over the UNMODIFIED reference library ("streamix",
// /root/reference/proj/src/*.cpp), built by oracle/Makefile into
// oracle/_ref/libstreamix_ref.so. TEST INFRASTRUCTURE ONLY: used to pin the
// C restatement (streamix_oracle.c), to generate tests/golden/ fixtures, and
// as the CPU baseline of bench.py (`cpu_baseline.kind = "reference"`).
//
// Everything below goes through the reference's public API only: World,
// run_ranks, Proc::{stream_create, stream_comm_create, *_enqueue},
// exec_queue_create/enqueue_task/queue_synchronize (world.hpp:35-159,
// exec_queue.hpp:16-80), Info (info.hpp), wire codec (wire.hpp),
// oracle::reference_outcome / run_interleaving_oracle (oracle.hpp).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "streamix/bench.hpp"
#include "streamix/exec_queue.hpp"
#include "streamix/info.hpp"
#include "streamix/oracle.hpp"
#include "streamix/result.hpp"
#include "streamix/wire.hpp"
#include "streamix/world.hpp"

using namespace streamix;

namespace {

struct RankSetup {
  ExecQueue* q = nullptr;
  int stream = 0;
  CommH comm;
};

FabricConfig queue_config(int streams_per_rank) {
  FabricConfig cfg;
  cfg.implicit_pool_size = 1;
  cfg.explicit_pool_size = streams_per_rank;  // types.hpp:54 defaults to 0
  return cfg;
}

// exec_queue + type=exec_queue hint + stream comm per rank.
std::vector<RankSetup> setup_ranks(World& w) {
  std::vector<RankSetup> rs(w.size());
  run_ranks(w, [&](Proc& p) {
    RankSetup& s = rs[p.rank()];
    s.q = exec_queue_create();
    Info info;
    info.set("type", "exec_queue");
    info.set_hex("value", &s.q, sizeof(s.q));
    auto sid = p.stream_create(info);
    if (!sid.ok()) std::abort();
    s.stream = *sid;
    auto c = p.stream_comm_create(p.world_comm(), s.stream);
    if (!c.ok()) std::abort();
    s.comm = *c;
  });
  return rs;
}

void teardown(World& w, std::vector<RankSetup>& rs) {
  for (auto& s : rs) queue_synchronize(s.q);
  run_ranks(w, [&](Proc& p) {
    RankSetup& s = rs[p.rank()];
    p.comm_free(s.comm);
    p.stream_free(s.stream);
  });
  for (auto& s : rs) exec_queue_destroy(s.q);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

uint64_t fnv1a(const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

template <typename T>
T fold(T acc, T x, int op) {
  if (op == 1) return acc + x;
  if (op == 2) return x > acc ? x : acc;
  return x < acc ? x : acc;
}

}  // namespace

extern "C" {

const char* ref_err_name(int code) {
  static thread_local std::string s;
  s = std::string(to_string(static_cast<Err>(code)));
  return s.c_str();
}

void ref_hex_encode(const uint8_t* in, size_t len, char* out) {
  std::string s = hex_encode(in, len);
  std::memcpy(out, s.c_str(), s.size() + 1);
}

int ref_hex_decode(const char* s, uint8_t* out, size_t* outlen) {
  auto r = hex_decode(std::string(s));
  if (!r.ok()) return static_cast<int>(r.error());
  std::memcpy(out, r->data(), r->size());
  *outlen = r->size();
  return 0;
}

// Info::get_hex on a missing key (info.cpp:31-35): NOT_FOUND.
int ref_info_get_hex_missing() {
  Info info;
  auto r = info.get_hex("missing");
  return r.ok() ? 0 : static_cast<int>(r.error());
}

void ref_encode_header(uint32_t ctx, uint32_t src_rank, int32_t src_idx, int32_t dst_idx,
                       int32_t tag, uint64_t seq, uint64_t len, uint8_t out[36]) {
  Envelope e;
  e.context_id = ctx;
  e.src_rank = src_rank;
  e.src_idx = src_idx;
  e.dst_idx = dst_idx;
  e.tag = tag;
  e.seq = seq;
  e.payload_len = len;
  encode_header(e, out);
}

// The 1000-vector generation of proj/tests/test_info.cpp:60-76 (mt19937_64(42),
// len = rng() % 33, bytes = rng()) encoded by the reference.
int ref_hex_random_vectors(uint64_t seed, int n, uint8_t* bytes_out, int* lens_out,
                           char* enc_out) {
  std::mt19937_64 rng(seed);
  for (int i = 0; i < n; ++i) {
    size_t len = rng() % 33;
    std::vector<uint8_t> b(len);
    for (auto& x : b) x = static_cast<uint8_t>(rng());
    Info info;
    info.set_hex("v", b.data(), b.size());
    std::string e = *info.get("v");
    lens_out[i] = static_cast<int>(len);
    std::memcpy(bytes_out + 32 * i, b.data(), len);
    std::memcpy(enc_out + 65 * i, e.c_str(), e.size() + 1);
  }
  return 0;
}

// oracle.cpp:33-74 on one program set + interleaving. ops are (is_send,peer,tag)
// triples, lens per rank; pairs_out[rank*max_pos+pos] = send op id / UINT64_MAX.
void ref_reference_outcome(int n_ranks, const int* ops, const int* lens, const int* order,
                           int n_order, uint64_t* pairs_out, int max_pos) {
  std::vector<std::vector<oracle::Op>> progs(n_ranks);
  int k = 0;
  for (int r = 0; r < n_ranks; ++r)
    for (int i = 0; i < lens[r]; ++i, ++k)
      progs[r].push_back(oracle::Op{ops[3 * k] != 0, ops[3 * k + 1], ops[3 * k + 2]});
  std::vector<int> il(order, order + n_order);
  oracle::Outcome o = oracle::reference_outcome(progs, il);
  for (int i = 0; i < n_ranks * max_pos; ++i) pairs_out[i] = UINT64_MAX;
  for (auto& [rid, sid] : o.pairs) pairs_out[(rid >> 16) * max_pos + (rid & 0xffff)] = sid;
}

void ref_interleaving_oracle(int max_ops, uint64_t* program_pairs, uint64_t* executions,
                             uint64_t* divergences) {
  oracle::Report r = oracle::run_interleaving_oracle(max_ops);
  *program_pairs = r.program_pairs;
  *executions = r.executions;
  *divergences = r.divergences;
}

// Enqueue-path edge semantics. out[i] = Err code of:
//  0 send_enqueue(count=-1, tag=-1)          (A5 enqueue order -> INVALID_TAG)
//  1 isend(count=-1, tag=-1) on world comm    (A5 p2p order     -> INVALID_COUNT)
//  2 waitall_enqueue({})                      (A6 -> OK)
//  3 waitall_enqueue({nullptr})               (A6 -> INVALID_REQUEST)
//  4 waitall_enqueue({conventional irecv})    (A6 -> STREAM_MISMATCH)
//  5 send_enqueue on a multiplex comm         (A12 -> NOT_ENQUEUE_COMM)
//  6 send_enqueue on a serial-context comm    (A7 -> NOT_ENQUEUE_COMM)
//  7 send_enqueue on the world comm           (-> NOT_ENQUEUE_COMM)
//  8 recv_enqueue(ANY_SOURCE, ANY_TAG)        (A4 -> OK, accepted)
//  9 send_enqueue(dest=n)                     (-> INVALID_RANK)
// 10 waitall_enqueue across two queues        (SPEC.md:420 -> STREAM_MISMATCH)
// 11 stream_create(type=bogus)                (-> BAD_HINT)
// 12 stream_create(type=exec_queue, no value) (-> BAD_HINT)
// 13 stream_create(value bad hex)             (-> BAD_HINT)
// 14 stream_create(value wrong length)        (-> BAD_HINT)
// 15 stream_create(endpoint_policy=bogus)     (-> BAD_HINT)
// 16 stream_comm_create_multiple({})          (-> EMPTY_LIST)
// 17 stream_free(in use by a comm)            (-> IN_USE)
// 18 stream_free(STREAM_NULL)                 (-> INVALID_STREAM)
// 19 wait_enqueue twice on one request        (A9 -> OK, second call)
int ref_enqueue_errors(int* out, int n) {
  if (n < 20) return -1;
  World w(2, queue_config(8));
  std::vector<RankSetup> rs = setup_ranks(w);
  Proc& p = w.proc(0);
  RankSetup& s = rs[0];
  int32_t buf[4] = {0, 0, 0, 0};
  int32_t sink[64];
  out[0] = (int)p.send_enqueue(s.comm, buf, -1, Elem::i32, 1, -1).error();
  {
    auto r = p.isend(p.world_comm(), buf, -1, Elem::i32, 1, -1);
    out[1] = r.ok() ? 0 : (int)r.error();
  }
  out[2] = (int)p.waitall_enqueue({}).error();
  out[3] = (int)p.waitall_enqueue({Req{}}).error();
  {
    auto r = p.irecv(p.world_comm(), sink, 4, Elem::i32, 1, 77);
    out[4] = (int)p.waitall_enqueue({*r}).error();
    // satisfy it so teardown does not leave a pending receive
    w.proc(1).send(w.proc(1).world_comm(), buf, 4, Elem::i32, 0, 77);
    p.wait(*r);
  }
  // multiplex + serial-context comms (collective: both ranks)
  std::vector<CommH> mux(2), serial(2);
  std::vector<int> serial_ids(2);
  run_ranks(w, [&](Proc& pr) {
    int r = pr.rank();
    auto m = pr.stream_comm_create_multiple(pr.world_comm(), {rs[r].stream});
    mux[r] = *m;
    serial_ids[r] = *pr.stream_create();
    serial[r] = *pr.stream_comm_create(pr.world_comm(), serial_ids[r]);
  });
  out[5] = (int)p.send_enqueue(mux[0], buf, 1, Elem::i32, 1, 0).error();
  out[6] = (int)p.send_enqueue(serial[0], buf, 1, Elem::i32, 1, 0).error();
  out[7] = (int)p.send_enqueue(p.world_comm(), buf, 1, Elem::i32, 1, 0).error();
  out[8] = (int)p.recv_enqueue(s.comm, sink, 4, Elem::i32, ANY_SOURCE, ANY_TAG).error();
  // satisfy the wildcard receive from rank 1
  w.proc(1).send_enqueue(rs[1].comm, buf, 4, Elem::i32, 0, 5);
  out[9] = (int)p.send_enqueue(s.comm, buf, 1, Elem::i32, 2, 0).error();
  {
    ExecQueue* q2 = exec_queue_create();
    Info info;
    info.set("type", "exec_queue");
    info.set_hex("value", &q2, sizeof(q2));
    int sid2 = *p.stream_create(info);
    std::vector<CommH> c2(2);
    std::vector<ExecQueue*> q1(2, nullptr);
    std::vector<int> sid1(2, 0);
    q1[1] = exec_queue_create();
    run_ranks(w, [&](Proc& pr) {
      int sid = sid2;
      if (pr.rank() == 1) {
        Info i1;
        i1.set("type", "exec_queue");
        i1.set_hex("value", &q1[1], sizeof(q1[1]));
        sid1[1] = *pr.stream_create(i1);
        sid = sid1[1];
      }
      c2[pr.rank()] = *pr.stream_comm_create(pr.world_comm(), sid);
    });
    auto ra = p.irecv_enqueue(s.comm, sink, 4, Elem::i32, 1, 40);
    auto rb = p.irecv_enqueue(c2[0], sink + 8, 4, Elem::i32, 1, 41);
    out[10] = (int)p.waitall_enqueue({*ra, *rb}).error();
    w.proc(1).send_enqueue(rs[1].comm, buf, 4, Elem::i32, 0, 40);
    w.proc(1).send_enqueue(c2[1], buf, 4, Elem::i32, 0, 41);
    p.wait_enqueue(*ra);
    p.wait_enqueue(*rb);
    // A9: wait twice
    auto rc = p.isend_enqueue(s.comm, buf, 1, Elem::i32, 1, 42);
    int e1 = (int)p.wait_enqueue(*rc).error();
    int e2 = (int)p.wait_enqueue(*rc).error();
    out[19] = e1 == 0 && e2 == 0 ? 0 : 1;
    w.proc(1).recv_enqueue(rs[1].comm, sink + 16, 1, Elem::i32, 0, 42);
    queue_synchronize(s.q);
    queue_synchronize(q2);
    queue_synchronize(rs[1].q);
    queue_synchronize(q1[1]);
    run_ranks(w, [&](Proc& pr) { pr.comm_free(c2[pr.rank()]); });
    p.stream_free(sid2);
    w.proc(1).stream_free(sid1[1]);
    exec_queue_destroy(q2);
    exec_queue_destroy(q1[1]);
  }
  {
    Info bogus;
    bogus.set("type", "bogus");
    out[11] = (int)p.stream_create(bogus).error();
    Info novalue;
    novalue.set("type", "exec_queue");
    out[12] = (int)p.stream_create(novalue).error();
    Info badhex;
    badhex.set("type", "exec_queue");
    badhex.set("value", "zz");
    out[13] = (int)p.stream_create(badhex).error();
    Info wronglen;
    wronglen.set("type", "exec_queue");
    uint8_t three[3] = {1, 2, 3};
    wronglen.set_hex("value", three, 3);
    out[14] = (int)p.stream_create(wronglen).error();
    Info badpol;
    badpol.set("endpoint_policy", "bogus");
    out[15] = (int)p.stream_create(badpol).error();
  }
  {
    // EMPTY_LIST is checked before any rendezvous, so one rank suffices.
    out[16] = (int)p.stream_comm_create_multiple(p.world_comm(), {}).error();
  }
  out[17] = (int)p.stream_free(s.stream).error();
  out[18] = (int)p.stream_free(STREAM_NULL).error();
  for (auto& r : rs) queue_synchronize(r.q);
  run_ranks(w, [&](Proc& pr) {
    pr.comm_free(mux[pr.rank()]);
    pr.comm_free(serial[pr.rank()]);
    pr.stream_free(serial_ids[pr.rank()]);
  });
  teardown(w, rs);
  return 0;
}

// cfg1: 2 ranks, Send_enqueue/Recv_enqueue ping-pong of `nbytes`; rank 0
// sends x and receives it back. Returns seconds for `iters` round trips and
// FNV-1a-64 of rank 0's returned buffer and rank 1's received buffer.
double ref_pingpong(const void* x, uint64_t nbytes, int iters, uint64_t* fnv0, uint64_t* fnv1) {
  World w(2, queue_config(1));
  std::vector<RankSetup> rs = setup_ranks(w);
  std::vector<uint8_t> back(nbytes), mid(nbytes);
  double t0 = 0, t1 = 0;
  run_ranks(w, [&](Proc& p) {
    RankSetup& s = rs[p.rank()];
    if (p.rank() == 0) {
      t0 = now_s();
      for (int i = 0; i < iters; ++i) {
        p.send_enqueue(s.comm, x, (int)nbytes, Elem::byte, 1, 0);
        p.recv_enqueue(s.comm, back.data(), (int)nbytes, Elem::byte, 1, 1);
      }
      queue_synchronize(s.q);
      t1 = now_s();
    } else {
      for (int i = 0; i < iters; ++i) {
        p.recv_enqueue(s.comm, mid.data(), (int)nbytes, Elem::byte, 0, 0);
        p.send_enqueue(s.comm, mid.data(), (int)nbytes, Elem::byte, 0, 1);
      }
      queue_synchronize(s.q);
    }
  });
  *fnv0 = fnv1a(back.data(), nbytes);
  *fnv1 = fnv1a(mid.data(), nbytes);
  teardown(w, rs);
  return t1 - t0;
}

// 1-rank loopback on one exec queue (Appendix A1): per iteration
// mode 0: isend+irecv+waitall_enqueue; mode 1: send_enqueue then recv_enqueue.
// Returns seconds for `iters` messages; dst receives the payload.
double ref_selfmsg(const void* src, void* dst, uint64_t nbytes, int iters, int mode) {
  World w(1, queue_config(1));
  std::vector<RankSetup> rs = setup_ranks(w);
  Proc& p = w.proc(0);
  RankSetup& s = rs[0];
  double t0 = now_s();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      auto a = p.isend_enqueue(s.comm, src, (int)nbytes, Elem::byte, 0, 0);
      auto b = p.irecv_enqueue(s.comm, dst, (int)nbytes, Elem::byte, 0, 0);
      p.waitall_enqueue({*a, *b});
    } else {
      p.send_enqueue(s.comm, src, (int)nbytes, Elem::byte, 0, 0);
      p.recv_enqueue(s.comm, dst, (int)nbytes, Elem::byte, 0, 0);
    }
  }
  queue_synchronize(s.q);
  double t = now_s() - t0;
  teardown(w, rs);
  return t;
}

// Composed allreduce: per rank irecv_enqueue from every
// peer, isend_enqueue to every peer, waitall_enqueue, then a queued host task
// folding in rank order 0..P-1. dtype: 1=i32 2=f32 3=f64 4=bf16(u16);
// op: 1=sum 2=max 3=min. in/out: P contiguous arrays of `count` elements.
double ref_allreduce(int P, uint64_t count, int dtype, int op, const void* in, void* out,
                     int iters) {
  const size_t es = dtype == 3 ? 8 : dtype == 4 ? 2 : 4;
  const size_t nbytes = count * es;
  World w(P, queue_config(1));
  std::vector<RankSetup> rs = setup_ranks(w);
  std::vector<std::vector<uint8_t>> tmp(P * P);
  for (auto& t : tmp) t.resize(nbytes);
  const uint8_t* inb = static_cast<const uint8_t*>(in);
  uint8_t* outb = static_cast<uint8_t*>(out);
  double t0 = now_s();
  run_ranks(w, [&](Proc& p) {
    const int r = p.rank();
    RankSetup& s = rs[r];
    for (int it = 0; it < iters; ++it) {
      std::vector<Req> reqs;
      for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        reqs.push_back(*p.irecv_enqueue(s.comm, tmp[r * P + q].data(), (int)nbytes, Elem::byte, q, it));
      }
      for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        reqs.push_back(*p.isend_enqueue(s.comm, inb + r * nbytes, (int)nbytes, Elem::byte, q, it));
      }
      p.waitall_enqueue(reqs);
      s.q->enqueue_task([&, r] {
        auto src = [&](int q) -> const uint8_t* { return q == r ? inb + r * nbytes : tmp[r * P + q].data(); };
        uint8_t* o = outb + r * nbytes;
        for (uint64_t i = 0; i < count; ++i) {
          if (dtype == 1) {
            int32_t acc;
            std::memcpy(&acc, src(0) + 4 * i, 4);
            for (int q = 1; q < P; ++q) {
              int32_t x;
              std::memcpy(&x, src(q) + 4 * i, 4);
              acc = op == 1 ? (int32_t)((uint32_t)acc + (uint32_t)x) : fold(acc, x, op);
            }
            std::memcpy(o + 4 * i, &acc, 4);
          } else if (dtype == 2 || dtype == 4) {
            auto ld = [&](const uint8_t* b) {
              float f;
              if (dtype == 2) {
                std::memcpy(&f, b + 4 * i, 4);
              } else {
                uint16_t h;
                std::memcpy(&h, b + 2 * i, 2);
                uint32_t u = (uint32_t)h << 16;
                std::memcpy(&f, &u, 4);
              }
              return f;
            };
            volatile float acc = ld(src(0));
            for (int q = 1; q < P; ++q) acc = fold<float>(acc, ld(src(q)), op);
            if (dtype == 2) {
              float a = acc;
              std::memcpy(o + 4 * i, &a, 4);
            } else {
              float a = acc;
              uint32_t u;
              std::memcpy(&u, &a, 4);
              u += 0x7fffu + ((u >> 16) & 1u);
              uint16_t h = (uint16_t)(u >> 16);
              std::memcpy(o + 2 * i, &h, 2);
            }
          } else {
            volatile double acc;
            double x;
            std::memcpy(&x, src(0) + 8 * i, 8);
            acc = x;
            for (int q = 1; q < P; ++q) {
              std::memcpy(&x, src(q) + 8 * i, 8);
              acc = fold<double>(acc, x, op);
            }
            double a = acc;
            std::memcpy(o + 8 * i, &a, 8);
          }
        }
      });
    }
    queue_synchronize(s.q);
  });
  double t = now_s() - t0;
  teardown(w, rs);
  return t;
}

// cfg4 analog: P ranks x S exec-queue stream comms, stream k of rank r
// exchanges 8-B messages with stream k of ranks r+-1 (ring), window W,
// waitall per batch. Returns seconds for `batches` batches.
double ref_msgrate(int P, int S, int W, int batches, uint64_t* messages) {
  World w(P, queue_config(S));
  struct St {
    std::vector<ExecQueue*> q;
    std::vector<int> sid;
    std::vector<CommH> c;
  };
  std::vector<St> st(P);
  run_ranks(w, [&](Proc& p) {
    St& s = st[p.rank()];
    for (int k = 0; k < S; ++k) {
      ExecQueue* q = exec_queue_create();
      Info info;
      info.set("type", "exec_queue");
      info.set_hex("value", &q, sizeof(q));
      s.q.push_back(q);
      s.sid.push_back(*p.stream_create(info));
    }
    for (int k = 0; k < S; ++k) s.c.push_back(*p.stream_comm_create(p.world_comm(), s.sid[k]));
  });
  std::vector<uint64_t> sbuf(P * S * 2, 1), rbuf(P * S * 2 * W);
  double t0 = now_s();
  run_ranks(w, [&](Proc& p) {
    const int r = p.rank();
    St& s = st[r];
    const int right = (r + 1) % P, left = (r + P - 1) % P;
    for (int b = 0; b < batches; ++b) {
      for (int k = 0; k < S; ++k) {
        std::vector<Req> reqs;
        for (int i = 0; i < W; ++i) {
          reqs.push_back(*p.irecv_enqueue(s.c[k], &rbuf[((r * S + k) * 2 + 0) * W + i], 8, Elem::byte, left, i));
          reqs.push_back(*p.isend_enqueue(s.c[k], &sbuf[(r * S + k) * 2], 8, Elem::byte, right, i));
        }
        p.waitall_enqueue(reqs);
      }
    }
    for (auto* q : s.q) queue_synchronize(q);
  });
  double t = now_s() - t0;
  *messages = (uint64_t)P * S * W * batches;
  run_ranks(w, [&](Proc& p) {
    St& s = st[p.rank()];
    for (auto& c : s.c) p.comm_free(c);
    for (int id : s.sid) p.stream_free(id);
  });
  for (auto& s : st)
    for (auto* q : s.q) exec_queue_destroy(q);
  return t;
}

// The reference's own lock-regime message-rate bench (paper Fig. 3,
// proj/src/bench.cpp:118-235), called unmodified: mode 0 global_lock,
// 1 per_vci_implicit, 2 stream_explicit; 8-B messages. Returns elapsed s
// (-1 on failure) and the reference's msgs/s.
double ref_fig3(int mode, int threads, int window, int iters, double* msgs_per_s) {
  streamix::bench::BenchConfig cfg;
  cfg.mode = mode == 0 ? streamix::bench::Mode::global_lock
                       : (mode == 1 ? streamix::bench::Mode::per_vci_implicit
                                    : streamix::bench::Mode::stream_explicit);
  cfg.threads = threads;
  cfg.msg_bytes = 8;
  cfg.window = window;
  cfg.iters = iters;
  cfg.warmup = window;
  auto r = streamix::bench::run_msgrate(cfg);
  if (!r.ok()) return -1.0;
  *msgs_per_s = r->msgs_per_s;
  return r->elapsed_s;
}

}  // extern "C"
