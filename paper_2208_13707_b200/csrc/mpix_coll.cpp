// mpix_coll.cpp — enqueued collectives behind include/mpix.h:
// MPIX_Allreduce_enqueue (new) and Reduce,
// Reduce_scatter_block, Bcast, Allgather, Barrier, all on
// the flag-barriered P2P kernels of mpix_kernels.cu.
#include "mpix_state.h"

namespace mpix {

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

int coll_enqueue(int kind, const void* sbuf, void* rbuf, int count, MPI_Datatype dt, MPI_Op op,
                 int root, mpix_comm_s* c) {
  if (!g_world) return MPIX_ERR_NOT_INITIALIZED;
  if (!c) return MPIX_ERR_INVALID_COMM;
  if (!c->enqueue_ok) return MPIX_ERR_NOT_ENQUEUE_COMM;
  if (int h = rank_health(rank_of(c->rank))) return h;  // sticky watchdog state
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
      if (!rbuf) return MPIX_ERR_INVALID_ARG;
      // In place the input is recvbuf (P blocks) and the result goes to its
      // first block, which rank 0 is still reading: fold into my own block
      // (read by nobody else) and move it to the front after the exit barrier.
      if (sbuf == MPI_IN_PLACE) sbuf = rbuf;
      break;
    case CK_BCAST:
      sbuf = rbuf;  // one buffer: the root's is the source
      break;
    case CK_ALLTOALL:
      // in place, a peer would read my blocks while I overwrite them
      if (!rbuf || !sbuf || sbuf == MPI_IN_PLACE) return MPIX_ERR_INVALID_ARG;
      break;
    case CK_ALLGATHER:
      if (!rbuf) return MPIX_ERR_INVALID_ARG;
      if (sbuf == MPI_IN_PLACE) sbuf = static_cast<uint8_t*>(rbuf) + (uint64_t)me * bytes;
      break;
    default:
      break;
  }
  RankState& rs = rank_of(me);
  // Multi-process mode: peers read send buffers and write receive buffers.
  {
    const uint64_t sb_bytes = (kind == CK_REDUCE_SCATTER || kind == CK_ALLTOALL) ? bytes * P : bytes;
    const uint64_t rb_bytes = (kind == CK_ALLGATHER || kind == CK_ALLTOALL) ? bytes * P : bytes;
    if ((sbuf && !peer_ok(sbuf, sb_bytes)) || (rbuf && !peer_ok(rbuf, rb_bytes)))
      return MPIX_ERR_INVALID_ARG;
  }

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
  // two-shot moves fewer bytes than one-shot for every P > 1 (per rank: 2S/P·(P-1) peer
  // traffic + 2S/P local vs (P-1)·S peer + 2S local), so one-shot only where latency rules
  a.algo = bytes <= g_world->cfg.oneshot_max ? AR_ONESHOT : AR_TWOSHOT;
  a.chunk_bytes = bytes;  // ALLGATHER: per rank; REDUCE_SCATTER: my block; BCAST: the buffer
  const bool rsb_in_place = kind == CK_REDUCE_SCATTER && sbuf == rbuf;
  if (rsb_in_place) a.rbuf = static_cast<uint8_t*>(rbuf) + (uint64_t)me * bytes;
  const RegionLayout& L = sh.L;
  for (int q = 0; q < P; ++q) {
    a.peer_in[q] = reinterpret_cast<CollSlot*>(sh.base[q] + L.coll_in(me));
    a.peer_exit[q] = reinterpret_cast<uint64_t*>(sh.base[q] + L.coll_exit(me));
  }
  a.my_in = reinterpret_cast<CollSlot*>(sh.base[me] + L.coll_in(0));
  a.my_exit = reinterpret_cast<uint64_t*>(sh.base[me] + L.coll_exit(0));
  a.err_word = rs.d_err;
  a.spin_limit_ns = g_world->cfg.spin_limit_ns;
  // CUDA-Graph capture: only graph-capturable comms (device epoch counter,
  // a decision record of its own); elsewhere the epoch would repeat on replay
  bool capturing = false;
  {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c->cu, &cs) != cudaSuccess) return MPIX_ERR_CUDA;
    capturing = cs != cudaStreamCaptureStatusNone;
    if (capturing && !c->graph) return MPIX_ERR_UNSUPPORTED;
  }
  if (c->graph) {
    a.gseq = c->d_gseq + 2 * P;
    const bool fused = kind == CK_ALLREDUCE && bytes <= g_world->cfg.oneshot_max;
    a.gbump = (fused || P > 1) ? GB_EXIT : GB_ENTRY;  // the chain's last epoch reader
  }
  if (capturing) {
    uint64_t k = rs.grec_next.fetch_add(1);
    if (k >= kGraphRecs) return MPIX_ERR_NO_MEM;
    a.rec = rs.d_grec + k;
    a.opid = k;
  } else {
    uint64_t opid = rs.op_next.fetch_add(1);
    a.rec = rs.d_rec + (opid % kOpRecords);
    a.opid = opid;
  }
  bool sys = g_world->cfg.force_sys;
  for (int q = 0; q < P; ++q) sys |= rank_of(q).device != rs.device;
  // every member waits for every other one: members sharing my GPU must be
  // able to run concurrently (fail now instead of at the watchdog)
  if (!rs.coresident && !g_world->mp)
    for (int q = 0; q < P; ++q)
      if (q != me && rank_of(q).device == rs.device) return MPIX_ERR_NOT_CORESIDENT;
  CK(cudaSetDevice(rs.device));
  if (!c->batch) c->batch = &batch_of(c->cu, rs.device);
  StreamBatch& b = *c->batch;
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
    else if (kind == CK_ALLGATHER || kind == CK_ALLTOALL)
      grid = (uint64_t)P * p2p_copy_grid(bytes);
    nk = launch_collective(a, sys, grid, c->cu);
    if (nk >= 0 && rsb_in_place && me != 0 && bytes) {
      if (cudaMemcpyAsync(rbuf, a.rbuf, bytes, cudaMemcpyDeviceToDevice, c->cu) != cudaSuccess)
        return MPIX_ERR_CUDA;
    }
  }
  if (nk < 0) return MPIX_ERR_CUDA;
  g_launches.fetch_add(nk);
  return MPI_SUCCESS;
}

}  // namespace mpix

using namespace mpix;

extern "C" {

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

int MPIX_Alltoall_enqueue(const void* sendbuf, int sendcount, MPI_Datatype sendtype, void* recvbuf,
                          int recvcount, MPI_Datatype recvtype, MPI_Comm comm) {
  if ((uint64_t)sendcount * type_size(sendtype) != (uint64_t)recvcount * type_size(recvtype))
    return MPIX_ERR_INVALID_COUNT;
  return coll_enqueue(CK_ALLTOALL, sendbuf, recvbuf, recvcount, recvtype, MPI_SUM, 0, comm);
}

int MPIX_Barrier_enqueue(MPI_Comm comm) {
  return coll_enqueue(CK_BARRIER, nullptr, nullptr, 0, MPI_BYTE, MPI_SUM, 0, comm);
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

}  // extern "C"
