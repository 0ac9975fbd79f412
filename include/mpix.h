/*
 * mpix.h — C ABI of the B200-native MPIX-stream GPU-enqueue path
 * (arXiv 2208.13707, "MPIX Stream: An Explicit Solution to Hybrid MPI+X
 * Programming").
 *
 * This is the drop-in boundary. The reference (`/root/reference/proj`,
 * "streamix") exposes the same operations as C++ methods on
 * `streamix::Proc` (proj/include/streamix/world.hpp:35-92) returning
 * `Result<T>` (proj/include/streamix/result.hpp:39-81). The paper gives the C
 * signatures this header follows.
 * Each declaration below cites the reference entry point it replaces.
 *
 * Plain C types only: no torch, no C++ in the signatures. Buffers are device
 * pointers (any allocation visible to the rank's GPU through UVA; peer GPUs
 * reach them over NVLink after MPIX_World_init enabled peer access).
 *
 * Rank model: one process hosts a world of N ranks, rank r bound to one GPU
 * (several ranks may share a GPU). This mirrors the reference's
 * `World(n)` + `run_ranks` (world.hpp:129-159): collective calls
 * (communicator creation/free, barrier) are made once per member, normally
 * from one host thread per rank. Every MPI_Comm handle is one rank's view of
 * a communicator, so point-to-point and enqueue calls need no thread-bound
 * rank.
 */
#ifndef MPIX_H
#define MPIX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Handles                                                                   */
/* ------------------------------------------------------------------------ */

typedef struct mpix_info_s *MPI_Info;     /* streamix::Info   info.hpp:16-31   */
typedef struct mpix_stream_s *MPIX_Stream; /* streamix::Stream stream.hpp:15-24 */
typedef struct mpix_comm_s *MPI_Comm;     /* streamix::CommH  comm.hpp:38-41   */
/* streamix::Req (request.hpp:52). Opaque 64-bit ticket; 0 = MPI_REQUEST_NULL. */
typedef uint64_t MPI_Request;
typedef int MPI_Datatype;
typedef int MPI_Op;

/* streamix::Status (request.hpp:13-19). Enqueue calls never surface a status
 * in the reference (proc_enqueue.cpp:61,130-137); see MPIX_Wait_enqueue. */
typedef struct {
  int MPI_SOURCE;
  int MPI_TAG;
  int MPI_ERROR;
  int source_index;
  uint64_t count_bytes; /* UINT64_MAX when not known on the host */
  int truncated;
} MPI_Status;

#define MPI_INFO_NULL ((MPI_Info)0)
#define MPIX_STREAM_NULL ((MPIX_Stream)0) /* types.hpp:19 STREAM_NULL */
#define MPI_COMM_NULL ((MPI_Comm)0)
#define MPI_REQUEST_NULL ((MPI_Request)0)
#define MPI_STATUS_IGNORE ((MPI_Status *)0)
#define MPI_STATUSES_IGNORE ((MPI_Status *)0)
#define MPI_IN_PLACE ((void *)1)

#define MPI_ANY_SOURCE (-1) /* types.hpp:10 */
#define MPI_ANY_TAG (-1)    /* types.hpp:11 */
#define MPIX_ANY_INDEX (-1) /* types.hpp:12 */

/* Datatypes. BYTE/INT/DOUBLE are the reference's Elem::{byte,i32,f64}
 * (types.hpp:27-31); FLOAT and BFLOAT16 are added for Allreduce. */
#define MPI_BYTE 1
#define MPI_INT 2
#define MPI_DOUBLE 3
#define MPI_FLOAT 4
#define MPIX_BFLOAT16 5

/* Reduction ops for MPIX_Allreduce_enqueue (no reference: SPEC.md:19,443). */
#define MPI_SUM 1
#define MPI_MAX 2
#define MPI_MIN 3

/* ------------------------------------------------------------------------ */
/* Error codes. 0..22 mirror streamix::Err in declaration order             */
/* (result.hpp:9-33); names from MPIX_Error_string match to_string()         */
/* (result.cpp:5-32). 100+ are conditions the simulation cannot have.        */
/* ------------------------------------------------------------------------ */
#define MPI_SUCCESS 0
#define MPIX_ERR_POOL_EXHAUSTED 1
#define MPIX_ERR_NO_EXPLICIT_POOL 2
#define MPIX_ERR_PENDING_OPS 3
#define MPIX_ERR_IN_USE 4
#define MPIX_ERR_BAD_HINT 5
#define MPIX_ERR_INVALID_STREAM 6
#define MPIX_ERR_INVALID_COMM 7
#define MPIX_ERR_INVALID_RANK 8
#define MPIX_ERR_INVALID_COUNT 9
#define MPIX_ERR_INVALID_TAG 10
#define MPIX_ERR_INVALID_REQUEST 11
#define MPIX_ERR_INVALID_INDEX 12
#define MPIX_ERR_MULTIPLEX_COMM 13
#define MPIX_ERR_NOT_MULTIPLEX 14
#define MPIX_ERR_WILDCARD_DST 15
#define MPIX_ERR_EMPTY_LIST 16
#define MPIX_ERR_NOT_ENQUEUE_COMM 17
#define MPIX_ERR_STREAM_MISMATCH 18
#define MPIX_ERR_QUEUE_BUSY 19
#define MPIX_ERR_CONFIG_INVALID 20
#define MPIX_ERR_NOT_FOUND 21
#define MPIX_ERR_BAD_ENCODING 22
#define MPIX_ERR_CUDA 100          /* a CUDA runtime call failed            */
#define MPIX_ERR_NOT_INITIALIZED 101
#define MPIX_ERR_UNSUPPORTED 102   /* documented v1 divergence  */
#define MPIX_ERR_INVALID_ARG 103
#define MPIX_ERR_TYPE 104          /* unknown datatype                      */
#define MPIX_ERR_OP 105            /* unknown / unsupported reduction op    */
#define MPIX_ERR_NO_MEM 106
/* A device-side watchdog (MPIX_SPIN_TIMEOUT_MS) expired in one of the rank's
 * kernels: a flag wait never saw its peer. The rank's communication state is
 * undefined from then on, so the condition is STICKY: every later call that
 * names the rank (enqueue, conventional p2p, waits, collectives,
 * MPIX_Comm_check) returns it. The reference reports every failure through
 * Result<Err> (result.hpp:36-45); an unbounded spin has no Err there, so the
 * code is new. */
#define MPIX_ERR_TIMEOUT 107
/* A device-side protocol check failed (a descriptor another agent must not
 * have taken was taken). Sticky like MPIX_ERR_TIMEOUT. */
#define MPIX_ERR_DEVICE 108
/* A collective among ranks that share a GPU was enqueued while kernels of
 * different streams of that GPU cannot run concurrently (kernel
 * serialisation by a profiler or sanitizer; probed at MPIX_World_init, see
 * MPIX_Device_coresident). Every rank's barrier would wait for a kernel that
 * can only start after it, so the call fails at once instead of hanging until
 * the watchdog. Not sticky. */
#define MPIX_ERR_NOT_CORESIDENT 109

/* Name of an error code, e.g. "NOT_ENQUEUE_COMM" (result.cpp:5-32). */
const char *MPIX_Error_string(int code);

/* ------------------------------------------------------------------------ */
/* World bootstrap — replaces streamix::World(n) / run_ranks                 */
/* (world.hpp:129-159, world.cpp:53-84). Not part of the paper's API: in    */
/* MPI this is MPI_Init; here one process owns all ranks.                    */
/* ------------------------------------------------------------------------ */

/* Create the world: rank r runs on GPU devices[r] (devices may be NULL:
 * rank r -> device r % device_count). Enables peer access between every
 * pair of distinct devices. */
int MPIX_World_init(int nranks, const int *devices);
/* Destroy the world and every communicator. Caller synchronises its streams
 * first. */
int MPIX_World_finalize(void);
int MPIX_World_size(int *nranks);
/* Rank r's view of the bootstrap world communicator (ctx 0) —
 * Proc::world_comm() (world.hpp:40). */
int MPIX_World_comm(int rank, MPI_Comm *comm);
/* Bind the calling host thread to a rank (optional; lets single-rank-per-
 * thread code call MPIX_Comm_world_self). */
int MPIX_Rank_bind(int rank);
int MPIX_Comm_world_self(MPI_Comm *comm);

int MPI_Comm_rank(MPI_Comm comm, int *rank);
int MPI_Comm_size(MPI_Comm comm, int *size);
/* Collective. Proc::barrier (proc_comm.cpp:31-46). Host-side barrier. */
int MPI_Barrier(MPI_Comm comm);
/* Collective. Proc::comm_free (proc_comm.cpp:178-194). Sets *comm to
 * MPI_COMM_NULL. The world communicator cannot be freed (INVALID_COMM). */
int MPI_Comm_free(MPI_Comm *comm);

/* ------------------------------------------------------------------------ */
/* Info hints — streamix::Info (info.hpp:16-31, info.cpp:17-59)             */
/* ------------------------------------------------------------------------ */
int MPI_Info_create(MPI_Info *info);
int MPI_Info_free(MPI_Info *info);
int MPI_Info_set(MPI_Info info, const char *key, const char *value);
/* Copies the value (NUL-terminated) into value[0..valuelen); *flag = 0 when
 * the key is absent. */
int MPI_Info_get(MPI_Info info, const char *key, int valuelen, char *value,
                 int *flag);
/* PAPER.md:333. Lowercase hex, high nibble first (info.cpp:37-46). */
int MPIX_Info_set_hex(MPI_Info info, const char *key, const void *value,
                      int vallen);
/* Info::get_hex (info.cpp:31-35, 48-59): NOT_FOUND / BAD_ENCODING.
 * *outlen receives the decoded length; at most maxlen bytes are written. */
int MPIX_Info_get_hex(MPI_Info info, const char *key, void *value, int maxlen,
                      int *outlen);

/* ------------------------------------------------------------------------ */
/* Streams — Proc::stream_create / stream_free (proc_stream.cpp:7-60)       */
/* ------------------------------------------------------------------------ */

/* PAPER.md:310. info == MPI_INFO_NULL (or no "type" key): a serial-context
 * (host thread) stream. info{type="cudaStream_t", value=hex(cudaStream_t)}:
 * a GPU stream; the value must decode to exactly sizeof(cudaStream_t) bytes
 * and name a live CUDA stream, else BAD_HINT (proc_stream.cpp:12-17). The
 * optional key "endpoint_policy" accepts "shared"/"exclusive", anything else
 * is BAD_HINT (proc_stream.cpp:27-33). */
int MPIX_Stream_create(MPI_Info info, MPIX_Stream *stream);
/* IN_USE while a communicator references the stream; INVALID_STREAM for
 * MPIX_STREAM_NULL. Sets *stream to MPIX_STREAM_NULL on success. */
int MPIX_Stream_free(MPIX_Stream *stream);
/* The cudaStream_t a GPU stream wraps (NULL for serial-context streams). */
int MPIX_Stream_get_cuda(MPIX_Stream stream, void **cuda_stream);

/* ------------------------------------------------------------------------ */
/* Communicators — Proc::stream_comm_create(_multiple)                      */
/* (proc_comm.cpp:48-176). Collective over the parent's members.             */
/* ------------------------------------------------------------------------ */

/* PAPER.md:366. stream may be MPIX_STREAM_NULL (a member without a local
 * stream; enqueue on that member gives NOT_ENQUEUE_COMM, A7). For a GPU
 * stream, the CUDA stream's device must be the rank's device
 * (INVALID_STREAM otherwise). */
int MPIX_Stream_comm_create(MPI_Comm parent, MPIX_Stream stream,
                            MPI_Comm *newcomm);
/* PAPER.md:391 (named _multiple at PAPER.md:477). count == 0 gives
 * EMPTY_LIST (proc_comm.cpp:55). Enqueue on a multiplex communicator gives
 * NOT_ENQUEUE_COMM (proc_enqueue.cpp:24). */
int MPIX_Stream_comm_create_multiplex(MPI_Comm parent, int count,
                                      MPIX_Stream streams[], MPI_Comm *newcomm);
int MPIX_Stream_comm_create_multiple(MPI_Comm parent, int count,
                                     MPIX_Stream streams[], MPI_Comm *newcomm);

/* ------------------------------------------------------------------------ */
/* Enqueue operations — Proc::*_enqueue (proc_enqueue.cpp:30-141).          */
/* Each call validates (NOT_ENQUEUE_COMM, then rank -> tag -> count,        */
/* proc_enqueue.cpp:8-28), launches one sm_100a kernel into the comm's CUDA  */
/* stream and returns; it never blocks on the peer.            */
/* Matching is MPI non-overtaking per (comm, source, dest, tag).             */
/* MPI_ANY_SOURCE / MPI_ANY_TAG receives need a dynamic-matching comm        */
/* (MPIX_MATCHING=dynamic or the "mpix_matching" stream hint), else         */
/* UNSUPPORTED. Non-blocking calls are coalesced into the stream's next      */
/* ordering call.                                             */
/* ------------------------------------------------------------------------ */

/* PAPER.md:427. Blocking in the stream: later work in the stream sees the
 * send buffer reusable. Completes without the receiver (eager, like
 * proc_p2p.cpp:60-62): small messages go into the receiver's eager ring,
 * large ones are pushed zero-copy when the receive is already posted and
 * staged in local HBM otherwise. */
int MPIX_Send_enqueue(const void *buf, int count, MPI_Datatype datatype,
                      int dest, int tag, MPI_Comm comm);
/* PAPER.md:428. Blocking in the stream until the message has landed in buf.
 * Delivers min(len, capacity) bytes (endpoint.cpp:17-24). */
int MPIX_Recv_enqueue(void *buf, int count, MPI_Datatype datatype, int source,
                      int tag, MPI_Comm comm, MPI_Status *status);
/* PAPER.md:429-430. Non-blocking in the stream; buffer owned by the
 * runtime until a Wait(all)_enqueue on the same stream. */
int MPIX_Isend_enqueue(const void *buf, int count, MPI_Datatype datatype,
                       int dest, int tag, MPI_Comm comm, MPI_Request *request);
int MPIX_Irecv_enqueue(void *buf, int count, MPI_Datatype datatype, int source,
                       int tag, MPI_Comm comm, MPI_Request *request);
/* PAPER.md:431-432. Waitall: n == 0 is success with nothing enqueued; a
 * MPI_REQUEST_NULL entry is INVALID_REQUEST; requests from different
 * streams are STREAM_MISMATCH (proc_enqueue.cpp:120-126). The request stays
 * valid afterwards (waiting twice is ok/ok, Appendix A9); release it with
 * MPIX_Request_free. Statuses: only source/tag are filled (count_bytes =
 * UINT64_MAX), the reference never surfaces enqueue statuses. */
int MPIX_Wait_enqueue(MPI_Request *request, MPI_Status *status);
int MPIX_Waitall_enqueue(int count, MPI_Request requests[],
                         MPI_Status statuses[]);

/* ------------------------------------------------------------------------ */
/* Conventional (host-thread) p2p on GPU buffers — Proc::isend/irecv/send/  */
/* recv/wait/waitall (proc_p2p.cpp:96-212). Arguments are checked rank ->   */
/* count -> tag (proc_p2p.cpp:9-23); a multiplex comm gives MULTIPLEX_COMM.  */
/* The operation runs at once on the rank's internal CUDA stream with the   */
/* same kernels and rings as the enqueue family, so a conventional send     */
/* matches a peer's Recv_enqueue on the same comm (mixed mode). */
/* MPI_Send is eager (returns once the payload is delivered or staged),     */
/* MPI_Recv returns once the payload has landed. MPI_Wait/Waitall block the */
/* host; a request can be waited once (INVALID_REQUEST after), and passing  */
/* one to MPIX_Wait(all)_enqueue gives STREAM_MISMATCH (Appendix A6).       */
/* ------------------------------------------------------------------------ */
int MPI_Send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm);
int MPI_Recv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
             MPI_Status *status);
int MPI_Isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag, MPI_Comm comm,
              MPI_Request *request);
int MPI_Irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag, MPI_Comm comm,
              MPI_Request *request);
int MPI_Wait(MPI_Request *request, MPI_Status *status);
int MPI_Waitall(int count, MPI_Request requests[], MPI_Status statuses[]);

/* Multiplex stream p2p — PAPER.md:484-487, Proc::stream_isend/irecv
 * (proc_p2p.cpp:115-144). NOT_MULTIPLEX on a single-stream comm; indices
 * are checked like the reference (INVALID_INDEX, WILDCARD_DST for an
 * MPIX_ANY_INDEX destination). The operation runs on the CUDA stream of
 * local stream src_idx (send) / dst_idx (receive), or on the rank's internal
 * stream if that MPIX stream is not a GPU stream; the stream indices are
 * part of the match. MPIX_ANY_INDEX sources need a dynamic-matching comm
 * (UNSUPPORTED on a static one). The blocking forms synchronise that
 * stream. */
int MPIX_Stream_send(const void *buf, int count, MPI_Datatype datatype, int dest, int tag,
                     MPI_Comm comm, int src_idx, int dst_idx);
int MPIX_Stream_recv(void *buf, int count, MPI_Datatype datatype, int source, int tag,
                     MPI_Comm comm, int src_idx, int dst_idx, MPI_Status *status);
int MPIX_Stream_isend(const void *buf, int count, MPI_Datatype datatype, int dest, int tag,
                      MPI_Comm comm, int src_idx, int dst_idx, MPI_Request *request);
int MPIX_Stream_irecv(void *buf, int count, MPI_Datatype datatype, int source, int tag,
                      MPI_Comm comm, int src_idx, int dst_idx, MPI_Request *request);
int MPIX_Request_free(MPI_Request *request);

/* New (absent from the reference): in-stream sum/max/min
 * allreduce over peer memory. sendbuf may be MPI_IN_PLACE. Every element is
 * reduced in rank order 0..P-1 with an fp32 accumulator for bf16 (one final
 * round-to-nearest-even), fp32/fp64 adds in that order, wrapping int32. */
int MPIX_Allreduce_enqueue(const void *sendbuf, void *recvbuf, int count,
                           MPI_Datatype datatype, MPI_Op op, MPI_Comm comm);

/* ------------------------------------------------------------------------ */
/* Symmetric heap for one-process-per-GPU use (csrc/mpix_heap.cpp). Every    */
/* process reserves the same virtual range and maps each rank's slice at     */
/* base + rank * slice, so heap pointers are valid in every process. The     */
/* caller exchanges the POSIX file descriptors (e.g. SCM_RIGHTS over a Unix  */
/* socket): rank 0 creates with base_hint 0, the others pass rank 0's base.  */
/* MPIX_Alloc_mem returns heap memory (cudaMalloc without a heap).           */
/* ------------------------------------------------------------------------ */
/* Multi-process world: this process hosts rank `rank` of `nranks`
 * (devices[q] = rank q's GPU). Collective host steps (communicator creation,
 * barrier, free) call `allgather(in, bytes, out, ctx)`, which must gather
 * `bytes` from every rank into out[rank * bytes] (e.g. torch.distributed over
 * gloo) and return 0. The symmetric heap must already exist and be attached;
 * enqueue receive buffers, Isend buffers and collective buffers must be heap
 * memory (MPIX_Alloc_mem), everything else is unchanged. */
typedef int (*MPIX_Allgather_fn)(const void *in, uint64_t bytes, void *out, void *ctx);
int MPIX_World_init_mp(int rank, int nranks, const int *devices, MPIX_Allgather_fn allgather,
                       void *ctx);
int MPIX_World_local_rank(int *rank);
int MPIX_Heap_create(int rank, int nranks, int device, uint64_t bytes_per_rank, uint64_t base_hint,
                     uint64_t *base_out, uint64_t *slice_out, int *fd_out);
int MPIX_Heap_attach(int peer, int fd);
int MPIX_Heap_contains(const void *ptr, uint64_t bytes);
int MPIX_Heap_destroy(void);
int MPIX_Alloc_mem(uint64_t bytes, void **ptr);
int MPIX_Free_mem(void *ptr);

/* More enqueued collectives ("The enqueue APIs can be
 * extended to collectives"; no reference implementation). Same entry/exit
 * barrier as MPIX_Allreduce_enqueue, same stream-order semantics; folds are
 * rank-ordered (bit-exact with oracle/streamix_oracle.c orc_allreduce_*).
 * Reduce: the result lands in the root's recvbuf; sendbuf may be
 * MPI_IN_PLACE at the root. Reduce_scatter_block: rank r receives the fold
 * of block r (recvcount elements) of every sendbuf; MPI_IN_PLACE takes the
 * P blocks from recvbuf and leaves the result in its first block.
 * Bcast: the root's buffer is copied into every other member's buffer.
 * Allgather: block q of every recvbuf = member q's sendbuf (MPI_IN_PLACE:
 * my block is already in place). Alltoall: block q of member r's sendbuf
 * lands in block r of member q's recvbuf (no MPI_IN_PLACE). Barrier: entry +
 * exit barrier only. */
int MPIX_Reduce_enqueue(const void *sendbuf, void *recvbuf, int count, MPI_Datatype datatype,
                        MPI_Op op, int root, MPI_Comm comm);
int MPIX_Reduce_scatter_block_enqueue(const void *sendbuf, void *recvbuf, int recvcount,
                                      MPI_Datatype datatype, MPI_Op op, MPI_Comm comm);
int MPIX_Bcast_enqueue(void *buffer, int count, MPI_Datatype datatype, int root, MPI_Comm comm);
int MPIX_Allgather_enqueue(const void *sendbuf, int sendcount, MPI_Datatype sendtype,
                           void *recvbuf, int recvcount, MPI_Datatype recvtype, MPI_Comm comm);
int MPIX_Alltoall_enqueue(const void *sendbuf, int sendcount, MPI_Datatype sendtype,
                          void *recvbuf, int recvcount, MPI_Datatype recvtype, MPI_Comm comm);
int MPIX_Barrier_enqueue(MPI_Comm comm);

/* ------------------------------------------------------------------------ */
/* Introspection (tests / bench)                                             */
/* ------------------------------------------------------------------------ */

/* Number of runtime kernels launched so far (all ranks). */
uint64_t MPIX_Launch_count(void);
/* Effective configuration: eager bytes, ring slots, max CTAs per op,
 * one-shot/two-shot crossover bytes. */
int MPIX_Config_get(uint64_t *eager_bytes, int *ring_slots, int *max_ctas,
                    uint64_t *oneshot_max_bytes);
/* Communicator context id (equal on every member, recycled lowest-first,
 * world.cpp:43-51). */
int MPIX_Comm_get_ctx(MPI_Comm comm, uint32_t *ctx);
/* 1 when enqueue calls are accepted on comm (single-stream comm with a GPU
 * stream on this member), else 0. */
int MPIX_Comm_is_enqueue(MPI_Comm comm, int *flag);
/* Datatype width in bytes, or 0 if unknown. */
int MPIX_Type_size(MPI_Datatype datatype);
/* Watchdog word of a rank: 0 = healthy, else the first timeout a kernel
 * recorded (1 slot wait, 2 completion wait, 3 collective barrier, 4 protocol)
 * before exiting instead of hanging. Reading clears nothing. */
int MPIX_Rank_error(int rank, uint64_t *code);
/* Health of this member of comm without blocking: MPI_SUCCESS, or the
 * sticky MPIX_ERR_TIMEOUT / MPIX_ERR_DEVICE once a kernel of the rank hit its
 * watchdog (see MPIX_ERR_TIMEOUT). Work already enqueued is not waited for:
 * synchronise the stream first to check it. */
int MPIX_Comm_check(MPI_Comm comm);
/* 1 in *coresident when two spinning kernels of different streams of
 * `device` run at the same time (probed with two one-thread kernels and a
 * 200 ms bound), else 0 — e.g. under ncu's kernel serialisation. Ranks that
 * share a GPU rely on it for every cross-rank wait. */
int MPIX_Device_coresident(int device, int *coresident);
/* Tracing (MPIX_TRACE=1 at MPIX_World_init): copies up to max_records
 * 128-byte per-operation records (struct TraceRec in csrc/mpix_internal.h:
 * op sequence, kind/mode/decision, bytes, key, clock64 stamps of the
 * handshake phases, globaltimer start/end) of `rank`. Synchronises the
 * rank's device. */
int MPIX_Trace_read(int rank, void *out, int max_records, int *n_records);
/* Debug: this member's peer-mapped region of comm (device pointer) and its
 * size; the layout is RegionLayout in csrc/mpix_internal.h. */
int MPIX_Comm_region(MPI_Comm comm, void **base, uint64_t *bytes);
/* Library build string (arch, version). */
const char *MPIX_Version(void);

#ifdef __cplusplus
}
#endif

#endif /* MPIX_H */
