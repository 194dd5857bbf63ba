/*
 * forestcoll.h — C ABI of the B200-native ForestColl schedule executor.
 *
 * The reference (`collsched` 0.1.0, /root/reference/pkg) ships a schedule
 * *generator* and no executor: runtime execution is a stated non-goal
 * (the hardware criterion is a bare pytest.skip at
 * pkg/tests/test_acceptance.py:159-163).  Its public boundary for this path is
 * the `Schedule` forest (pkg/src/collsched/schedule.py:31-81) and its JSON wire
 * format (schedule.py:348-448), produced by `generate()` (pipeline.py:43-78).
 * This library is the additive executor behind that boundary.  Entry points
 * are NCCL-shaped so a binding (ctypes / cffi) can call
 * them exactly where the reference's users would call a collective.
 *
 * Each entry point below names the reference interface it consumes/replaces:
 *
 *  fc_comm_init / fc_comm_export / fc_comm_connect
 *      one communicator per rank process; the reference has no runtime
 *      (SPEC.md:8).  Peer workspaces (flags + reduction scratch) are mapped
 *      over NVLink with CUDA IPC handles exchanged by the caller.
 *  fc_comm_init_virtual
 *      all N ranks of one forest on a single device (one cooperative grid),
 *      the single-GPU test mode of SURVEY.md §4.
 *  fc_plan_load
 *      consumes the lowered `Schedule` forest (schedule.py:31-81; lowering by
 *      paper_2402_06787_b200/compiler.py): one table per collective —
 *      allgather (schedule.py:88-129), reduce_scatter
 *      (reverse_for_reduce_scatter, schedule.py:166-174), allreduce
 *      (combine_allreduce, schedule.py:177-211).
 *  fc_allgather / fc_reduce_scatter / fc_allreduce (+ _multi variants)
 *      execute the forest: "a 1/k shard of data is broadcast along each
 *      out-tree"; RS/AR per PAPER.md:1036.
 *  fc_buffer_export / fc_buffer_register
 *      zero-copy peer mapping of caller-owned output buffers.
 *  fc_last_error / fc_comm_check
 *      error reporting; the Python wrapper maps codes onto the reference's
 *      CollschedError hierarchy (errors.py:10-140).
 *
 * Conventions: every function returns 0 (FC_SUCCESS) or an FC_ERR_* code;
 * pointers are plain device pointers; `stream` is a cudaStream_t passed as
 * void*; calls are stream-ordered and asynchronous; a communicator is not
 * re-entrant across host threads and all calls on one communicator must be
 * issued in the same order on every rank (NCCL semantics).
 *
 * Ordering: the collectives of one communicator execute one at a time in
 * issue order, also when issued on different streams (a call on a new stream
 * waits for an event recorded on the previous call's stream at issue time).
 * Outside CUDA-graph capture no further synchronisation is needed.
 *
 * Output buffers: only the chunk-flag protocol stores into peers' outputs
 * (allgather recv, allreduce buf; fc_call_path tells which path a call
 * takes).  For it, the allocation holding the output must be registered
 * (fc_buffer_export / fc_buffer_register, collective), and every rank must
 * pass a buffer at the same offset from the buffer it registered, with the
 * same size (SPMD allocation order).  Each launch publishes a tag of its
 * output with its entry epoch; a mismatch is a device error (FC_ERR_DEVICE
 * from fc_comm_check) rather than misplaced peer stores.  The one-hop,
 * one-shot and LL128 paths write only the library's own staging and accept
 * any device buffers, at any alignment.
 *
 * Workspace: scratch_bytes (fc_comm_init) sizes two regions of that many
 * bytes each: reduce-scatter windows of the chunk-flag protocol, and the
 * LL128 staging (two halves alternating by launch parity).  LL128 and the
 * one-hop paths apply only when their staging fits in half a region.
  */
#ifndef FORESTCOLL_H_
#define FORESTCOLL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_MAX_RANKS 16

/* status codes */
#define FC_SUCCESS 0
#define FC_ERR_INVALID_ARG 1
#define FC_ERR_CUDA 2
#define FC_ERR_UNSUPPORTED 3
#define FC_ERR_NOT_REGISTERED 4
#define FC_ERR_PLAN 5
#define FC_ERR_DEVICE 6 /* device-side failure: flag wait timed out, or peers passed different outputs */

/* collectives (plan slots) */
#define FC_ALLGATHER 0
#define FC_REDUCE_SCATTER 1
#define FC_ALLREDUCE 2

/* dtypes: numbering follows ncclDataType_t */
#define FC_INT8 0
#define FC_UINT8 1
#define FC_INT32 2
#define FC_UINT32 3
#define FC_INT64 4
#define FC_UINT64 5
#define FC_FLOAT16 6
#define FC_FLOAT32 7
#define FC_FLOAT64 8
#define FC_BFLOAT16 9

/* reduction ops: numbering follows ncclRedOp_t (SUM and AVG are implemented).
 * AVG (floating-point dtypes only): the tree root multiplies its fp32 sum by
 * the fp32 value 1/N once, before the final rounding to the buffer dtype. */
#define FC_SUM 0
#define FC_AVG 4

/* options for fc_comm_set_option */
#define FC_OPT_CTAS_PER_RANK 1 /* CTAs per rank (default 128 real, 16 virtual) */
#define FC_OPT_CHUNK_MAX 2     /* max bytes per chunk, flag protocol (default 256 KiB) */
#define FC_OPT_CHUNK_MIN 3     /* min bytes per pipeline chunk (default 16 KiB) */
#define FC_OPT_ITEMS_PER_WORKER 4 /* target work items per CTA (default 4) */
#define FC_OPT_TIMEOUT_MS 5    /* device flag-wait timeout (default 120000 ms, or the
                                  FORESTCOLL_TIMEOUT_MS environment variable at init);
                                  a timed-out wait becomes a sticky FC_ERR_DEVICE */
#define FC_OPT_LAG 6           /* claim-order skew, chunks per tree stage (default 64) */
#define FC_OPT_COPY_MODE 7     /* 0: TMA bulk stores, 1: TMA loads + vector stores (default 1) */
#define FC_OPT_DMA_ROOT_COPY 8 /* allgather: copy engine places the own shard (default 0) */
#define FC_OPT_WORKER_WARPS 9  /* warps per work item: 1, 2, 4, 8 (default 8 real, 1 virtual) */
#define FC_OPT_PROTO 10        /* -1 auto, 0 chunk flags + fences, 1 LL128 lines (default -1) */
#define FC_OPT_LL_MAX 11       /* auto: LL128 when bytes per rank <= this (default 512 MiB) */
#define FC_OPT_LL_CHUNK_MAX 12 /* max bytes per chunk, LL128 protocol (default 64 KiB) */
#define FC_OPT_LL_WORKER_WARPS 13 /* warps per work item, LL128 (default 4 real, 1 virtual) */
#define FC_OPT_NVLS_CTAS 14    /* CTAs of the NVLS (multicast) kernel (default 32) */
#define FC_OPT_PDL 15          /* programmatic dependent launch (default 1) */
#define FC_OPT_CHUNK_TAIL 16   /* chunk flags: last k chunks of a slice halve in size (default 4; 0 virtual) */
#define FC_OPT_NVLS_LL_MAX 17  /* NVLS allgather: LL multicast when output bytes <= this (default max(2 MiB, N x 512 KiB)) */
#define FC_OPT_NVLS_LL_HALF 18 /* read-only: bytes per LL staging half, reserved x2 at the pool top */
#define FC_OPT_NVLS_LL_RED_MAX 19 /* NVLS allreduce: LL multicast + local tree evaluation up to
                                     this many bytes (default N x 64 KiB; reduce-scatter: 1/N) */
#define FC_OPT_ONESHOT_MAX 20  /* tree engine: one-shot allreduce (peer stores + local tree
                                  evaluation) up to this many bytes (default 2 MiB,
                                  reduce-scatter 2/N of it; 0 disables) */
#define FC_OPT_ONESHOT_AG_MAX 21 /* tree engine: one-hop allgather (LL128 lines to every peer)
                                    up to this output size (default 16 MiB; 0 disables) */
#define FC_OPT_MAX_CTAS_PER_RANK 22 /* read-only: largest FC_OPT_CTAS_PER_RANK this
                                       device co-schedules for the comm's local ranks */
#define FC_OPT_CE_MIN 23       /* 2-rank single-switch forest: allgathers whose output is at
                                  least this many bytes move each shard with the copy engine
                                  (one cudaMemcpyAsync into the peer's registered output) and
                                  the SMs only synchronise (default 24 MiB; 0 disables) */
#define FC_OPT_TWOHOP_MAX 25   /* tree engine, single-switch forest: reduce-scatters /
                                  allreduces above the one-shot limit and up to this many
                                  input bytes per rank run in two hops (shards to their
                                  roots, in-tree evaluated there, reduced shards to every
                                  rank; default 6 MiB at N=2, 12 MiB above, reduce-scatter
                                  2/3 of it; 0 disables) */

typedef struct fc_comm fc_comm_t;

const char* fc_version(void);
size_t fc_handle_bytes(void);

int fc_comm_init(int rank, int nranks, int device, size_t scratch_bytes,
                 fc_comm_t** out);
int fc_comm_init_virtual(int nranks, int device, size_t scratch_bytes,
                         fc_comm_t** out);
/* several ranks per process/device (one cooperative grid): fc_comm_export
 * then writes one handle per local rank, and output buffers are registered
 * with the _multi variants (one pointer per local rank). */
int fc_comm_init_ranks(const int* ranks, int nlocal, int nranks, int device,
                       size_t scratch_bytes, fc_comm_t** out);
int fc_comm_export(fc_comm_t* comm, void* handle);
int fc_comm_connect(fc_comm_t* comm, const void* handles);
int fc_comm_set_option(fc_comm_t* comm, int option, long long value);
int fc_comm_get_option(fc_comm_t* comm, int option, long long* value);
int fc_comm_check(fc_comm_t* comm, int* device_error);
int fc_comm_destroy(fc_comm_t* comm);
const char* fc_last_error(const fc_comm_t* comm);

int fc_buffer_export(fc_comm_t* comm, const void* ptr, size_t bytes,
                     void* handle);
int fc_buffer_register(fc_comm_t* comm, const void* ptr, size_t bytes,
                       const void* handles);
int fc_buffer_deregister(fc_comm_t* comm, const void* ptr);
int fc_buffer_export_multi(fc_comm_t* comm, const void* const* ptrs, size_t bytes,
                           void* handles);
int fc_buffer_register_multi(fc_comm_t* comm, const void* const* ptrs,
                             size_t bytes, const void* handles);
/* Registration covers the whole allocation (cudaMalloc segment) holding the
 * buffer, identified by the driver's buffer id; it never pins a buffer.
 * fc_buffer_query: is [ptr, ptr+bytes) inside a live registration?
 * fc_buffer_count: number of live registrations. */
int fc_buffer_query(fc_comm_t* comm, const void* ptr, size_t bytes, int* registered);
int fc_buffer_count(const fc_comm_t* comm);
/* The path the next collective of this size would take: 0 chunk flags,
 * 1 LL128, 4 one-hop / one-shot, 5 copy engine (2-rank allgather), 6 the 1-rank
 * forest's local copy, 7 two-hop reduction, -1 empty.
 * Paths 0 and 5 store into peers' outputs: allgather / allreduce outputs
 * must then be registered.  The
 * choice depends only on values equal on every rank (count, dtype, plan,
 * options), never on buffer addresses. */
int fc_call_path(fc_comm_t* comm, int collective, size_t count, int dtype, int* path);
/* Workspace sizing.  fc_call_scratch: the scratch_bytes (per region, see
 * "Workspace" above) the path this call would take with a workspace of `cap`
 * bytes per region needs -- 0 when it needs none.  fc_comm_grow: re-allocate
 * every local workspace with scratch_bytes per region; collective (all ranks,
 * same value, after all their collectives on this communicator completed),
 * and followed by fc_comm_export / fc_comm_connect.  The Python layer starts
 * small and grows on demand up to a cap (executor.ForestCollComm). */
int fc_call_scratch(fc_comm_t* comm, int collective, size_t count, int dtype, size_t cap,
                    size_t* bytes);
size_t fc_comm_scratch_bytes(const fc_comm_t* comm);
int fc_comm_grow(fc_comm_t* comm, size_t scratch_bytes);

int fc_plan_load(fc_comm_t* comm, int collective, const int32_t* table,
                 size_t nwords);

int fc_allgather(fc_comm_t* comm, const void* send, void* recv,
                 size_t sendcount, int dtype, void* stream);
int fc_reduce_scatter(fc_comm_t* comm, const void* send, void* recv,
                      size_t recvcount, int dtype, int op, void* stream);
int fc_allreduce(fc_comm_t* comm, const void* send, void* recv, size_t count,
                 int dtype, int op, void* stream);

/* one send/recv pointer per local rank (nranks entries for a virtual comm) */
int fc_allgather_multi(fc_comm_t* comm, const void* const* sends,
                       void* const* recvs, size_t sendcount, int dtype,
                       void* stream);
int fc_reduce_scatter_multi(fc_comm_t* comm, const void* const* sends,
                            void* const* recvs, size_t recvcount, int dtype,
                            int op, void* stream);
int fc_allreduce_multi(fc_comm_t* comm, const void* const* sends,
                       void* const* recvs, size_t count, int dtype, int op,
                       void* stream);

/* statistics of the last collective call (launches, chunks, bytes) */
int fc_last_call_info(const fc_comm_t* comm, long long* info, int ninfo);

/* NVLS engine (NVSwitch multicast / in-switch aggregation) for forests whose
 * switch hops are pruned (schedule.py:237-306).  Setup is collective:
 * rank 0 fc_nvls_create -> pass the handle (its int32 at byte offset 4 is a
 * POSIX fd: send it over a unix socket with SCM_RIGHTS and patch in the
 * receiver's fd) -> every rank fc_nvls_attach -> barrier -> every rank
 * fc_nvls_bind (returns the local base of a symmetric pool; buffers passed
 * to fc_nvls_* must lie inside it). */
int fc_nvls_supported(int device);
int fc_nvls_create(fc_comm_t* comm, size_t bytes, void* handle);
int fc_nvls_attach(fc_comm_t* comm, const void* handle);
int fc_nvls_bind(fc_comm_t* comm, void** pool);
/* allgather: small calls (output <= FC_OPT_NVLS_LL_MAX, 8-byte aligned, staging
 * fits) use the LL multicast protocol and accept any device buffers; larger
 * calls need `recv` inside the pool (below the reserved LL staging). */
int fc_nvls_allgather(fc_comm_t* comm, const void* send, void* recv,
                      size_t sendcount, int dtype, void* stream);
int fc_nvls_reduce_scatter(fc_comm_t* comm, const void* send, void* recv,
                           size_t recvcount, int dtype, int op, void* stream);
int fc_nvls_allreduce(fc_comm_t* comm, void* buf, size_t count, int dtype,
                      int op, void* stream);

/* item tracing: 40-byte records {u64 t_start, u64 t_end (ns, %globaltimer),
 * u32 t_wait (ns waiting on flags), u32 t_move (ns moving data), i32 chunk,
 * i16 rank, i16 task, i16 worker, u16 launch, u32 pad} appended at
 * atomicAdd(*count) while *count < capacity; records == NULL disables. */
int fc_comm_set_trace(fc_comm_t* comm, void* records, unsigned int* count,
                      unsigned int capacity);

#ifdef __cplusplus
}
#endif

#endif /* FORESTCOLL_H_ */
