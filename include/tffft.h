/* tffft — transpose-free slab 3D real FFT for NVIDIA B200 (sm_100a).
 *
 * C ABI of the hot path.  Every pointer passed to a transform is a DEVICE
 * pointer on the plan's device; every transform call is asynchronous on the
 * given cudaStream_t (passed as void*, NULL = legacy default stream) and
 * returns an int status.  Status codes map 1:1 onto the reference's
 * exception classes (reference pkg/src/slabfft/errors.py:4-33); the message
 * of the last failure on the calling thread is in tffft_last_error().
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   tffft_plan_create      <- slabfft.dfft.plan            pkg/src/slabfft/dfft.py:93-145
 *   tffft_forward          <- slabfft.dfft.forward         pkg/src/slabfft/dfft.py:148-176
 *   tffft_inverse          <- slabfft.dfft.inverse         pkg/src/slabfft/dfft.py:179-215
 *   tffft_comm_init_local  <- slabfft.transport.make_communicators  transport.py:425-430
 *   tffft_comm_init_rank   <- (MPI communicator; NCCL over NVLink)
 *   tffft_comm_init_all    <- slabfft.transport.run_spmd across GPUs   transport.py:425-468
 *   tffft_comm_init_ipc    <- Endpoint.all_to_all over process-shared memory  transport.py:359-419
 *   tffft_plan_create_batched <- dfft.plan + a batch of fields  dfft.py:93-145
 *   tffft_stage_times      <- FftPlan.timers_us            dfft.py:84-90, 173-175
 *   tffft_counters         <- CopyCounter.snapshot         transport.py:97-114
 *   tffft_consistency      <- FftPlan.last_imag_residue + ConsistencyError  dfft.py:73,211; kernels.py:212-239
 *   tffft_exchange_schedule<- ExchangePlan STRIDED descriptors  exchange.py:106-121
 */
#ifndef TFFFT_H
#define TFFFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py) */
enum {
  TFFFT_OK = 0,
  TFFFT_ERR_SIZE = 1,          /* SizeError          errors.py:8-9   */
  TFFFT_ERR_LAYOUT = 2,        /* LayoutError        errors.py:12-13 */
  TFFFT_ERR_CONFIGURATION = 3, /* ConfigurationError errors.py:16-17 */
  TFFFT_ERR_CONTRACT = 4,      /* ContractError      errors.py:20-21 */
  TFFFT_ERR_PROTOCOL = 5,      /* ProtocolError      errors.py:24-25 */
  TFFFT_ERR_TRANSPORT = 6,     /* TransportError     errors.py:28-29 */
  TFFFT_ERR_CONSISTENCY = 7,   /* ConsistencyError   errors.py:32-33 */
  TFFFT_ERR_CUDA = 8,          /* CUDA runtime failure (SlabFftError) */
  TFFFT_ERR_INTERNAL = 9
};

/* element precision of a plan: real element f64 (complex128) or f32 (complex64) */
enum { TFFFT_F64 = 0, TFFFT_F32 = 1 };

/* exchange pattern (transport.py:51-53) */
enum { TFFFT_PAIRWISE = 0, TFFFT_COLLECTIVE = 1 };

typedef struct tffft_comm_s* tffft_comm_t;
typedef struct tffft_plan_s* tffft_plan_t;
/* host barrier of an IPC communicator: returns 0 once every rank has entered
 * it, non-zero on failure (the plan's call then fails with TFFFT_ERR_TRANSPORT) */
typedef int (*tffft_barrier_fn)(void* ctx);

const char* tffft_last_error(void);
int tffft_version(void);

/* --- communicators ------------------------------------------------------ */
/* NCCL unique id (128 bytes) for tffft_comm_init_rank; call on one rank and broadcast. */
int tffft_get_unique_id(uint8_t out[128]);
/* One process (or thread) per GPU: NCCL communicator over NVLink/NVSwitch. */
int tffft_comm_init_rank(int p, int rank, const uint8_t id[128], int device, tffft_comm_t* comm);
/* p endpoints sharing one in-process fabric on ONE device (the reference's
 * in-process multi-rank fabric, transport.py:188-302).  Each endpoint is
 * driven by its own host thread; forward/inverse are collectives. */
int tffft_comm_init_local(int p, int device, tffft_comm_t* comms);
/* Single process driving p GPUs (ncclCommInitAll over devices[0..p-1], one
 * device per rank): the reference's run_spmd (transport.py:425-468) across
 * GPUs, one host thread per communicator. */
int tffft_comm_init_all(int p, const int* devices, tffft_comm_t* comms);
/* One process per rank, exchange over CUDA IPC: each plan exports its exchange
 * buffers and events (tffft_plan_ipc_export), the caller all-gathers the blobs
 * and every rank attaches the peers' (tffft_plan_ipc_attach).  The exchange is
 * a device pull from the peers' staging (or, with TFFFT_FLAG_PEER_STORES, the
 * producing stage's stores into the peers' landing buffers), ordered by IPC
 * events; `barrier` is the only host-side collective (MPI, a gloo group, ...).
 * Ranks may share a device (several processes on one GPU) or not (P2P).
 * Destroy IPC plans after a host barrier: a peer may still be enqueueing work
 * that references this plan's exported buffers or events until it passes
 * the barrier that ends its last exchange. */
int tffft_comm_init_ipc(int p, int rank, int device, tffft_barrier_fn barrier, void* ctx, tffft_comm_t* comm);
/* host barrier of a local-fabric or IPC communicator (TFFFT_ERR_CONFIGURATION on NCCL) */
int tffft_comm_barrier(tffft_comm_t comm);
/* asynchronous communicator failure (ncclCommGetAsyncError) as TFFFT_ERR_TRANSPORT;
 * TFFFT_OK for a healthy or local communicator (transport.py:209-219 abort propagation) */
int tffft_comm_check(tffft_comm_t comm);
int tffft_comm_rank(tffft_comm_t comm, int* rank);
int tffft_comm_size(tffft_comm_t comm, int* p);
int tffft_comm_device(tffft_comm_t comm, int* device);
/* Abort: wakes every rank blocked in the fabric with TFFFT_ERR_TRANSPORT (transport.py:209-219). */
int tffft_comm_abort(tffft_comm_t comm);
int tffft_comm_destroy(tffft_comm_t comm);

/* --- plans -------------------------------------------------------------- */
/* n0, n1, n2: powers of two in [2, 4096]; p = comm size must divide n0 and n1
 * (layout.py:83-93).  pattern (transport.py:359-419): TFFFT_PAIRWISE = one send
 * and one receive per peer in one NCCL group; TFFFT_COLLECTIVE = one
 * ncclAlltoAll over the p-band staging/landing buffers (grouped send/recv when
 * the loaded NCCL predates 2.28).  Both give bitwise-identical spectra. */
int tffft_plan_create(int n0, int n1, int n2, int dtype, int pattern, tffft_comm_t comm,
                      tffft_plan_t* plan);
/* algorithm flags for tffft_plan_create_ex (0 = the default kernels) */
enum {
  TFFFT_FLAG_FUSED_STAGE1 = 1,   /* one persistent kernel per direction for stage 1 (planes in L2) */
  TFFFT_FLAG_FOURSTEP_STAGE3 = 2, /* stage 3 as an L2-resident four-step with 1 KB row visits */
  TFFFT_FLAG_TRANSPOSE = 4,       /* Strategy.TRANSPOSE (exchange.py:195-260): pack, contiguous exchange,
                                     unpack; the spectrum comes out CONTIGUOUS_FLIPPED, element (j, r, k)
                                     at j*n0*n2c + r*n2c + k (layout.py:42-44) -- the paper's baseline */
  TFFFT_FLAG_PEER_STORES = 8,     /* fused exchange: the stage-1 / stage-3' epilogues store every peer band
                                     straight into the peer's landing buffer (peer memory), and the
                                     exchange reduces to a barrier.  Local fabric communicators. */
  TFFFT_FLAG_CHUNKED_EXCHANGE = 32, /* p > 1 forward: stage 1 in plane chunks, each chunk's part of every band
                                     exchanged (on the plan's exchange stream) while the next chunk computes;
                                     inverse: the bands exchanged plane chunk after plane chunk, stage 1' of a
                                     chunk running as soon as it has landed;
                                     the default on NCCL communicators (TFFFT_XCHUNKS chunks, default 4),
                                     opt-in on the local fabric and IPC */
  TFFFT_FLAG_TMA_COLUMNS = 16     /* column passes of length 512 / 1024 / 2048 fed by TMA box copies: the
                                     warp-per-column kernels (col_wpc.cuh; 2048 points as 2 x 1024 through
                                     tensor memory, col_wpc2.cuh) and col_tma.cuh, any p; the default
                                     (flags < 0) unless TFFFT_TMA_COLS=0 (TFFFT_WPC picks among them);
                                     explicit flags without it select the cp.async column kernel */
};
/* as tffft_plan_create with explicit algorithm flags; flags < 0 = environment defaults */
int tffft_plan_create_ex(int n0, int n1, int n2, int dtype, int pattern, int flags, tffft_comm_t comm,
                         tffft_plan_t* plan);
/* Batched plan (SURVEY.md §8(b) plan_create(..., batch, ...)): every forward /
 * inverse call transforms `batch` fields stored back to back (real slabs of
 * n0/p*n1*n2, spectral slabs of n0/p*n1*(n2/2+1) elements).  p = 1: each stage
 * is ONE launch over all fields; p > 1: a two-deep pipeline in which field c's
 * exchange (on the plan's exchange stream) overlaps field c+1's producing
 * stage.  The inverse's consistency statistics cover every field and are
 * checked once per call (tffft_consistency).  The optional fused-stage-1 and
 * four-step schedules are single-field (dropped when batch > 1). */
int tffft_plan_create_batched(int n0, int n1, int n2, int dtype, int pattern, int flags, int batch,
                              tffft_comm_t comm, tffft_plan_t* plan);
int tffft_plan_batch(tffft_plan_t plan, int* batch);
/* CUDA IPC exchange buffers of NCCL (peer stores) and IPC plans, p > 1.  The
 * blob holds, per buffer set, handles of the staging and landing buffers and
 * (IPC communicators) of the ready / done events.  attach takes p blobs in rank
 * order and is collective. */
int tffft_plan_ipc_blob_bytes(tffft_plan_t plan, size_t* bytes);
int tffft_plan_ipc_export(tffft_plan_t plan, uint8_t* blob);
int tffft_plan_ipc_attach(tffft_plan_t plan, const uint8_t* blobs);
/* Fused exchange on an NCCL communicator (TFFFT_FLAG_PEER_STORES, p > 1): each
 * rank exports a CUDA IPC handle of its landing buffer, the handles are
 * all-gathered by the caller (rank order, 64 bytes each), and attach_peers
 * maps the peers' landing buffers so the stage-1 / stage-3' epilogues store
 * every peer band straight into the peer's memory over NVLink; the exchange is
 * then a one-int ncclAllReduce barrier (exchange.py:263-290 with the strided
 * datatype realised by the stores themselves).  Collective: every rank of the
 * communicator must call attach_peers. */
int tffft_plan_landing_handle(tffft_plan_t plan, uint8_t handle[64]);
int tffft_plan_attach_peers(tffft_plan_t plan, const uint8_t* handles /* p * 64 bytes */);
/* algorithm flags actually in effect (a flag is dropped when the grid has no such kernel) */
int tffft_plan_flags(tffft_plan_t plan, int* flags);
/* device bytes owned by the plan (staging, twiddles, statistics) */
int tffft_plan_workspace_bytes(tffft_plan_t plan, size_t* bytes);
/* element counts: real slab n0/p*n1*n2 reals, spectral slab n1/p*n0*(n2/2+1) complex */
int tffft_plan_sizes(tffft_plan_t plan, int64_t* real_elems, int64_t* spec_elems);
int tffft_plan_destroy(tffft_plan_t plan);

/* Forward r2c (collective).  real_in: (n0/p, n1, n2) row-major, not modified.
 * spec_out: STRIDED_INPLACE spectral slab, logical (j, r, k) at
 * (r % n0p)*n1*n2c + (r / n0p)*n1p*n2c + j*n2c + k (layout.py:189-198),
 * value = unnormalised global bin (r, rank*n1p + j, k). */
int tffft_forward(tffft_plan_t plan, const void* real_in, void* spec_out, void* stream);
/* Inverse c2r (collective), normalised by 1/(n0 n1 n2).  spec_inout is
 * consumed (overwritten) as in dfft.py:182-184; real_out: (n0/p, n1, n2). */
int tffft_inverse(tffft_plan_t plan, void* spec_inout, void* real_out, void* stream);

/* --- instrumentation ---------------------------------------------------- */
/* enable CUDA-event stage timing (adds events, no host sync inside calls) */
int tffft_set_timing(tffft_plan_t plan, int enable);
/* accumulated {stage1, exchange, stage3} milliseconds since the last reset;
 * synchronises on the recorded events */
int tffft_stage_times(tffft_plan_t plan, double ms[3]);
/* {bytes_packed, bytes_wire, bytes_unpacked} since the last reset */
int tffft_counters(tffft_plan_t plan, uint64_t bytes[3]);
int tffft_reset_instrumentation(tffft_plan_t plan);
/* Hermitian consistency of the LAST inverse: synchronises on it, returns the
 * largest discarded imaginary magnitude and TFFFT_ERR_CONSISTENCY when a plane
 * violates the reference tolerance 1e-9*n2*max|X| (kernels.py:223-238). */
int tffft_consistency(tffft_plan_t plan, double* residue);
/* diagnostic: the exchange's NCCL calls (grouped ncclSend / ncclRecv, ncclAlltoAll when the loaded NCCL has it,
 * the one-int ncclAllReduce barrier, the async-error poll) as a ONE-rank loopback on `device`, `count` real
 * elements of `dtype`; received data must equal what was sent.  As much of the NCCL path (exchange.py:263-290
 * over transport.py:359-419) as a one-GPU box can execute: NCCL refuses two ranks on one device. */
int tffft_nccl_loopback(int device, long long count, int dtype, int* ran_alltoall);
/* debug: fill the plan's exchange staging / landing buffers and c2r row
 * records with 0xFF bytes (NaN), so a read of an element no stage wrote shows
 * up as NaN in the output; synchronous */
int tffft_plan_poison(tffft_plan_t plan);
/* Deferred consistency mode (deferred = 1): every inverse folds its Hermitian
 * check (the same test as tffft_consistency) into a device accumulator, with no
 * host synchronisation per call; tffft_consistency_collect synchronises,
 * returns the largest residue and TFFFT_ERR_CONSISTENCY if any inverse since
 * the last collect violated the tolerance.  deferred = 0: tffft_consistency. */
int tffft_set_consistency_mode(tffft_plan_t plan, int deferred);
int tffft_consistency_collect(tffft_plan_t plan, double* residue, uint64_t* calls);
/* number of kernels this library launched on the plan since the last reset */
int tffft_launch_count(tffft_plan_t plan, uint64_t* launches);

/* --- host-only geometry (no GPU needed) ---------------------------------- */
/* STRIDED exchange schedule of one rank: up to max_ops rows of
 * {peer, send_offset, recv_offset, count} in complex elements: one send of the
 * staging band [q][i][j][k] and one receive into the landing band, per peer.
 * The FFT stage after the exchange reads the landing band through the
 * STRIDED_INPLACE addressing (exchange.py:114-121's strided descriptor applied
 * by the kernel).  Same list for forward and inverse (exchange.py:120-121). */
int tffft_exchange_schedule(int n0, int n1, int n2, int p, int rank, int64_t* ops, int64_t max_ops,
                            int64_t* nops);
/* twiddle-table geometry of the radix schedule for length 2^log2n (for tests) */
int tffft_radix_schedule(int log2n, int* radices, int* npasses);

#ifdef __cplusplus
}
#endif
#endif /* TFFFT_H */
