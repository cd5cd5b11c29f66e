/*
 * ttn_cbc.h — C ABI of libttncbc.so: Cholesky-based compression (CBC) of a tree tensor
 * network operator (TTNO) applied to a tree tensor network state (TTNS) on B200 (sm_100a).
 *
 * Method: M. Milbradt, S. Sun, C. B. Mendl, J. Gray, G. K.-L. Chan, arXiv 2601.19650,
 * "Efficient Application of Tensor Network Operators to Tensor Network States".
 * Citations are PAPER.md line numbers (P:n) with the section / equation they fall in.
 *
 * Conventions (all calls):
 *  - Complex numbers are ttn_c128 = {double re, im} (layout of C99 double _Complex and
 *    cuDoubleComplex).  All tensors are dense, row-major (last index fastest).
 *  - Every call returns a ttn_status.  Nothing throws across the ABI.  On error every
 *    output handle is set to NULL and ttn_last_error(ctx) describes the failure.
 *  - A ttn_ctx binds one CUDA device and one CUDA stream.  All device work of a call is
 *    enqueued on that stream; calls that return host values synchronise it.  A ctx is not
 *    thread-safe; distinct ctxs may be used concurrently.
 *  - Handles (ttn) are immutable, library-owned and device-resident.  The caller destroys
 *    every handle it receives (ttn_destroy) before destroying the ctx that created it.
 */
#ifndef TTN_CBC_H
#define TTN_CBC_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TTN_API __attribute__((visibility("default")))
#else
#define TTN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TTN_OK = 0,
  TTN_ERR_ARG = 1,          /* NULL pointer, max_bond < 1, tol outside [0,1), bad node id   */
  TTN_ERR_TOPOLOGY = 2,     /* not a single rooted tree; op and state parent arrays differ  */
  TTN_ERR_SHAPE = 3,        /* bond / physical-dimension mismatch across an edge or op-state */
  TTN_ERR_OOM = 4,          /* device or pinned-host allocation failed                       */
  TTN_ERR_CUDA = 5,         /* a CUDA runtime call or kernel launch failed                   */
  TTN_ERR_NUMERIC = 6,      /* non-finite values, eigensolver / Cholesky breakdown            */
  TTN_ERR_UNSUPPORTED = 7,  /* a size beyond the compiled limits (see ttn_last_error)        */
  TTN_ERR_NCCL = 8          /* NCCL missing or a collective failed (multi-GPU apply)          */
} ttn_status;

typedef enum { TTN_STATE = 0, TTN_OPERATOR = 1 } ttn_kind;

typedef struct { double re, im; } ttn_c128;

typedef struct ttn_ctx_s* ttn_ctx;
typedef struct ttn_s* ttn;

/* Per-apply report (§IV.B metrics; SPEC ApplyReport).            */
typedef struct {
  double norm;                 /* ||phi|| = ||T'_root||_F (non-root tensors are isometries) */
  double discarded_weight_sum; /* sum over all compress steps of the dropped eigenvalues     */
  int64_t max_bond;            /* largest bond of the result                                */
  int64_t peak_entries;        /* largest number of complex entries held by one intermediate */
  double seconds;              /* host wall time of the call                                */
  double flops_algorithmic;    /* 8 * complex MACs of every contraction / Gram / factor GEMM */
  int32_t rank_fallbacks;      /* Eq. 13 QRs that fell back from CholeskyQR2 (rank-deficient) */
  int32_t host_syncs;          /* stream synchronisations taken for data-dependent ranks     */
  int32_t split_compresses;    /* partitioned apply: compresses whose Gram was row-split over
                                  ranks (partial Grams summed by allreduce); 0 otherwise      */
  int32_t exact_factors;       /* compresses taken by the exact-factor shortcut (untruncated,
                                  certified full rank: factor = Cholesky factor of the Gram, no
                                  eigensolver)                       */
  double flops_gemm_exec;      /* flops issued to the complex GEMM kernel (all contraction,
                                  Gram, factor, S, CholeskyQR and R products as executed)    */
  double flops_gemm_min;       /* the same work at its algorithmic minimum: node contractions
                                  at their cheapest pairwise order (the executed order may trade
                                  flops for speed), Grams as Hermitian products (4 n^2 K)    */
} ttn_cbc_report;

/* ---------------------------------------------------------------- context             */
/* Device memory source (PyTorch interop): alloc(state, bytes, stream) returns
 * `bytes` of device memory usable in stream order on `stream` (NULL = out of memory);
 * free(state, ptr, stream) returns it.  The library calls free only after the ctx stream
 * has completed all work on the block, so the allocator may reuse it on any stream at once
 * (e.g. torch.cuda.caching_allocator_alloc / caching_allocator_delete).  Callbacks may run on
 * library worker threads (ttn_ctx_set_workers).                                          */
typedef struct {
  void* (*alloc)(void* state, size_t bytes, void* stream);
  void (*free)(void* state, void* ptr, void* stream);
  void* state;
} ttn_allocator;

/* Create a context on CUDA device `device` using stream `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream).  `alloc` (may be NULL) supplies all device memory of
 * TTN handles and of the per-apply workspaces; with NULL the context owns a stream-ordered
 * memory pool (cudaMemPoolCreate; memory returns to the device when the ctx is destroyed).
 * The allocator struct is copied.  Errors: ARG (bad device, NULL out, half-filled allocator),
 * CUDA, OOM.                                                                              */
TTN_API ttn_status ttn_ctx_create(int device, void* cuda_stream, const ttn_allocator* alloc, ttn_ctx* out);
TTN_API ttn_status ttn_ctx_destroy(ttn_ctx ctx);
/* Text of the last error on this ctx; valid until the next call on the ctx.             */
TTN_API const char* ttn_last_error(ttn_ctx ctx);
/* Library version string, e.g. "ttncbc 0.1 sm_100a".                                    */
TTN_API const char* ttn_version(void);

/* ---------------------------------------------------------------- tree tensor networks */
/* Create a TTNS (kind = TTN_STATE, Eq. 2) or TTNO (TTN_OPERATOR, Eq. 4).
 *  n_nodes   number of sites L >= 1
 *  parent    parent[i] of node i; exactly one -1 (the root).  Children of a node are
 *            ordered by ascending node id, which fixes the leg order below.
 *  phys_dim  d_i >= 1 ("d_i can be 1")
 *  bond      bond[i] = extent of edge (i, parent[i]) >= 1; ignored for the root (extent 1)
 *  data      data[i] points to node i's tensor, row-major in the ABI leg order
 *              state    : [d_i, bond(parent edge), bond(child c1), bond(child c2), ...]
 *              operator : [d_i (out sigma'), d_i (in sigma), bond(parent), bond(c1), ...]
 *            The root's parent leg is present with extent 1; leaves have no child
 *            legs.  MPS / MPO: parent[i] = i-1, site i's tensor is [d, a_left, a_right]
 *            (Eq. 3).
 *  data_on_device  0: data[i] are host pointers (copied H2D); 1: device pointers (D2D).
 * The data is copied; the caller keeps ownership of its buffers.  Consecutive nodes whose
 * tensors are adjacent in memory (one packed buffer, node 0 first) are copied in one
 * transfer.  Pageable host data is fully copied when the call returns; page-locked
 * (pinned) host data and device data are copied asynchronously on the ctx stream, so the
 * caller must not modify them until the stream has passed the copy (every call that
 * returns host values, e.g. cbc_apply, synchronises it).
 * Errors: TOPOLOGY (no single root, cycle), ARG (NULL, d < 1, bond < 1).               */
TTN_API ttn_status ttn_create(ttn_ctx ctx, ttn_kind kind, int32_t n_nodes, const int32_t* parent,
                      const int32_t* phys_dim, const int64_t* bond,
                      const ttn_c128* const* data, int data_on_device, ttn* out);
TTN_API ttn_status ttn_destroy(ttn t);
TTN_API ttn_status ttn_n_nodes(ttn t, int32_t* out);
/* Shape of node `node` in ABI leg order; dims must hold >= 16 entries.                   */
TTN_API ttn_status ttn_node_shape(ttn t, int32_t node, int32_t* ndim, int64_t* dims);
/* Copy node `node` (ABI leg order) to host memory `host_out` with room for
 * `capacity_elems` complex entries (ARG if too small).  Synchronises the ctx stream.    */
TTN_API ttn_status ttn_get_tensor(ttn_ctx ctx, ttn t, int32_t node, ttn_c128* host_out, size_t capacity_elems);

/* Copy every node (node 0 first, each in ABI leg order, concatenated) to host memory with
 * one D2H copy; capacity_elems must cover the sum of the node sizes.  Synchronises.     */
TTN_API ttn_status ttn_get_data(ttn_ctx ctx, ttn t, ttn_c128* host_out, size_t capacity_elems);
/* ttn_get_data for n TTNs (host_out[i], capacity_elems[i]): all D2H copies are enqueued,
 * then the ctx stream is synchronised once.  Pinned host buffers let the copies run at
 * full link speed.  ARG if any buffer is too small (nothing copied then).                */
TTN_API ttn_status ttn_get_data_batch(ttn_ctx ctx, int32_t n, const ttn* t, ttn_c128* const* host_out,
                                      const size_t* capacity_elems);

/* ---------------------------------------------------------------- CBC                  */
/* phi ~= O |psi> by CBC (§III.B, Eqs. 10-14; tensor train §III.A,
 * Eqs. 5-9, is the special case of a chain rooted at site 0).
 *  op, state  TTNO and TTNS on the same parent array and physical dimensions.
 *  max_bond   D-bar >= 1: every bond of the result is <= max_bond.
 *  tol        relative singular-value cutoff in [0, 1): directions with
 *             sigma_j <= tol * sigma_1 are dropped ("setting a tolerance for the SVD";
 *             reading A3 in DESIGN.md).  tol = 0 keeps min(max_bond, numerical rank).
 *  out        new TTNS, same topology; non-root tensors are isometries toward the root
 *             (Q of Eq. 13), the root carries the norm; no renormalisation.
 *  rep        optional report (may be NULL).
 * Errors: TOPOLOGY, SHAPE, ARG, NUMERIC, OOM, CUDA.                                      */
TTN_API ttn_status cbc_apply(ttn_ctx ctx, ttn op, ttn state, int64_t max_bond, double tol,
                     ttn* out, ttn_cbc_report* rep);
/* n independent applies in one level-synchronous schedule (all instances share the parent
 * array and physical dimensions; bonds may differ).  outs[n]; reps[n] may be NULL.       */
TTN_API ttn_status cbc_apply_batch(ttn_ctx ctx, int32_t n, const ttn* ops, const ttn* states,
                           int64_t max_bond, double tol, ttn* outs, ttn_cbc_report* reps);

/* <a|b> = sum over all indices of conj(a) b, conjugate-linear in a (the inner product of
 * Eq. 2 states; the overlap the paper's error Err = ||psi0 - U psi0|| and the
 * fidelity checks of §IV.B rest on), by a leaves-to-root environment sweep:
 * every node contracts conj(a_i), b_i and its children's environments into its parent-edge
 * environment (bond_a x bond_b).  a and b share the parent array and physical dimensions,
 * bonds may differ.  Synchronises the stream.  Errors: ARG, TOPOLOGY, SHAPE.             */
TTN_API ttn_status ttn_overlap(ttn_ctx ctx, ttn a, ttn b, ttn_c128* out);
/* <bra| op |ket> (one leaves-to-root sweep through bra*, op, ket); all three on one parent
 * array and physical dimensions.  With bra = cbc_apply(op, ket) this is the projection
 * identity <phi|O|psi> = ||phi||^2 (phi = W W^dagger O psi).  Synchronises the stream.     */
TTN_API ttn_status ttn_sandwich(ttn_ctx ctx, ttn bra, ttn op, ttn ket, ttn_c128* out);
/* ||op |ket>||^2 = <ket| op^dagger op |ket> by one sweep (environments carry four legs), so
 * the truncation error eps^2 = 1 - ||phi||^2 / ||O psi||^2 (A19) needs no dense vector.     */
TTN_API ttn_status ttn_op_norm2(ttn_ctx ctx, ttn op, ttn ket, double* out);
/* Batched overlaps <a_j|b_j>, j < n.                                                      */
TTN_API ttn_status ttn_overlap_batch(ttn_ctx ctx, int32_t n, const ttn* a, const ttn* b, ttn_c128* out);
/* Split every later cbc_apply_batch of >= 2n instances on ctx into n concurrent sub-batches,
 * each on an internal worker context (its own non-blocking stream, staging ring and arenas)
 * driven by its own host thread; the worker streams wait for ctx's stream at the start and
 * ctx's stream waits for them at the end, and the results belong to ctx.  Batches of small
 * trees (config 5's circuit layers) are bound by host-side planning and the per-level rank
 * synchronisations; overlapping sub-batches hides them.  n = 1 (default) turns it off.
 * Not combined with ttn_ctx_set_comm (a partitioned apply runs on ctx itself).  Errors: ARG. */
TTN_API ttn_status ttn_ctx_set_workers(ttn_ctx ctx, int n);

/* Schedule of cbc_apply / cbc_apply_batch on ctx (both on by default):
 *  speculate = 1: with tol = 0 the host plans every compress with the generic rank
 *    k = min(max_bond, m, n) and every QR of Eq. 13 as full rank, and the device checks
 *    that the eigensolver / CholeskyQR agree; the apply then synchronises ONCE (for its
 *    results) instead of once per tree level.  When a check fails (rank-deficient data, e.g.
 *    circuit states) the result is discarded and the apply re-runs with the ranks read per
 *    level; those shapes are not speculated again on this ctx.  tol > 0 and partitioned
 *    (multi-GPU) applies always read ranks per level.
 *  graphs = 1 (needs speculate): a successful speculative apply is captured as a CUDA graph
 *    keyed by the shapes and the input handles' device addresses; a later apply with the same
 *    key replays the graph (one launch, no host planning) and copies its outputs into fresh
 *    handles.  Up to 8 graphs per ctx (least recently used evicted).  Applies that need the
 *    Chebyshev solver (Grams of order > 512) synchronise inside and are not captured.
 * Resets the graph cache.  Errors: ARG.                                                   */
TTN_API ttn_status ttn_ctx_set_schedule(ttn_ctx ctx, int speculate, int graphs);

/* ---------------------------------------------------------------- multi-GPU            */
/* 128-byte NCCL unique id for a new communicator: create it on one rank and hand the same
 * bytes to every rank (e.g. by a torch.distributed broadcast).  NCCL is loaded at run time
 * (libnccl.so.2).  Errors: NCCL.                                                          */
TTN_API ttn_status ttn_comm_unique_id(void* out128);
/* Make ctx rank `rank` of a `world`-rank communicator (one process per GPU, NCCL over
 * NVLink / NVSwitch) and split every later cbc_apply / cbc_apply_batch on it into
 * `parts` >= world subtree groups (SURVEY §8(e) mechanism 2, B:5 (e), B:10):
 *  - the tree is cut below a replicated top: starting from the root's child subtrees, the
 *    largest subtree is replaced by its children until there are >= parts subtrees; the
 *    subtrees are dealt to the groups by size (largest first, to the lightest group) and
 *    group g belongs to rank g % world;
 *  - every rank passes the SAME op and state (replicated inputs) and receives the full result;
 *  - per apply: each rank runs the up-sweep (Eq. 10) of its subtrees; the subtree roots'
 *    up-factors (boundary environments) are broadcast from their owners; the top is swept
 *    up and down on every rank (replicated); each rank runs the down-sweep (Eq. 11) and the
 *    final sweep (Eqs. 12-14) of its subtrees; the subtree roots' R factors and every
 *    subtree's new tensors are broadcast; the top's final sweep closes the apply.
 *    The sequence of collectives depends only on the tree, never on data, so all ranks
 *    issue them in the same order.
 * world = 1 with parts > 1 runs the same partitioned schedule on one GPU (all groups local,
 * 1-rank NCCL collectives): the single-GPU check of the schedule.  unique_id128 = NULL
 * detaches the communicator (plain applies).  Errors: ARG, NCCL.                          */
TTN_API ttn_status ttn_ctx_set_comm(ttn_ctx ctx, const void* unique_id128, int rank, int world, int parts);
/* In-process loopback group of `world` ranks for the same partitioned schedule on ONE device
 * (tests, and machines with fewer GPUs than ranks): each rank is a ctx on its own stream,
 * driven by its own host thread; collectives are host barriers between the rank threads plus
 * stream-event dependencies and device copies / reductions (no kernel waits on another
 * rank).  All ranks' contexts must be on the same device.  The group is reference counted:
 * ttn_loopback_destroy drops the creator's reference.  Errors: ARG.                        */
TTN_API ttn_status ttn_loopback_create(int world, void** group_out);
TTN_API ttn_status ttn_loopback_destroy(void* group);
/* ttn_ctx_set_comm with a loopback group instead of NCCL (same partition, same schedule). */
TTN_API ttn_status ttn_ctx_set_comm_loopback(ttn_ctx ctx, void* group, int rank, int parts);
/* The partition ttn_ctx_set_comm would use (host-only, no device needed): group_out[i] = -1
 * for nodes of the replicated top, else the subtree group of node i (rank = group % world).
 * Errors: ARG, TOPOLOGY.                                                                  */
TTN_API ttn_status ttn_partition_plan(int32_t n_nodes, const int32_t* parent, int parts, int32_t* group_out);

/* ---------------------------------------------------------------- measurement          */
/* Process-wide kernel-family timing with CUDA events on the launching stream (used by
 * bench.py for the roofline).  on = 1 resets and enables, 0 disables.                    */
TTN_API ttn_status ttn_profile_enable(int on);
/* Totals since enable for one family ("zgemm", "heev", "potrf", "trtri", "geqr", "permute",
 * "scale_rows", "misc", or "all"): summed event time (ms), algorithmic flops and bytes of the
 * launches, and the number of launches.  Synchronises the recorded events.              */
TTN_API ttn_status ttn_profile_read(const char* family, double* ms, double* flops, double* bytes,
                                    int64_t* launches);
/* Number of kernels this library has launched in this process.                           */
TTN_API ttn_status ttn_launch_count(int64_t* out);

/* ---------------------------------------------------------------- eigensolver test hook */
/* The compress step's batched Hermitian eigensolver (B:5 (c); the truncation of
 * P:119, "compressed down to the desired new bond dimension", with the tolerance of P:362) on
 * nmat host matrices, for tests: a_host holds nmat n x n Hermitian matrices (row-major, full
 * storage, consecutive); on return lam_host[i*kmax + t] are the kmax largest eigenvalues of
 * matrix i (descending; entries past the kept rank are 0), vt_host[(i*kmax + t)*n + j] the
 * j-th entry of eigenvector t (rows past the kept rank are 0), k_host[i] the kept rank
 * k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > 1e-13 lam_1}) >= 1 and w_host[i] the
 * discarded weight trace - sum_{t<k} lam_t.  route: 0 = the library's choice, 1 = one-stage
 * tridiagonalisation, 2 = two-stage (band) reduction wherever 65 <= n <= 256.  Host buffers
 * are the caller's; synchronises.  Errors: ARG (sizes, kmax > n, tol outside [0, 1), route),
 * UNSUPPORTED (n beyond the eigensolver), CUDA.                                           */
TTN_API ttn_status ttn_test_heev(ttn_ctx ctx, int32_t nmat, int32_t n, int32_t kmax, int32_t max_bond, double tol,
                                 int32_t route, const ttn_c128* a_host, double* lam_host, ttn_c128* vt_host,
                                 int32_t* k_host, double* w_host);

/* ||a|| = sqrt(Re <a|a>) (ttn_overlap of a with itself; Eq. 2, used to normalise the
 * initial state, reading A16, and as ||phi|| in the report).  Synchronises.
 * Errors: ARG, TOPOLOGY.                                                                  */
TTN_API ttn_status ttn_norm(ttn_ctx ctx, ttn a, double* out);

#ifdef __cplusplus
}
#endif
#endif /* TTN_CBC_H */
