/*
 * vr.h — C ABI of libvr, the B200-native Vietoris–Rips persistence barcode library.
 *
 * The operation (PAPER.md Ch.5, "Ripser++"): given a finite metric space by its
 * distance matrix (Def 5.1.1), compute the persistence barcode over Z/2
 * of the Vietoris–Rips filtration Rips_t(X) = { s : diam(s) <= t } (Eq 5.3,
 * P:4668-4672) for homology dimensions 0..max_dim, i.e. the persistence pairs of the
 * simplex-wise refinement of §5.1.4 as the standard algorithm (Alg 11,
 * P:4724-4745) defines them.  The data-parallel hot path per dimension d >= 1 runs on
 * the GPU (sm_100a): enumeration of the d-simplices through the combinatorial number
 * system (Eq 5.6) with their diameters and the threshold filter (Alg 17/18,
 * P:5691-5731), the apparent-pair test (Def 5.3.4 / Lemma 5.3.6 / Alg 13,
 * P:4926-5025), clearing (§5.2.3, Lemma 4.2.3, Prop 5.3.9), stream compaction
 * (§5.5.3) and the radix sort into coboundary order (Fig 5.2 caption).  The
 * few non-apparent columns are reduced on the host (Alg 12 / §5.2.9-5.2.11); dimension
 * 0 is union-find (§5.2.5).
 *
 * Conventions
 *   - dist_lower_tri: n(n-1)/2 fp32 values in Ripser lower-distance order: the entry for
 *     (i, j), i > j, is at index i(i-1)/2 + j.  Distances must be >= 0 and
 *     not NaN.  Zero distances (duplicate points) are accepted (reading A35).
 *   - threshold: +INFINITY = full Rips; the library then cuts at the enclosing radius
 *     R = min_x max_y d(x, y) (§5.2.12, Prop 5.2.13), which leaves every
 *     positive-length and essential bar unchanged.  A finite threshold t >= 0 is
 *     inclusive: a simplex is present iff diam <= t (Eq 5.3, Alg 17 line 3).
 *   - Output per dimension 0..max_dim: (birth, death) fp32 pairs with birth < death,
 *     death = +INFINITY for essential classes, sorted by (birth, death).  Births and
 *     deaths are copies of distance-matrix entries (bit-exact).  Zero-length pairs are
 *     only counted (vr_stats) unless vr_options.include_zero is set.
 *   - Ownership: every pointer argument is owned by the caller and only read during the
 *     call; a vr_result is library-owned and released with vr_free; pointers returned by
 *     accessors stay valid until vr_free.
 *   - Errors: every int-returning entry returns 0 (VR_OK) or a VR_E* code and sets a
 *     thread-local message readable with vr_last_error(); on error *out is set to NULL.
 *     Capacity problems (C(n, max_dim+2) >= 2^63, a key that cannot be packed in 64
 *     bits, device memory) are raised before any GPU work.
 *   - Determinism: the output bytes do not depend on the launch configuration.
 */
#ifndef VR_H
#define VR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_OK 0
#define VR_EINVAL 1    /* usage: n < 1, max_dim < 0 or > VR_MAX_DIM, NaN/negative threshold, NULL */
#define VR_EINPUT 2    /* bad input: a negative or NaN distance */
#define VR_ECAPACITY 3 /* C(n, max_dim+2) >= 2^63, unpackable key, or out of device memory */
#define VR_EDEVICE 4   /* CUDA failure (no device, launch error, ...) */

#define VR_MAX_DIM 6

typedef struct {
  float birth;
  float death; /* +INFINITY for an essential class */
} vr_pair;

/* Index-level pair: the birth simplex (dim p) and death simplex (dim p+1) by their
 * combinatorial index (Eq 5.6).  death_cidx = UINT64_MAX for an essential class. */
typedef struct {
  uint64_t birth_cidx;
  uint64_t death_cidx;
} vr_index_pair;

typedef struct {
  int32_t include_zero;  /* 0 (default): report birth < death only; 1: also zero-length pairs */
  int32_t index_pairs;   /* 1: also keep the index-level pairing (every pair, apparent ones
                            included; intended for tests on small inputs); k > 1: the same,
                            but at most k apparent pairs per dimension (an arbitrary subset —
                            for sampled checks of full-size inputs).  The apparent pairs come
                            first, then one entry per residual column */
  int32_t residual_mode; /* 0: reduction-matrix (V) mode (§5.2.9, default); 1: oblivious (Alg 12) */
  int32_t apparent_steps;/* cofacets tested per column in the first (lane-per-column) phase of
                            the apparent test before a column moves to the warp-cooperative
                            phase; 0 = library default */
  int32_t device;        /* CUDA device ordinal used by vr_barcodes (host-pointer entry) */
  int32_t rows_per_grab; /* tuning: prefix rows a warp takes per atomic grab; 0 = default
                            (4 for n < 384, else 1) */
  int32_t scan_variant;  /* tuning: phase-1 scan loop, 0 = default, 1: one warp vote per cofacet
                            vertex, 2: per 4 vertices, 3: per 4 vertices then the unresolved
                            columns resolved warp-cooperatively in the same kernel; same results */
  int32_t sparse_mode;   /* -1/0 = auto (output-sensitive when <= 25% of the edges are under the
                            threshold, or when the dense index space is too large),
                            1 = always dense, 2 = always output-sensitive; same results */
  int32_t num_gpus;      /* vr_barcodes only: 0/1 = one GPU (options.device); G > 1 = devices
                            0..G-1 of this process, one host thread each, NCCL between them
                            (ncclCommInitAll), same result */
  int32_t hot_path_only; /* diagnostics: 1 = run the GPU hot path of every dimension but not the
                            host residual reduction (no pairs in dimensions >= 1; the counters
                            of dimension 1 are exact, higher dimensions miss the clearing by
                            residual deaths).  One GPU only */
  int32_t reserved[2];
} vr_options;

/* Per-dimension statistics (Table 5.1 / 5.5 counters, stage times). */
typedef struct {
  int64_t candidates;      /* C(n, d+1): every d-simplex index */
  int64_t survivors;       /* d-simplices with diam <= t */
  int64_t apparent;        /* apparent columns (each an apparent pair (s, t)) */
  int64_t cleared;         /* columns zeroed by clearing (deaths of dimension d-1) */
  int64_t residual_columns;/* non-apparent, non-cleared columns reduced on the host */
  int64_t emergent;        /* residual columns paired by the emergent shortcut (§5.2.11) */
  int64_t pairs_all;       /* finite pairs incl. zero-length, this dimension */
  int64_t pairs_positive;  /* finite pairs with birth < death */
  int64_t essential;       /* essential classes */
  int64_t queued;          /* columns sent to the warp-cooperative apparent phase */
  int64_t scanned;         /* cofacet vertices examined by the apparent tests and the
                              clearing recomputation (both phases) */
  double ms_enumerate;     /* GPU: enumerate + threshold + apparent phase 1 (+ dim-0 edge keys) */
  double ms_resolve;       /* GPU: apparent phase 2 + clearing + compaction */
  double ms_sort;          /* GPU: radix sort of the columns into coboundary order */
  double ms_residual;      /* host: residual reduction (dim 0: union-find) */
  double ms_transfer;      /* host<->device copies of this dimension's columns / pairs */
  int64_t kernels;         /* VR_KERNEL_* flags of the enumeration kernels this dimension ran */
  int64_t bytes_l2;        /* algorithmic L2 bytes of the dimension's kernels: 4 per rank read
                              (vr_plan_dim_timing [5]-[7]) */
  int64_t bytes_hbm;       /* algorithmic HBM bytes of its outputs: 16 per row kept for a later
                              dimension, 8 + 16 per residual column (written, then sorted: one
                              read + write), 24 per column queued for phase 2 */
  double ms_exchange;      /* sharded runs: wall ms of the dimension's exchanges (clearing input,
                              residual keys all-gather + merge, deaths broadcast); 0 on one GPU */
} vr_stats;
#define VR_KERNEL_ROW 1          /* k_enumerate: one warp per prefix row (dense) */
#define VR_KERNEL_FLAT 2         /* k_enumerate_flat: flattened (u_1, v_0) chunks (dense) */
#define VR_KERNEL_SPARSE 4       /* output-sensitive kernels (threshold-graph bitmap rows) */
#define VR_KERNEL_SMEM_WINDOW 8  /* dense: the 32-vertex scan window staged in shared memory */

typedef struct vr_result vr_result;

/* Host-pointer entry: copies dist_lower_tri to the device (options->device), computes
 * everything, returns a result handle.  opt may be NULL (defaults). */
int vr_barcodes(const float* dist_lower_tri, int64_t n, int32_t max_dim, float threshold,
                const vr_options* opt, vr_result** out);

/* Device-pointer entry: d_dist_lower_tri is a device pointer on the CURRENT device,
 * `stream` a cudaStream_t (NULL = legacy default stream) on which all GPU work is
 * ordered.  Intended for callers that already hold the matrix in HBM (e.g. a torch
 * tensor). */
int vr_barcodes_device(const float* d_dist_lower_tri, int64_t n, int32_t max_dim, float threshold,
                       const vr_options* opt, void* stream, vr_result** out);

/* Sparse-input entry (SPEC's sparse format): the distance matrix as
 * nnz (rows[k], cols[k], dist[k]) entries, host pointers, rows[k] != cols[k] in [0, n),
 * dist[k] finite and >= 0; a pair given twice keeps the smaller distance; absent pairs are
 * absent edges (never in the complex).  The dense lower triangle is built on the device
 * (+inf for absent pairs; any +inf entry in a dense input means the same).  With absent
 * edges the enclosing radius is +inf, so threshold = +inf keeps every given edge. */
int vr_barcodes_coo(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, const float* dist, int32_t max_dim,
                    float threshold, const vr_options* opt, vr_result** out);

int32_t vr_max_dim(const vr_result* r);
int64_t vr_num_pairs(const vr_result* r, int32_t dim);
const vr_pair* vr_pairs(const vr_result* r, int32_t dim);
int64_t vr_num_index_pairs(const vr_result* r, int32_t dim); /* 0 unless options.index_pairs */
const vr_index_pair* vr_index_pairs(const vr_result* r, int32_t dim);
int vr_stats_get(const vr_result* r, int32_t dim, vr_stats* s);
float vr_threshold_used(const vr_result* r); /* t actually applied (R when threshold = +inf) */
void vr_free(vr_result* r);
const char* vr_last_error(void);

/* ----------------------------------------------------------------------------------
 * Hot-path replay (benchmarking).  A vr_plan holds the device tables and the clearing
 * inputs (residual deaths of every dimension) found by one full run, so the GPU hot
 * path of all dimensions 1..max_dim — tables (a0), enumeration + threshold + apparent
 * test (a1, a5), clearing (a2), compaction (a3, a6) and the radix sort of the columns
 * into coboundary order (a4) — can be re-run on the device with no host work in
 * between beyond launch bookkeeping.  The residual reduction and dimension 0 are not
 * part of the replay ("off path, reported separately").
 * ---------------------------------------------------------------------------------- */
typedef struct vr_plan vr_plan;

/* Builds the plan from a device matrix and runs the full computation once (the result
 * of that run is returned in *out if out != NULL, else dropped). */
int vr_plan_create(const float* d_dist_lower_tri, int64_t n, int32_t max_dim, float threshold,
                   const vr_options* opt, void* stream, vr_plan** plan, vr_result** out);
/* Re-runs the hot path for all dimensions, asynchronously on the plan's stream.
 * Returns the number of kernels launched in *launches (may be NULL). */
int vr_plan_replay(vr_plan* plan, int64_t* launches);
/* Survivors (sum over d = 1..max_dim) — the numerator of hot-path simplices/s. */
int64_t vr_plan_survivors(const vr_plan* plan);
/* Apparent and residual column totals counted by the last replay (synchronizes the
 * plan's stream), to verify that a replay did the work. */
int vr_plan_check(vr_plan* plan, int64_t* apparent_total, int64_t* residual_total);
/* Device time (ms, CUDA events on the plan's stream) of the last replay's stages, summed
 * over dimensions: [0] tables (a0), [1] enumerate + apparent phase 1 (with each
 * dimension's setup), [2] apparent phase 2 + clearing + compaction, [3] radix sort.
 * Synchronizes the plan's stream.  Also the algorithmic work of the plan's first run,
 * summed over d: [4] candidates examined, [5] survivors, [6] cofacet vertices scanned (both
 * phases), [7] integer ops of the enumeration kernels = 2 per rank read (vr_plan_dim_timing
 * [5] + [6]) + the decode compares, [8] the same for the phase-2 kernels (DESIGN.md
 * "Roofline"). */
int vr_plan_timing(vr_plan* plan, double out[9]);
/* Per dimension d (1..max_dim) of the last replay (synchronizes the plan's stream):
 * [0] device ms of the enumeration kernel(s) (a1 + a2 + a5 phase 1 + a3), [1] phase-2
 * kernel(s) (a5 phase 2 + a2 + a6), [2] the radix sort of the residual columns (a4, + the
 * next dimension's death bits / clearing-set inserts), [3] the dimension's setup (counter
 * reset, next clearing bitmap / set reset); and the algorithmic work of the plan's first
 * run: [4] survivors, [5] rank reads of the
 * enumeration (dense: d per candidate index, every C(n, d+1); output-sensitive: the reads
 * of the candidate examination — d per listed C(σ) entry in one level, d-1 per C(τ) entry
 * plus 1 per (σ, C(τ) entry) in two levels), [6] rank reads of the apparent test in the enumeration kernel
 * ((d+1) per scanned cofacet vertex + C(d+2, 2) per tested column), [7] rank reads of the
 * phase-2 kernel, [8] decode compares ((d+1)·⌈log2 n⌉ per tested column — credited work the
 * fused kernels do not execute), [9] the VR_KERNEL_* flags. */
int vr_plan_dim_timing(vr_plan* plan, int32_t d, double out[10]);
void vr_plan_free(vr_plan* plan);

int64_t vr_plan_launches(const vr_plan* plan); /* kernels launched through this plan so far */

/* ----------------------------------------------------------------------------------
 * Multi-GPU (the a7 exchange).  The distance matrix is replicated; the
 * rows of every dimension are sharded over the ranks (dense prefix rows and sparse vertex
 * rows interleaved; sparse rows of higher dimensions are each rank's own survivors of a lower
 * dimension, which partitions the simplices — Cor 5.3.7: columns are
 * independent).  Per dimension, inside the library:
 *   A. the next dimension's clearing input: SUM all-reduce of the clearing bitmap (every
 *      death bit is set by exactly one rank, so the sum is the OR), or, for the hash-set
 *      clearing of the output-sensitive mode, an all-gather of every rank's apparent
 *      cofacets, inserted into each rank's set;
 *   B. the residual columns: all-gather of the locally sorted keys (padded to the largest
 *      count with ~0) and a device merge (every key's output position = its index + the
 *      number of smaller keys in every other rank's list, by binary search);
 *   C. rank 0 runs the host residual on the merged columns and broadcasts the deaths,
 *      which every rank turns into the next dimension's clearing input.
 * At the end rank 0 broadcasts the barcode (pairs + index pairs) and the counters are
 * summed, so every rank returns the same vr_result, byte-identical to the one-GPU result.
 *
 * The transport is a vr_comm: three collectives on DEVICE buffers, ordered on `stream`
 * (the caller's stream of that rank); each returns 0 or a VR_E* code.  The library
 * provides NCCL communicators (one process per GPU: vr_comm_nccl with an id from
 * vr_nccl_unique_id shared by any out-of-band channel, e.g. torch.distributed; one process
 * driving several GPUs: vr_options.num_gpus in vr_barcodes) and an in-process group whose
 * ranks are host threads sharing one GPU (vr_comm_local: tests of the multi-rank logic on
 * one device; the collectives stage through host memory, no kernel waits on another).
 * ---------------------------------------------------------------------------------- */
typedef struct vr_comm {
  void* ctx;
  int32_t rank, world;
  int (*allreduce_sum_u64)(void* ctx, uint64_t* buf, int64_t n, void* stream);          /* in place */
  int (*allgather_u64)(void* ctx, const uint64_t* send, uint64_t* recv, int64_t n_each, void* stream);
  int (*broadcast_u64)(void* ctx, uint64_t* buf, int64_t n, int32_t root, void* stream); /* in place */
  void (*destroy)(void* ctx);
} vr_comm;

/* a fresh NCCL unique id (128 bytes) for vr_comm_nccl (call on one rank, share the bytes) */
int vr_nccl_unique_id(uint8_t id[128]);
/* this process's rank of an NCCL communicator over `world` ranks on CUDA device `device` */
int vr_comm_nccl(const uint8_t id[128], int32_t rank, int32_t world, int32_t device, vr_comm** out);
/* `world` ranks in this process sharing the current device (each rank is run by its own
 * host thread); comms[r] is rank r's communicator */
int vr_comm_local(int32_t world, vr_comm** comms);
void vr_comm_free(vr_comm* c);

/* This rank's part of a distributed computation: every rank calls it with the same input
 * (host pointer, copied to the rank's current device), the same options and its own
 * communicator; all ranks return the same result.  Collective: blocks until every rank has
 * called it. */
int vr_barcodes_comm(const float* dist_lower_tri, int64_t n, int32_t max_dim, float threshold, const vr_options* opt,
                     const vr_comm* comm, vr_result** out);
/* The same from a device matrix on the current device and `stream`, keeping a plan whose
 * vr_plan_replay re-runs the sharded hot path with exchanges A and B (bench.py's timed
 * multi-GPU step); *out (may be NULL) receives the result. */
int vr_plan_create_comm(const float* d_dist_lower_tri, int64_t n, int32_t max_dim, float threshold, const vr_options* opt,
                        const vr_comm* comm, void* stream, vr_plan** plan, vr_result** out);

/* ----------------------------------------------------------------------------------
 * Component entry (tests, no GPU needed): the library's host residual reduction of
 * dimension d (Alg 12 / §5.2.9-5.2.11) on caller-provided columns.  rank: host n x n rank
 * matrix (see vr_common.cuh), values[r] = the distance with rank r, keys: the
 * non-apparent, non-cleared columns ((maxr - rank) << cbits | cidx) sorted ascending.
 * Writes one entry per column (death = +inf, death_cidx = UINT64_MAX for essential).
 * ---------------------------------------------------------------------------------- */
int vr_host_residual(const uint32_t* rank, const float* values, int64_t nvalues, int64_t n, int32_t d, uint32_t maxr,
                     int32_t cbits, const uint64_t* keys, int64_t nkeys, int32_t mode, float* birth, float* death,
                     uint64_t* birth_cidx, uint64_t* death_cidx, int64_t* emergent);

/* ----------------------------------------------------------------------------------
 * HYPHA (PAPER.md Ch.4, Algs 3-10): pivots of an EXPLICIT Z/2
 * boundary matrix given in CSC — col_ptr[ncols+1] (int64), rows[] ascending within each
 * column and strictly below the column (rows[k] < j: a filtration's boundary matrix is
 * strictly upper triangular).  GPU-scan (leftmost 1s, 0-addition pivots, clearing marks,
 * unstable columns) on the current device, then on the host optional compression
 * (VR_HYPHA_COMPRESSION) and the reduction of the unstable columns (twist order when
 * dims[] — the dimension of every column — is given, else left to right).
 * Clearing (VR_HYPHA_CLEARING, and the twist order) and compression use ∂∂ = 0: set them
 * only for a boundary matrix; with flags = 0 and dims = NULL any strictly upper-triangular
 * Z/2 matrix is reduced exactly (Alg 2's pivots).
 * low_out[j] = the pivot row of column j in the reduced matrix, or -1 (a zero column).
 * Returns VR_EINPUT for a malformed matrix.
 * ---------------------------------------------------------------------------------- */
#define VR_HYPHA_COMPRESSION 1
#define VR_HYPHA_CLEARING 2
typedef struct {
  int64_t stable;      /* columns the GPU scan found final (zero, 0-addition pivots, cleared) */
  int64_t unstable;    /* columns left for the host */
  int64_t cleared;     /* nonzero columns zeroed by clearing (Lemma 4.2.3) */
  int64_t compressed;  /* entries removed by compression (Lemma 4.2.4/4.2.5) */
  int64_t additions;   /* column additions on the host */
  double ms_gpu_scan;  /* device time of the three scan kernels (CUDA events) */
  double ms_host;      /* host phase: compression + reduction */
  double ms_compress_scan; /* of which FIND-COMPRESSIBLE over all rows */
  double ms_reduce;    /* of which the reduction of the unstable columns */
  double ms_total;     /* the whole call: checks, H2D, scan, D2H, host phase */
  double ms_prepare;   /* of which before the scan (col_ptr checks, buffers, H2D issue) */
  int64_t threads;     /* host threads of the reduction */
} vr_hypha_stats;
int vr_hypha_pivots(const int64_t* col_ptr, const int32_t* rows, int64_t ncols, const int32_t* dims, int32_t flags,
                    int32_t* low_out, vr_hypha_stats* stats);

/* ----------------------------------------------------------------------------------
 * Min-cost flow (§6.3.7, Def 6.2.2 / Eq 6.38; SURVEY.md §8(f) NEXT-4 component):
 * the uncapacitated transshipment problem — nodes 0..nodes-1 with integer supply (Σ = 0;
 * positive = source), arcs tail[a] -> head[a] with cost[a] >= 0 (finite) and no capacity;
 * *total_cost = min Σ cost·flow.  Primal network simplex with block search pivot (block
 * √arcs), host C++, no GPU needed.  max_blocks > 0 stops after that many searched blocks
 * (the C√(mn)+b criterion of P:7112; stats->optimal = 0 then); 0 = run to optimality.
 * VR_EINPUT: supplies not balanced, an arc out of range / negative / non-finite cost, or
 * an infeasible network.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int64_t pivots;      /* basis changes */
  int64_t degenerate;  /* of which with zero flow change */
  int64_t blocks;      /* arc blocks searched */
  int32_t optimal;     /* 1 = no arc with a negative reduced cost left */
  int32_t infeasible;  /* 1 = an artificial arc still carries flow */
  double ms_pricing;   /* time in the block search */
  double ms_update;    /* time in the basis updates */
} vr_mcf_stats;
int vr_min_cost_flow(int64_t nodes, const int64_t* supply, int64_t arcs, const int32_t* tail, const int32_t* head,
                     const double* cost, int64_t max_blocks, double* total_cost, vr_mcf_stats* stats);

/* ----------------------------------------------------------------------------------
 * PDoptFlow (PAPER.md Ch.6, Alg 22): the 1-Wasserstein distance
 * (Eq 6.36, l2 ground metric, unmatched points go to the diagonal at (d-b)/√2) between two
 * persistence diagrams A (nA points) and B (nB points), each point (birth, death) as two
 * fp32 (the layout of vr_pair), finite.  s > 0: the (1+O(ε)) approximation — RWMD lower
 * bound (Alg 20), δ-condensation (Alg 21, seeded perturbation), s-WSPD spanner on a split
 * tree (Algs 23-25), diagonal arcs (Alg 26), min-cost flow by network simplex; the
 * guaranteed band is stats.bound_lo·W1 <= *w1 <= stats.bound_hi·W1 (Prop 6.3.2 x
 * Thm 6.3.6, for s > 2).  s <= 0 or VR_W1_EXACT: the exact W1 (complete network on the
 * 0-condensed points).  VR_W1_NO_CONDENSE: spanner without δ-condensation.  max_blocks as
 * in vr_min_cost_flow.  Device work on the current device, default stream.
 * ---------------------------------------------------------------------------------- */
#define VR_W1_EXACT 1
#define VR_W1_NO_CONDENSE 2
#define VR_W1_WARM_DIAGONAL 4 /* start the simplex from the all-to-diagonal basis (default: big-M) */
typedef struct {
  int64_t points_a, points_b;  /* input points */
  int64_t nodes;               /* network nodes (condensed points + the two diagonal nodes) */
  int64_t arcs;                /* network arcs after de-duplication */
  int64_t wspd_pairs;          /* s-WSPD pairs (biarcs) */
  int64_t tree_height;         /* split tree height */
  int64_t wspd_levels;         /* frontier passes of the level-synchronous WSPD */
  int64_t pivots, degenerate, blocks;
  int32_t optimal;             /* 1 = the simplex ran to optimality */
  int32_t condensed;           /* 1 = δ-condensation applied */
  int32_t warm_start;          /* 1 = the simplex started from the all-to-diagonal basis */
  int32_t pad_;
  double rwmd;                 /* L of Alg 20 (0 in exact mode) */
  double delta;                /* δ of Alg 21 line 7 (0 = not condensed) */
  double eps_condense;         /* ε of Alg 21 line 3-6 */
  double eps_spanner;          /* ε' = 4/s + 4/(s-2) (Thm 6.3.6) */
  double bound_lo, bound_hi;   /* guaranteed band around the exact W1 */
  double ms_h2d, ms_rwmd, ms_condense, ms_tree, ms_wspd, ms_arcs, ms_d2h, ms_build, ms_simplex, ms_total;
  double ms_pricing, ms_update; /* of ms_simplex: block search, basis update */
} vr_w1_stats;
int vr_w1(const float* A, int64_t nA, const float* B, int64_t nB, double s, uint64_t seed, int32_t flags,
          int64_t max_blocks, double* w1, vr_w1_stats* stats);
/* the network of Alg 22 lines 1-5 (tests, inspection): nodes = condensed points then ā
   (absorbs A) then b̄ (feeds B); xy of the diagonal nodes is NaN */
typedef struct vr_w1_net vr_w1_net;
int vr_w1_network(const float* A, int64_t nA, const float* B, int64_t nB, double s, uint64_t seed, int32_t flags,
                  vr_w1_net** out, vr_w1_stats* stats);
int64_t vr_w1_net_nodes(const vr_w1_net* net);
int64_t vr_w1_net_arcs(const vr_w1_net* net);
void vr_w1_net_get(const vr_w1_net* net, double* xy, int64_t* supply, int32_t* tail, int32_t* head, double* cost);
void vr_w1_net_free(vr_w1_net* net);

/* ----------------------------------------------------------------------------------
 * Component entry (tests): the library's device radix sort on
 * caller keys.  keys: HOST pointer to n uint64 values, sorted ascending in place on bits
 * [begin_bit, end_bit) (LSD, stable; bits outside the range do not take part in the
 * order), using the current device.  Returns VR_OK or an error code.
 * ---------------------------------------------------------------------------------- */
int vr_radix_sort_u64(uint64_t* keys, int64_t n, int32_t begin_bit, int32_t end_bit);
/* Component entry (tests): the residual-column sort — keys = (field << cbits) | low with
 * field < bins, ascending on bits [0, end_bit) (the keys must be distinct).  *mode in: -1
 * choose (counting sort on the field + the runs of equal field sorted, falling back to the
 * radix sort when runs are too long or too many), 0 radix sort, 1 counting sort; out: the
 * path taken. */
int vr_sort_columns_u64(uint64_t* keys, int64_t n, int32_t cbits, int32_t end_bit, uint64_t bins, int32_t* mode);

/* ----------------------------------------------------------------------------------
 * Diagnostics (bench.py): measured on-chip peaks of `device` — the integer-ALU throughput
 * (IMNMX/LOP3 chains, ops/s) and the L2 read bandwidth (a 48 MiB L2-resident buffer,
 * bytes/s) — the roofline denominators of the hot kernels.  Synchronous;
 * allocates 48 MiB on the device for the call.
 * ---------------------------------------------------------------------------------- */
int vr_probe_peaks(int32_t device, double* alu_ops_per_s, double* l2_bytes_per_s);

#ifdef __cplusplus
}
#endif
#endif /* VR_H */
