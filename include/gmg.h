/* gmg.h -- C ABI of libgmg: the data-parallel hot path of the local-smoothing
 * adaptive geometric multigrid of Clevenger, Heister, Kanschat, Kronbichler,
 * "A Flexible, Parallel, Adaptive Geometric Multigrid method for FEM"
 * (arXiv 1904.03317), built for NVIDIA B200 (sm_100a).  Citations "P:n" are
 * line numbers of PAPER.md (the paper's LaTeX); readings of the paper are the
 * "R#" entries of DESIGN.md.
 *
 * Conventions (all calls):
 *  - Every call returns gmg_status; GMG_OK == 0.  No exception crosses the ABI.
 *    On error, gmg_last_error() returns a thread-local message.
 *  - Handles are opaque, owned by the library, immutable after creation except
 *    through the documented setters, and destroyed by the matching *_destroy.
 *  - "host" pointers are caller-owned host memory, "device" pointers
 *    caller-owned CUDA device memory (fp64, int32, ...) on the hierarchy's device.
 *  - Export functions follow the size-query idiom: pass NULL arrays to obtain
 *    the count in *n, then call again with arrays of that size.
 *  - Device work is enqueued on the caller's `cuda_stream` (cudaStream_t, NULL =
 *    legacy default stream); calls return without synchronising unless stated.
 */
#ifndef GMG_H
#define GMG_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GMG_OK = 0,
  GMG_E_INVALID_ARG = 1,   /* null pointer, out-of-range argument */
  GMG_E_UNSORTED = 2,      /* leaves not strictly increasing in SFC order */
  GMG_E_NOT_TILING = 3,    /* leaves overlap or leave holes in the brick */
  GMG_E_UNBALANCED = 4,    /* 2:1 vertex balance violated */
  GMG_E_DEPTH = 5,         /* level too deep for 64-bit lattice keys */
  GMG_E_STATE = 6,         /* call not valid in this state (e.g. no device data) */
  GMG_E_ZERO_DIAG = 7,     /* zero diagonal on a smoothed row */
  GMG_E_SINGULAR_COARSE = 8,/* coarse matrix not SPD */
  GMG_E_NOT_CONVERGED = 9, /* CG reached max_it (x = last iterate) */
  GMG_E_CUDA = 10,         /* CUDA runtime error */
  GMG_E_NCCL = 11,         /* NCCL error */
  GMG_E_OOM = 12           /* host or device allocation failed */
} gmg_status;

typedef struct gmg_forest gmg_forest;
typedef struct gmg_partitioning gmg_partitioning;  /* handle made by gmg_partition() */
typedef struct gmg_hierarchy gmg_hierarchy;

const char *gmg_last_error(void);
int gmg_abi_version(void);

/* ------------------------------------------------------------------ forest
 * A forest of quad-/octrees over a brick of unit trees.  A cell is
 * identified by (tree, level, morton): level = distance to the root, morton =
 * the path bits from the root, d bits per level, x the fastest bit (the z-curve
 * of P:603).  Trees are ordered by the z-order of their brick
 * positions.  Refinement is isotropic into 2^d children.
 */
#define GMG_CLOSE_BALANCE 1u   /* close to 2:1 vertex balance instead of rejecting */

/* tree_xyz: host [n_trees*dim] brick coordinates (>= 0) of the trees (any order,
 *   they are re-sorted to z-order; leaf_tree indexes the z-ordered list).
 * leaf_tree / leaf_level / leaf_morton: host [n_leaves], the leaves in SFC
 *   order (tree, then Morton within the tree).
 * Errors: INVALID_ARG (dim not 2/3, n_trees < 1, duplicate tree), DEPTH,
 *   UNSORTED, NOT_TILING, UNBALANCED (unless GMG_CLOSE_BALANCE). */
gmg_status gmg_forest_create(int dim, int n_trees, const int32_t *tree_xyz, int64_t n_leaves,
                             const int32_t *leaf_tree, const int8_t *leaf_level,
                             const uint64_t *leaf_morton, uint32_t flags, gmg_forest **out);

/* Synthetic config forests (BASELINE.json configs).
 * Each pass marks the leaves satisfying the rule, refines them and closes the
 * forest to 2:1 vertex balance ("completed by a closure after each refinement
 * step").  n_passes < 0: repeat until no leaf is marked. */
typedef enum {
  GMG_RULE_NONE = 0,
  GMG_RULE_CENTER_BALL = 1,    /* |centre(T) - c| <= r                      (config 1) */
  GMG_RULE_SPHERE_SURFACE = 2, /* min_T |x-c| <= r+w  and  max_T |x-c| >= r-w (3, 5) */
  GMG_RULE_CORNER_DIST = 3     /* level(T) < lmax and dist(T, corner) <= 2^(s-level) (2, 4) */
} gmg_rule;

typedef struct {
  int dim;
  int n_trees;
  int32_t tree_xyz[8 * 3];     /* brick positions */
  int global_refinements;
  gmg_rule rule;
  int n_passes;                /* < 0: to a fixed point */
  int64_t center_num[3], center_den[3]; /* rule point c (brick units, exact rational) */
  int64_t radius_num, radius_den;       /* r */
  int64_t shell_num, shell_den;         /* w (sphere shell half-width; 0/1 = surface) */
  int64_t corner[3];           /* integer brick point for CORNER_DIST */
  int s, lmax;                 /* CORNER_DIST parameters */
} gmg_recipe;

gmg_status gmg_forest_generate(const gmg_recipe *recipe, gmg_forest **out);

/* The mesh sequences of the paper's partitioning study (Fig. 3), one
 * coarse cell read as [-1,1]^d (reading R27), each step closed to 2:1 vertex
 * balance:
 *  UNIFORM   L global refinements;
 *  CIRCLE    L times: refine every leaf whose closed box meets the disc/ball of
 *            radius 1/(4 pi) about the origin;
 *  QUADRANT  one global refinement, then L-1 times: refine every leaf inside the
 *            negative quadrant/octant [-1,0]^d;
 *  ANNULUS   L-3 global refinements, then refine the leaves whose centre lies in
 *            |x| <= 0.55, then in 0.3 <= |x| <= 0.43, then in 0.335 <= |x| <= 0.39
 *            (L >= 4).
 * Errors: INVALID_ARG (dim, kind, L out of range). */
typedef enum { GMG_SEQ_UNIFORM = 0, GMG_SEQ_CIRCLE = 1, GMG_SEQ_QUADRANT = 2, GMG_SEQ_ANNULUS = 3 } gmg_sequence;
gmg_status gmg_forest_sequence(int dim, gmg_sequence kind, int L, gmg_forest **out);
gmg_status gmg_forest_destroy(gmg_forest *f);
gmg_status gmg_forest_info(const gmg_forest *f, int *dim, int *n_trees, int64_t *n_leaves,
                           int *max_level);
/* Number of distinct Q_k nodes of the leaves (hanging and Dirichlet nodes
 * included: the "DoFs" of the configs, reading R22) without building the level
 * topology (slab-wise key counting, bounded memory) -- sizes the config-5
 * weak-scaling forests.  Errors: INVALID_ARG (k outside 1..4), DEPTH. */
gmg_status gmg_forest_count_nodes(const gmg_forest *f, int k, int64_t *n_nodes);
/* host arrays [n_leaves] (any may be NULL) */
gmg_status gmg_export_leaves(const gmg_forest *f, int32_t *leaf_tree, int8_t *leaf_level,
                             uint64_t *leaf_morton);

/* ------------------------------------------------------------------ partition
 * First-child-rule partition: the SFC-ordered leaves are cut into
 * n_ranks contiguous intervals, the first (N mod n_ranks) ranks receiving
 * ceil(N/n_ranks) leaves (R4); every other cell is owned by the owner of its
 * first child, recursively -- equivalently by the owner of the first SFC leaf
 * of its subtree.  Pure integer work, no communication.
 * Errors: INVALID_ARG when n_ranks < 1. */
gmg_status gmg_partition(const gmg_forest *f, int n_ranks, gmg_partitioning **out);
/* mode GMG_PARTITION_FIRST_CHILD: as gmg_partition.  GMG_PARTITION_PER_LEVEL: the
 * alternative the paper contrasts with (reading R29):
 * every level is partitioned on its own along the SFC, families (the 2^d children
 * of one parent; single cells on level 0) kept whole: the family starting at cell
 * index c of the N_l cells of level l goes to rank floor(n_ranks c / N_l).  Leaves
 * keep the leaf-interval owners for the leaf vectors; level owners balance every
 * level (eta ~ 1) at the price of more ghost children (transfer communication). */
#define GMG_PARTITION_FIRST_CHILD 0
#define GMG_PARTITION_PER_LEVEL 1
gmg_status gmg_partition_mode(const gmg_forest *f, int n_ranks, int mode, gmg_partitioning **out);
/* As gmg_partition_mode, and the coarse levels gathered on rank 0: every level
 * from 0 up to the last one with at most coarse_cells cells (strictly on that
 * level) is owned entirely by rank 0 ("processors drop out automatically on
 * coarser levels"); the small levels then run without exchanges and
 * the handoff is the ghost exchange of the first finer level.  0 = off
 * (gmg_partition_mode).  The model of gmg_partition_model counts the owners as
 * assigned.  Errors: INVALID_ARG. */
gmg_status gmg_partition_ex(const gmg_forest *f, int n_ranks, int mode, int64_t coarse_cells,
                            gmg_partitioning **out);
gmg_status gmg_partition_destroy(gmg_partitioning *p);

#define GMG_MAX_LEVELS 64
/* Partition-efficiency model of P:622-666 in exact integers.  N_l counts the
 * cells strictly on level l (R2).  W0_override < 0: level 0 is an ordinary
 * level (the worked example P:699-711, R3); otherwise W_0 := W0_override in
 * W_opt, W_sync and W.  eta = W_opt / W as a reduced fraction. */
typedef struct {
  int n_levels;
  int n_ranks;
  int64_t W_opt_num, W_opt_den;
  int64_t W_sync;
  int64_t W;
  int64_t eta_num, eta_den;
  int64_t N[GMG_MAX_LEVELS];
  int64_t W_l[GMG_MAX_LEVELS];
  int64_t ghost_children[GMG_MAX_LEVELS]; /* cells of level l whose owner != parent's */
  int64_t children[GMG_MAX_LEVELS];
} gmg_model;
gmg_status gmg_partition_model(const gmg_partitioning *p, int64_t W0_override, gmg_model *out);
/* N_{l,p}: host [n_levels * n_ranks], row-major by level */
gmg_status gmg_export_tallies(const gmg_partitioning *p, int64_t *N_lp);
/* Cells of level l in SFC order: Morton key of the global brick coordinates on
 * the level-l lattice, owner, leaf flag.  Size query with NULL arrays. */
gmg_status gmg_export_level_cells(const gmg_partitioning *p, int level, int64_t *n, uint64_t *key,
                                  int32_t *owner, uint8_t *is_leaf);

/* ------------------------------------------------------------------ hierarchy
 * Level spaces (notation of DESIGN.md): C_l = cells of level l,
 * D_l = their Q_k nodes, B_l = D_l on the boundary (homogeneous Dirichlet),
 * E_l = D_l \ B_l on the closure of a leaf of level < l (refinement edge),
 * S_l = the rest (smoothed).  Level vectors hold the S u E DoFs in
 * global order (owner, Morton key of the node's finest-lattice coordinates);
 * owner of a level-l node (l >= 1) = min, over the level-l cells having it as a
 * node, of the rank that computes the cell's family (the owner of the family's
 * first child = its parent's owner under the first-child rule P:604; the
 * family's rank under GMG_PARTITION_PER_LEVEL); every level-0 node is owned by
 * rank 0 (coarse handoff).  P:519-521 leaves interface ownership open; this rule
 * (reading R25) makes every owned DoF part of a family its owner computes.
 * Free leaf DoFs (non-hanging, non-Dirichlet) are numbered (owner, key) with
 * owner = the level owner at lambda(n) = max{ l : n in S_l }.
 */
#define GMG_HOST_ONLY 1u      /* integer topology only, no device data (exports, CPU tests) */
#define GMG_NO_GRAPH 2u       /* do not capture the V-cycle in a CUDA graph */
#define GMG_MIXED_PRECISION 8u /* V-cycle in fp32 (vectors, operators, smoother, transfers;
                                 P:897) inside the fp64 CG; gmg_vcycle keeps its
                                 fp64 interface (conversion at copy_to/from_mg) */
#define GMG_LOCAL_RANKS 4u    /* all n_ranks ranks live in this process (one host thread and
                                 stream each, same GPU); params.nccl_comm is a gmg_local_world */
#define GMG_RANK_LOCAL 32u    /* build only this rank's part of the level topology:
                                 no global level numbering (global exports -> GMG_E_STATE), global
                                 sizes summed over the communicator (with GMG_HOST_ONLY and
                                 n_ranks > 1 there is none: gmg_info's global sizes are -1);
                                 implies GMG_EIG_KEY */
#define GMG_EIG_KEY 64u       /* eigen start vector -5.5 + (level-lattice Morton key mod 12) on the
                                 S DoFs (reading R10b, rank-local) instead of the canonical-rank
                                 pattern of R10 */
#define GMG_HOST_RANKS 16u    /* ranks are processes joined by a gmg_host_world, passed as params.nccl_comm */

/* ------------------------------------------------------------------ communicators
 * Multi-rank runs (one rank per GPU, "processor" = MPI rank): each rank
 * calls every collective entry point (gmg_setup, gmg_vcycle, gmg_solve_cg,
 * gmg_leaf_apply, gmg_rhs_constant) with its own leaf vectors (the DoFs it
 * owns, n_owned = gmg_info.n_owned).  Ghost exchanges use grouped
 * ncclSend/ncclRecv over NVLink, CG dots one ncclAllReduce.  libnccl.so.2 is
 * loaded at run time (GMG_NCCL_LIB overrides the path).
 * gmg_nccl_get_unique_id: rank 0 creates the id (128 bytes, host), the caller
 * broadcasts it; gmg_nccl_comm_init: every rank, collective. */
gmg_status gmg_nccl_get_unique_id(char id[128]);
gmg_status gmg_nccl_comm_init(const char id[128], int n_ranks, int rank, void **comm);
gmg_status gmg_nccl_comm_destroy(void *comm);
/* Test transport: n ranks as host threads of one process on one GPU.  Each
 * thread calls the collective entry points for its rank concurrently; the
 * exchanges are host barriers plus stream-ordered device copies (no kernel
 * waits on another). */
gmg_status gmg_local_world_create(int n_ranks, void **world);
gmg_status gmg_local_world_destroy(void *world);
/* Host-staged transport for ranks that are separate processes (the multi-process
 * path on a machine with fewer GPUs than ranks, e.g. bench.py --transport host):
 * every rank calls gmg_host_world_create with the same POSIX shared-memory name
 * ("/..."), n_ranks and its rank (collective: returns once all ranks have
 * attached); slot_bytes bounds one rank's packed send data per exchange (larger
 * exchanges fail with GMG_E_OOM).  Exchanges copy device -> shared host memory ->
 * device with host barriers between; kernels never wait on each other; the
 * V-cycle is not graph-captured.  Pass the handle as params.nccl_comm with
 * GMG_HOST_RANKS.  Destroy is collective; rank 0 unlinks the segment.
 * Errors: INVALID_ARG, STATE (shm_open failed, a rank missing for 600 s), OOM. */
gmg_status gmg_host_world_create(const char *name, int n_ranks, int rank, size_t slot_bytes, void **world);
gmg_status gmg_host_world_destroy(void *world);

typedef struct {
  int k;                    /* Q_k degree, 1 or 2 */
  int cheb_degree;          /* Chebyshev degree m (R6; default 4) */
  double cheb_lo, cheb_hi;  /* eigenvalue range factors (0.08, 1.2) */
  int eig_iters;            /* CG iterations of the eigenvalue estimate (10) */
  const double *coef_level2;/* host [#level-2 cells] coefficient per level-2 cell in SFC
                               order (config 4), NULL = constant 1 */
  int rank, n_ranks;        /* this process' rank; must equal the partition's n_ranks */
  void *nccl_comm;          /* n_ranks > 1: the communicator -- an ncclComm_t
                               from gmg_nccl_comm_init, a gmg_local_world with
                               GMG_LOCAL_RANKS or a gmg_host_world with GMG_HOST_RANKS;
                               NULL for p = 1.  It
                               must outlive the hierarchy. */
  int device;               /* CUDA device ordinal; -1 = current */
  uint32_t flags;           /* GMG_HOST_ONLY | GMG_NO_GRAPH | GMG_MIXED_PRECISION | ... */
  int coarse_solver;        /* GMG_COARSE_CHOLESKY (default: dense Cholesky of A_0^S, P:331-334,
                               reading R12) or GMG_COARSE_CHEBYSHEV (reading R28) */
  /* Device allocator hooks; NULL = cudaMalloc / cudaFree.  Every
   * device buffer of the hierarchy (level vectors, index tables, scratch) is
   * obtained through dev_alloc at gmg_setup on the hierarchy's device and given
   * back through dev_free at gmg_hierarchy_destroy, both called from the calling
   * thread with stream = NULL (the legacy stream: setup synchronises).  dev_alloc
   * returns NULL on failure (-> GMG_E_OOM).  The Python binding passes the torch
   * caching allocator. */
  void *(*dev_alloc)(size_t bytes, void *stream, void *ctx);
  void (*dev_free)(void *ptr, size_t bytes, void *stream, void *ctx);
  void *alloc_ctx;
} gmg_params;

#define GMG_COARSE_CHOLESKY 0
#define GMG_COARSE_CHEBYSHEV 1

/* Fills *p with the defaults above (k = 2). */
void gmg_params_default(gmg_params *p);

/* Builds the level topology (host, integer) and, unless GMG_HOST_ONLY, uploads
 * the hierarchy to the device, computes D^{-1} on S rows, the eigenvalue
 * estimates of D^{-1} A_l^S per level and factors the coarse matrix
 * A_0^S (dense Cholesky).  Synchronises the device.
 * Errors: INVALID_ARG, STATE, ZERO_DIAG, SINGULAR_COARSE, CUDA, OOM. */
gmg_status gmg_setup(const gmg_forest *f, const gmg_partitioning *p, const gmg_params *params,
                     gmg_hierarchy **out);
gmg_status gmg_hierarchy_destroy(gmg_hierarchy *h);

typedef struct {
  int dim, k, n_levels, n_ranks, rank;
  int64_t n_leaf_nodes;      /* all leaf nodes incl. hanging and Dirichlet (R22) */
  int64_t n_leaf_free;       /* free leaf DoFs (global) */
  int64_t n_leaf_hanging, n_leaf_dirichlet;
  int64_t n_owned;           /* free leaf DoFs owned by this rank */
  int64_t first_owned;       /* global leaf index of the first owned DoF */
  int64_t level_dofs[GMG_MAX_LEVELS];  /* |S_l u E_l| (global) */
  int64_t level_cells[GMG_MAX_LEVELS];
  int64_t level_families[GMG_MAX_LEVELS];
  int64_t level_S[GMG_MAX_LEVELS], level_E[GMG_MAX_LEVELS], level_B[GMG_MAX_LEVELS];
  int64_t level_leaf_cells[GMG_MAX_LEVELS];
  int64_t mg_vector_len;     /* sum of the level vector lengths */
  /* this rank's rows the level-operator kernel finishes itself (device order R1,
   * csrc/plan.hpp: owned rows exactly one local family patch touches and no
   * other rank needs); 0 on levels without the family-tensor kernel and for
   * GMG_HOST_ONLY hierarchies */
  int64_t level_r1[GMG_MAX_LEVELS];
  /* grandfamily patches of this rank run by the 9^3-patch kernel (complete
   * grandfamilies with one coefficient, 3D Q2 tensor levels; 0 elsewhere and with
   * GMG_GFAM=0) */
  int64_t level_gf[GMG_MAX_LEVELS];
  /* levels 1..small_levels (and the coarse solve) run as one persistent kernel
   * (small_vcycle; 0 = none): one rank, family-patch levels with <= GMG_SLK_FAM
   * (2048) families each, constant coefficient, Cholesky coarse solver; opt-in
   * with GMG_SLK=1 (measured slower than the graph of per-step kernels).
   * Grandfamily patches are not formed on these levels. */
  int64_t small_levels;
} gmg_info;
gmg_status gmg_hierarchy_info(const gmg_hierarchy *h, gmg_info *out);
/* Leaf vectors of this rank: n_owned free leaf DoFs, the global
 * indices [first, first + n_owned) of the global leaf order, n_global in total.
 * Any pointer may be NULL. */
gmg_status gmg_leaf_layout(const gmg_hierarchy *h, int64_t *n_owned, int64_t *n_global, int64_t *first);

/* Level DoFs of `level` in global order: Morton key, class (0 = S, 1 = E),
 * owner, canonical index (position in the Morton order = the p = 1 numbering). */
gmg_status gmg_export_level_dofs(const gmg_hierarchy *h, int level, int64_t *n, uint64_t *key,
                                 uint8_t *cls, int32_t *owner, int64_t *canonical);
/* Free leaf DoFs in global leaf order: key, lambda, owner, canonical index. */
gmg_status gmg_export_leaf_dofs(const gmg_hierarchy *h, int64_t *n, uint64_t *key, int8_t *lambda,
                                int32_t *owner, int64_t *canonical);
/* Rank-local layout of `level` for this hierarchy's rank: owned DoFs are the
 * global range [first_owned, first_owned + n_owned); ghosts (sorted global
 * indices, host [n_ghost]) are the DoFs owned elsewhere that this rank's
 * families (children of the refined cells it owns, first-child rule) or the
 * parents of its next-finer families touch.  ghosts may be NULL. */
gmg_status gmg_export_rank_level(const gmg_hierarchy *h, int level, int64_t *first_owned, int64_t *n_owned,
                                 int64_t *n_ghost, int64_t *ghosts);
/* Rank-local layout of `level` in keys (works for GMG_RANK_LOCAL and global
 * builds alike): owned DoFs (local order = Morton key order), ghosts (sorted by
 * (owner, key)) with their owners, and the exchange plan -- peers, per-peer
 * offsets [n_peers + 1] into send_idx (local indices of owned DoFs sent to the
 * peer) and recv_idx (local indices n_owned + i of the ghosts received).  Sizes:
 * query n_owned, n_ghost, n_peers with NULL arrays first; send/recv lengths are
 * send_off[n_peers] / recv_off[n_peers].  Keys are Morton keys of
 * finest-lattice node coordinates. */
gmg_status gmg_export_local_level(const gmg_hierarchy *h, int level, int64_t *n_owned, int64_t *n_ghost,
                                  uint64_t *owned_key, uint64_t *ghost_key, int32_t *ghost_owner,
                                  int32_t *n_peers, int32_t *peers, int64_t *send_off, int64_t *recv_off,
                                  int32_t *send_idx, int32_t *recv_idx);
/* The rank's local tables of `level` before the device reordering (GMG_HOST_ONLY
 * hierarchies only, else GMG_E_STATE): cell -> local DoF [n_cells][(k+1)^d] (-1
 * Dirichlet), transfer rows [n_fam][(2k+1)^d + (k+1)^d] (fine patch in transfer-
 * owner encoding v >= 0 / -2-v / -1, then the parent's level-(l-1) local DoFs),
 * class (0 S, 1 E) and lambda flag per local DoF, eigen start vector, global
 * C_l index of every local cell.  Query n_cells, n_fam with NULL arrays. */
gmg_status gmg_export_local_tables(const gmg_hierarchy *h, int level, int64_t *n_cells, int64_t *n_fam,
                                   int32_t *cell_dofs, int32_t *xfer, uint8_t *cls, uint8_t *lam,
                                   double *eig_v, int64_t *cell_global);
/* This rank's free leaf DoFs in leaf order: finest-lattice Morton key and level
 * lambda (size query with NULL arrays).  Random inputs drawn by key do not depend
 * on the rank count (gmg_inputs.uniform_pm1_keys). */
gmg_status gmg_export_owned_leaf_keys(const gmg_hierarchy *h, int64_t *n, uint64_t *key, int8_t *lambda);
/* Cell -> level-DoF table of `level` (global index, -1 for Dirichlet nodes):
 * host [n_cells * (k+1)^d], cells in SFC order, local nodes x fastest. */
gmg_status gmg_export_cell_dofs(const gmg_hierarchy *h, int level, int64_t *n_cells,
                                int64_t *dofs);

/* ------------------------------------------------------------------ hot path
 * All vectors below are DEVICE fp64 arrays on the hierarchy's device, caller
 * owned, contiguous.  "leaf vector": length n_owned (gmg_info) in the rank's
 * global leaf order; the collective calls (gmg_vcycle, gmg_solve_cg,
 * gmg_rhs_constant, gmg_leaf_apply) are made by every rank with its own part.
 * "level vector": length level_dofs[level] in global level order -- the
 * single-operator entry points gmg_level_apply, gmg_restrict, gmg_prolongate,
 * gmg_level_smooth, gmg_level_diagonal are defined for n_ranks == 1 only
 * (GMG_E_STATE otherwise); gmg_level_apply_kernel(_f32) runs the rank-local
 * kernel of any rank. */

/* One V-cycle (P:318-327 with local smoothing P:413-469), x = V(b), x0 = 0:
 * Chebyshev-Jacobi pre/post smoothing of degree m on S rows, residual with the
 * edge matrices (E rows), restriction R = P^T, recursion, dense coarse solve,
 * prolongation.  On the levels the family-patch kernels run, the residual and
 * the restriction are one pass (each patch restricts d|_own - K_patch x; by
 * linearity the same d_{l-1} += P^T (d_l - K_l x_l) up to the order of the
 * additions), and the prolongation rides on the first post-smoothing step.
 * The copy of b into the level vectors (copy_to_mg) also forms the
 * finest level's first smoothing iterate x_1 = c2_0 D^-1 d (P:882-887 from
 * x_0 = 0): the same expression on the same values as the separate pass.
 * b and x must not alias. */
gmg_status gmg_vcycle(gmg_hierarchy *h, const double *b_dev, double *x_dev, void *cuda_stream);

/* Preconditioned CG on the leaf system (hanging nodes condensed, Dirichlet
 * removed) with one V-cycle as preconditioner, x0 = 0, stopping at the first
 * iterate with ||b - A x||_2 <= rtol ||b||_2.  Returns
 * NOT_CONVERGED (x = last iterate) when max_it is reached.  *iters and
 * *rel_res (may be NULL) are set in both cases.  Synchronises the stream once
 * per iteration (convergence check). */
gmg_status gmg_solve_cg(gmg_hierarchy *h, const double *b_dev, double *x_dev, double rtol,
                        int max_it, int *iters, double *rel_res, void *cuda_stream);

/* b_i = int_Omega f phi_i for constant f on the free leaf DoFs (the weak form
 * of P:140-147; hanging-node condensed), leaf vector.  Collective. */
gmg_status gmg_rhs_constant(gmg_hierarchy *h, double f, double *b_dev, void *cuda_stream);

/* Single-operator entry points (parity checks, ncu runs). */
/* y = K_l x over all cells of C_l on S u E rows (edge rows included): the level
 * matrix A_l of P:337-347 applied matrix-free cell by cell; on the
 * E rows this is the edge matrix -A^{ES} part of P:459-469.  p = 1 only. */
gmg_status gmg_level_apply(gmg_hierarchy *h, int level, const double *x_dev, double *y_dev,
                           void *cuda_stream);
/* The level-operator kernel alone (no memset, no exchange): y must be zero on
 * entry, y = (rank-local part of) K_l x on exit; vectors have the rank-local
 * length n_owned + n_ghost (gmg_export_rank_level).  For timing the kernel in
 * isolation (repeated calls on the same y give a meaningless y but the same
 * work per launch). */
gmg_status gmg_level_apply_kernel(gmg_hierarchy *h, int level, const double *x_dev, double *y_dev,
                                  void *cuda_stream);
/* The same kernel in fp32 (the operator of the mixed-precision V-cycle,
 * GMG_MIXED_PRECISION): x_dev, y_dev are float arrays of the rank-local length. */
gmg_status gmg_level_apply_kernel_f32(gmg_hierarchy *h, int level, const float *x_dev, float *y_dev,
                                      void *cuda_stream);
/* d_coarse += P_l^T r_fine  (level >= 1; coarse = level-1): the restriction
 * R = P^T of P:286-295, cell-wise on the families of level l.  p = 1 only. */
gmg_status gmg_restrict(gmg_hierarchy *h, int level, const double *r_fine_dev,
                        double *d_coarse_dev, void *cuda_stream);
/* x_fine += P_l x_coarse on all fine rows (level >= 1): the prolongation
 * (embedding of V_{l-1} into V_l).  p = 1 only. */
gmg_status gmg_prolongate(gmg_hierarchy *h, int level, const double *x_coarse_dev,
                          double *x_fine_dev, void *cuda_stream);
/* v = A_leaf u: the leaf-mesh operator with hanging nodes eliminated
 * (P:403-407), leaf vectors (the CG operator of P:1039-1041).  Collective. */
gmg_status gmg_leaf_apply(gmg_hierarchy *h, const double *u_dev, double *v_dev,
                          void *cuda_stream);
/* x^S = Cheb(A^S, g^S - A^{SE} x^E, x^S) on one level (x_is_zero: start from 0):
 * the Chebyshev-Jacobi smoother of P:882-887 on the local-smoothing block
 * system of P:413-426.  p = 1 only. */
gmg_status gmg_level_smooth(gmg_hierarchy *h, int level, const double *g_dev, double *x_dev,
                            int x_is_zero, void *cuda_stream);
/* diagonal of A_l^S on S rows, 0 on E rows (level vector): the Jacobi part of
 * the smoother.  p = 1 only. */
gmg_status gmg_level_diagonal(gmg_hierarchy *h, int level, double *diag_dev, void *cuda_stream);

/* lambda_bar of D^{-1} A_l^S; set overrides it (parity decoupling). */
gmg_status gmg_get_eigen(const gmg_hierarchy *h, int level, double *lambda_bar);
/* GMG_COARSE_CHEBYSHEV: the coarse Chebyshev range [lo, hi] of D^-1 A_0^S and its
 * a priori degree (0 with the Cholesky coarse solver). */
gmg_status gmg_get_coarse_chebyshev(const gmg_hierarchy *h, double *lo, double *hi, int *degree);
gmg_status gmg_set_eigen(gmg_hierarchy *h, int level, double lambda_bar);

/* Launch profiler (measurement): runs n_rep V-cycles x = V(b) eagerly
 * (no CUDA graph; same kernels and arguments as the captured cycle) with every
 * launch bracketed by CUDA events on cuda_stream, and aggregates per (kind,
 * level): number of launches, summed kernel seconds, and the kernel's
 * algorithmic bytes per launch (DESIGN.md §6 definitions: the level operator
 * counts 2 vectors per level DoF + (k+1)^d int32 per cell; the fused
 * Chebyshev kinds add the R1 rows' vectors; transfers count their vectors, the
 * family's transfer row and the coarse read-modify-write) and the same with the
 * index layout the kernel actually reads (bytes_layout).  Exchanges (GMG_K_EXCHANGE)
 * include the transport.  Writes min(count, max_out) records to out and the
 * number of distinct records to *n_out; synchronises the stream.  Collective. */
typedef enum {
  GMG_K_APPLY = 0,          /* fam_tensor_apply / cell kernels, plain y = K_l x */
  GMG_K_CHEB_X1 = 1,        /* fused operator + Chebyshev step 1 after the start from 0 */
  GMG_K_CHEB_11 = 2,        /* fused, middle steps (read and write dv) */
  GMG_K_CHEB_10 = 3,        /* fused, last step (read dv) */
  GMG_K_CHEB_01 = 4,        /* fused, first post-smoothing step without prolongation */
  GMG_K_CHEB_00 = 5,        /* fused, degree 1 */
  GMG_K_CHEB_P01 = 6,       /* fused, first post-smoothing step with x += P x_{l-1} */
  GMG_K_CHEB_STREAM = 7,    /* streaming Chebyshev rows outside R1 (cheb_range) */
  GMG_K_CHEB_STREAM_FULL = 8, /* streaming Chebyshev over a whole level (cheb_step) */
  GMG_K_RESTRICT = 9,
  GMG_K_PROLONGATE = 10,
  GMG_K_COARSE = 11,
  GMG_K_EXCHANGE = 12,
  GMG_K_COPY_MG = 13,       /* copy_to_mg / copy_from_mg */
  GMG_K_LEAF_APPLY = 14,
  GMG_K_OTHER = 15,
  GMG_K_SMALL = 16,         /* the small levels' V-cycle in one persistent kernel (small_vcycle) */
  GMG_K_RES_RESTRICT = 17   /* residual + restriction in one operator pass, d_{l-1} += P^T (d_l - K_l x_l)
                               (TA_RES; replaces APPLY + RESTRICT on 3D tensor levels, GMG_FUSE_RES=0 off) */
} gmg_kernel_kind;
typedef struct {
  int kind;                 /* gmg_kernel_kind */
  int level;                /* -1 for whole-vector kernels */
  int64_t launches;
  double seconds;           /* summed over the launches */
  double bytes;             /* algorithmic bytes per launch */
  double bytes_layout;      /* bytes per launch with the index layout actually read */
} gmg_kernel_stat;
gmg_status gmg_profile_vcycle(gmg_hierarchy *h, const double *b_dev, double *x_dev, int n_rep,
                              gmg_kernel_stat *out, int max_out, int *n_out, void *cuda_stream);

/* Kernel launches issued by the library since creation (evidence counter). */
gmg_status gmg_launch_count(const gmg_hierarchy *h, int64_t *count);
/* Launches per V-cycle (graph nodes), per CG iteration. */
gmg_status gmg_launch_profile(const gmg_hierarchy *h, int64_t *per_vcycle, int64_t *per_leaf_apply);

#ifdef __cplusplus
}
#endif
#endif /* GMG_H */
