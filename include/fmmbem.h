/* fmmbem.h -- C ABI of the B200-native FMM-BEM hot path (arXiv 1007.4591).
 *
 * Pure C: no CUDA, NCCL or PyTorch types appear here.  Device pointers are plain
 * `float*`/`double*` in CUDA device memory of the ctx's device; streams are passed
 * as `void*` (a cudaStream_t, NULL = the legacy default stream).
 *
 * The user's problem (Sec. 2.1): given a closed triangulated
 * dielectric boundary Omega, interior point charges (q_i, r_i) and eps_I, eps_II,
 * compute the induced surface charge sigma of the second-kind integral equation
 * (Eq. 4) and the solvation energy dG = 1/2 sum q_i phi_reac(r_i)
 * (Eq. 5-6), either exactly (GMRES on A x = B q) or by the
 * BIBEE diagonal approximation (Eq. 7).  Discretisation: flat panels,
 * piecewise-constant sigma, K-point quadrature (K = 1 = the paper's centroid rule,
 * P:409-411).  Readings of the paper are listed in DESIGN.md (A1-A22).
 *
 * Ownership: fmmbem_create deep-copies every host input (the caller may free them on
 * return).  The ctx owns all of its device memory.  All output buffers are caller-owned.
 * Errors: every call returns fmmbem_status; nothing throws across the ABI; on a
 * negative status no output has been written ("no partial outputs") and
 * fmmbem_last_error() names the offending index.  A ctx is not thread-safe.
 * Ordering: fmmbem_matvec is stream-ordered on the caller's stream; every other call that touches
 * the device is BLOCKING (it returns when its results are written) and runs on the ctx's internal
 * stream.  Every call -- matvec included -- first waits (on the device) for the work of the previous
 * call on this ctx, whatever stream that ran on, because all calls share the ctx's expansion and
 * staging buffers.  Device buffers passed to a blocking call must not be in use by pending work on
 * other streams (the Python binding synchronises the caller's current stream before such calls).
 * Units: Angstrom and elementary charges; energies in internal units (kernels with the
 * explicit 1/(4 pi) of Eq. 4-5) and in kcal/mol = internal * 4 pi * 332.0637.
 */
#ifndef FMMBEM_H
#define FMMBEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMMBEM_ABI_VERSION 3  /* 3: options.charge_terms, tree_info expansion slots / LET counts, plan lists 10-14 */

typedef struct fmmbem_ctx fmmbem_ctx; /* opaque */

typedef enum {
  FMMBEM_OK = 0,
  FMMBEM_NOT_CONVERGED = 1,  /* solve: outputs hold the best iterate */
  FMMBEM_E_INVALID = -1,     /* null/size/NaN input, eps <= 0, eps_in == eps_out, bad options */
  FMMBEM_E_DEGENERATE = -2,  /* triangle index out of range or area < 1e-14*bbox_diag^2 */
  FMMBEM_E_COINCIDENT = -3,  /* charge on a panel point, duplicate centroids */
  FMMBEM_E_CUDA = -4,
  FMMBEM_E_NOMEM = -5,
  FMMBEM_E_NCCL = -6
} fmmbem_status;

/* Surface mesh: n_vertices x 3 doubles (Angstrom), n_triangles x 3 int32 vertex indices,
 * 0-based, outward winding (normal = cross(v1-v0, v2-v0) points into region II). */
typedef struct {
  int64_t n_vertices;
  const double* xyz;
  int64_t n_triangles;
  const int32_t* tri;
} fmmbem_mesh;

/* Point charges: n x 3 positions (Angstrom) and n charges (e); n may be 0. */
typedef struct {
  int64_t n;
  const double* xyz;
  const double* q;
} fmmbem_charges;

typedef struct {
  int32_t struct_size;   /* = sizeof(fmmbem_options) */
  int32_t terms;         /* P = number of expansion terms, degrees 0..P-1 (A9); 2..16, default 10 */
  int32_t leaf_points;   /* depth rule: mean panels per occupied leaf <= leaf_points (A10); default 64 */
  int32_t quad_points;   /* K in {1 (paper), 3, 6, 7}; default 1 */
  int32_t near_mode;     /* 0 = K-point quadrature only (paper); 1 = exact flat-panel integrals (closed form,
                            P:415-418) for pairs |c_i - c_j| < near_radius*sqrt(A_j) and the single-layer
                            self term; default 0 */
  float near_radius;     /* eta of the near criterion; default 3; eta*sqrt(A) must stay below the leaf width */
  int32_t self_term;     /* 0: K'_ii = 0 (flat panel); 1: curvature term
                            K'_ii = -H_i sqrt(A_i/pi)/4, H_i from area-weighted vertex normals
                            (computed on the host at create, FP64) */
  int32_t direct;        /* 1 = bypass the FMM: all-pairs P2P (paper Fig. 11 "direct") */
  int32_t deterministic; /* reductions have a fixed order (no atomics on results); always true */
  int32_t device;        /* CUDA ordinal used by this ctx */
  int32_t rank, nranks;  /* one process per GPU, nranks <= 64; every rank passes ALL charges */
  const void* nccl_id;   /* nranks > 1: the 128-byte id from fmmbem_get_unique_id() on rank 0, broadcast by the caller */
  int32_t input_mode;    /* nranks > 1 only.  0: every rank passes the FULL mesh (rank r prepares triangles
                            [r n/R, (r+1) n/R), global id = triangle index).  1: every rank passes only ITS
                            part of the mesh (its own vertex array; triangles index it); the global id of rank
                            r's triangle k is k + (triangles of ranks < r) -- memory O(N/R) per rank (SURVEY
                            8(e)); near_mode and self_term need mode 0.  Either way the panels move to the rank
                            owning their leaf; default 0 */
  int32_t charge_terms;  /* expansion order of the charge-FMM (E_n and psi from the charges; the
                            BIBEE energy and the GMRES right-hand side): 0 = terms (default); else one of the
                            rotation orders 8, 10, 12, 13, 14 and <= terms.  The charges sit >= 1.4 A inside the
                            surface, so their fields converge faster in P than a random-x K' product; the
                            bench's parity rows report the E_n / psi error at the order used */
} fmmbem_options;

/* FMMBEM_ABI_VERSION of the built library; sizes of the ABI structs (bindings check these). */
int32_t fmmbem_abi_version(void);
int64_t fmmbem_struct_size(const char* name); /* "options", "timing", "energy", "tree_info", "solve_options"; -1 if unknown */

/* Fill *out with the defaults above.  Returns FMMBEM_E_INVALID if out is NULL. */
fmmbem_status fmmbem_default_options(fmmbem_options* out);

/* Multi-GPU bootstrap: writes a 128-byte NCCL unique id into id128_out (host).
 * Call on rank 0 only and broadcast the bytes (e.g. torch.distributed) before fmmbem_create.
 * Returns FMMBEM_E_NCCL when libnccl.so.2 cannot be loaded. */
fmmbem_status fmmbem_get_unique_id(void* id128_out);

/* Domain decomposition helper (cost-weighted): split n items with non-negative
 * host costs into `parts` contiguous ranges of nearly equal total cost.  bounds (host, parts+1
 * entries) receives 0 = bounds[0] <= ... <= bounds[parts] = n.  Pure host code; the library uses
 * it on the leaves' P2P + M2L costs so that every rank derives the same partition. */
fmmbem_status fmmbem_split_costs(const double* costs, int64_t n, int32_t parts, int64_t* bounds);

/* Build the solver for one molecule (setup): validates and
 * deep-copies the inputs, derives panels and quadrature points (FP64, P:368-378,
 * P:409-411), builds the Morton-sorted uniform-depth octree, its neighbour and
 * interaction lists on the device.  opt may be NULL (defaults).
 * On success *out receives a new ctx; on failure *out is set to NULL. */
fmmbem_status fmmbem_create(const fmmbem_mesh* panels, const fmmbem_charges* charges,
                            double eps_in, double eps_out, const fmmbem_options* opt,
                            fmmbem_ctx** out);

/* Release every resource of ctx.  NULL-safe. */
void fmmbem_destroy(fmmbem_ctx* ctx);

/* Vectors passed to matvec/solve/bibee are in the library's LOCAL order (the octree's
 * Morton order) and, with nranks > 1, hold only this rank's panels (a contiguous range of
 * Morton-ordered leaves of equal estimated work).  fmmbem_local_panel_ids writes, for local
 * index i, the panel's GLOBAL id (host int64 array of fmmbem_num_local_panels entries): the caller's
 * triangle index (one rank, input_mode 0) or the id defined by input_mode 1. */
int64_t fmmbem_num_local_panels(const fmmbem_ctx* ctx);
fmmbem_status fmmbem_local_panel_ids(const fmmbem_ctx* ctx, int64_t* global_ids_out);

typedef enum {
  FMMBEM_OP_KPRIME = 0, /* y_i = sum_{j!=i} A_j x_j sum_g w_g dG/dn_i(c_i, y_jg)   (Eq. 4 operator) */
  FMMBEM_OP_SINGLE = 1, /* y_i = sum_{j!=i} A_j x_j sum_g w_g G(c_i, y_jg)         (Eq. 5, 1/r)     */
  FMMBEM_OP_A = 2,      /* y = x - f * KPRIME(x), f = 2(eps_II-eps_I)/(eps_I+eps_II) (GMRES operator, A1) */
  FMMBEM_OP_DOUBLE = 3  /* y_i = sum_{j!=i} A_j x_j sum_g w_g dG/dn_y(c_i, y_jg), n_y = n_j: the double layer K,
                           adjoint of KPRIME (dipole sources; not with near_mode) */
} fmmbem_op;

/* One FMM matrix-vector product.  x_dev, y_dev: caller-owned device
 * arrays of fmmbem_num_local_panels floats in local order; must not alias.  Stream-ordered:
 * returns after enqueueing on cuda_stream; y is valid when the stream completes.  With nranks > 1
 * the call is collective (all ranks, same order): x slices are all-gathered and the multipoles
 * each rank's interaction lists need are exchanged over NCCL (local essential tree). */
fmmbem_status fmmbem_matvec(fmmbem_ctx* ctx, fmmbem_op op, const float* x_dev, float* y_dev,
                            void* cuda_stream);

/* Same product with HOST buffers (pinned or pageable; pinned lets the transfers overlap):
 * x_host / y_host hold the rank's n_local values in local order.  Single GPU: x is copied in
 * Morton-contiguous chunks on an internal copy stream while P2M starts on the chunks that have
 * landed, and y leaves in chunks as P2P finishes them (same result as fmmbem_matvec up to the
 * rounding of the near + far addition).  nranks > 1: copy in, fmmbem_matvec, copy out.  Blocks
 * until y_host is written.  Errors as fmmbem_matvec. */
fmmbem_status fmmbem_matvec_host(fmmbem_ctx* ctx, fmmbem_op op, const float* x_host, float* y_host);

typedef struct {
  double tol;           /* relative residual ||b - A x|| / ||b||, default 1e-6 (A12) */
  int32_t restart;      /* GMRES(m) restart length, default 30 */
  int32_t max_iters;    /* default 200 */
  const float* x0_dev;  /* initial guess (device, local order) or NULL = zero */
} fmmbem_solve_options;

typedef struct {
  double dG_internal;   /* 1/2 sum_j A_j sigma_j psi_j (= 1/2 q^T C sigma, A20) */
  double dG_kcal_mol;   /* dG_internal * 4 pi * 332.0637 (A13) */
  int32_t iterations;   /* GMRES iterations (0 for BIBEE) */
  double rel_residual;  /* final GMRES relative residual estimate (0 for BIBEE) */
} fmmbem_energy;

/* Full BEM solve: E_n and psi by one charge-FMM, then GMRES on
 * (I - f K') sigma = f E_n, then dG.  sigma_dev (nullable): n_local floats; residual_hist
 * (nullable, host): max_iters+1 doubles, unused entries set to -1.  Returns FMMBEM_OK or
 * FMMBEM_NOT_CONVERGED (best iterate written). */
fmmbem_status fmmbem_solve(fmmbem_ctx* ctx, const fmmbem_solve_options* opt, float* sigma_dev,
                           double* residual_hist, fmmbem_energy* out);

typedef enum {
  FMMBEM_BIBEE_CFA = 0, /* s = -1/2 (Eq. 7) */
  FMMBEM_BIBEE_P = 1,   /* s = 0 */
  FMMBEM_BIBEE_LB = 2   /* s = +1/2 */
} fmmbem_bibee;

/* BIBEE energy: sigma_hat = f E_n / (1 - f s), dG = 1/2 sum A sigma_hat psi.
 * sigma_hat_dev nullable (n_local floats). */
fmmbem_status fmmbem_bibee_energy(fmmbem_ctx* ctx, fmmbem_bibee variant, float* sigma_hat_dev,
                                  fmmbem_energy* out);

/* Drop the cached E_n / psi of the charge-FMM, so that the next bibee / solve / charge_fields call
 * recomputes them (benchmarks of the uncached BIBEE energy).  Host only; never fails on a valid ctx. */
fmmbem_status fmmbem_reset_fields(fmmbem_ctx* ctx);

/* Diagnostics: E_n (with 1/eps_I) and psi_j = sum_g w_g sum_k q_k G(y_jg, r_k) at the panels
 * (device, local order; either may be NULL). */
fmmbem_status fmmbem_charge_fields(fmmbem_ctx* ctx, float* En_dev, float* psi_dev);

/* Reaction potential phi_reac(r_k) = sum_j sigma_j A_j sum_g w_g G(r_k, y_jg) at every charge
 * (Eq. 5), written to a host array of n_charges doubles in the caller's charge order. */
fmmbem_status fmmbem_reaction_potential(fmmbem_ctx* ctx, const float* sigma_dev, double* phi_host);

typedef struct {
  double tree, upward, m2l, p2p, l2p, near, comm, gmres, total; /* ms: tree = octree build at
                             create (keys, sort, levels, lists, point placement; host clock); the rest = the last
                             matvec (CUDA events on the stream each phase ran on): upward = P2M + M2M, m2l = M2L,
                             l2p = L2L + L2P, comm = NCCL exchanges, total = the whole product; gmres = last solve */
  int64_t p2p_interactions; /* exact pair count of the last matvec's P2P */
  int64_t m2l_pairs;        /* M2L translations of the last matvec */
  double p2m, m2m, l2l, leaf_l2p; /* ms, the last matvec: upward = p2m + m2m, l2p = l2l + leaf_l2p */
  double bibee;             /* ms of the last fmmbem_bibee_energy (charge-FMM if not cached + reduction; CUDA events) */
} fmmbem_timing;

fmmbem_status fmmbem_last_timing(const fmmbem_ctx* ctx, fmmbem_timing* out);

/* Tree statistics for tests / reporting. */
typedef struct {
  int32_t levels;       /* leaf level L (root = 0) */
  int64_t n_leaves;
  int64_t n_cells;      /* all levels */
  int64_t n_panels, n_charges;
  int64_t nbr_pairs;    /* leaf neighbour-list entries (incl. self) */
  int64_t m2l_pairs;    /* interaction-list entries over all levels */
  double root_width;    /* root cube width (Angstrom) */
  double root_origin[3];
  int64_t expansion_slots; /* cells with multipole / local storage on this rank: n_cells on one GPU; the
                              rank's windows + received LET cells with nranks > 1 (FMMBEM_PLAN_CELL_WINDOWS) */
  int32_t let_send_peers, let_recv_peers; /* nranks > 1: peers this rank sends / receives panel multipoles */
  int64_t let_cells_sent, let_cells_recv, let_shared_cells; /* per K' matvec (panel LET lists) */
  int64_t halo_panels_sent, halo_panels_recv;               /* near-field halo weights per matvec */
} fmmbem_tree_info;

fmmbem_status fmmbem_tree_info_get(const fmmbem_ctx* ctx, fmmbem_tree_info* out);

/* The multi-GPU exchange plan of a leaf skeleton, computed on the HOST by the same
 * code fmmbem_create runs on every rank: the cost-weighted contiguous leaf partition, the
 * near-field halo (leaves whose panels a peer's P2P needs) and the local essential tree (pure cells
 * whose multipoles a peer's M2L needs; cells straddling ranks, summed by all-reduce).  For
 * tests and tooling; no GPU is used.  leaf_keys: n_leaves sorted unique Morton keys at `level`
 * (x least significant); leaf_panels / leaf_charges (nullable): points per leaf of ALL ranks;
 * quad_points = K.  Lists are read with fmmbem_plan_list: returns the count and, if out is non-NULL,
 * writes the entries (int64).  Leaves are leaf indices; cells are level-major global cell indices
 * (FMMBEM_PLAN_CELL_KEYS / _LEVEL_OFFSETS give the cell numbering). */
typedef struct fmmbem_plan fmmbem_plan;
enum {
  FMMBEM_PLAN_HALO_SEND = 0,   /* peer: my leaves whose panels peer needs */
  FMMBEM_PLAN_HALO_RECV = 1,   /* peer: peer's leaves whose panels I need */
  FMMBEM_PLAN_LET_SEND = 2,    /* peer: my pure cells whose multipoles peer needs */
  FMMBEM_PLAN_LET_RECV = 3,    /* peer: peer's pure cells I need */
  FMMBEM_PLAN_LET_SHARED = 4,  /* cells straddling ranks (peer ignored) */
  FMMBEM_PLAN_LEAF_BOUNDS = 5, /* nranks + 1 leaf bounds */
  FMMBEM_PLAN_CELL_KEYS = 6,   /* every cell's key, level-major */
  FMMBEM_PLAN_LEVEL_OFFSETS = 7, /* level + 2 offsets into the cell numbering */
  FMMBEM_PLAN_NEIGHBOURS = 8,   /* `peer` = a leaf index: its neighbour leaves (incl. itself) */
  FMMBEM_PLAN_INTERACTION = 9,  /* `peer` = a cell index (level >= 2): its interaction list */
  FMMBEM_PLAN_LET_SEND_CHG = 10,   /* peer: my pure cells whose CHARGE multipoles peer's panels need */
  FMMBEM_PLAN_LET_RECV_CHG = 11,   /* peer: peer's pure cells whose charge multipoles I need */
  FMMBEM_PLAN_LET_SHARED_CHG = 12, /* cells with charges straddling ranks (peer ignored) */
  FMMBEM_PLAN_CELL_WINDOWS = 13,   /* 2 (level + 1) entries: per level l the cells [lo, hi) holding a
                                      leaf of this rank -- its expansion slots, in that order */
  FMMBEM_PLAN_EXTRA_CELLS = 14     /* received / shared LET cells outside the windows: the slots
                                      after the windows' (increasing) */
};
fmmbem_status fmmbem_plan_create(const uint64_t* leaf_keys, const int32_t* leaf_panels, const int32_t* leaf_charges,
                                 int64_t n_leaves, int32_t level, int32_t quad_points, int32_t nranks, int32_t rank,
                                 fmmbem_plan** out);
void fmmbem_plan_destroy(fmmbem_plan* plan);  /* NULL-safe */
int64_t fmmbem_plan_list(const fmmbem_plan* plan, int32_t list, int32_t peer, int64_t* out); /* -1: bad list / peer */

/* Thread-local message describing the last error (never NULL). */
const char* fmmbem_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FMMBEM_H */
