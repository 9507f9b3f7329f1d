/*
 * sweep.h -- C ABI of the B200 (sm_100a) implementation of the decomposed multi-frontal
 * SOR / SSOR / ILU(0) sweeps of arXiv 1008.3699 (Tavakoli, "Parallelizing sequential
 * sweeping on structured grids").  Citations "PAPER:n" are line numbers of the paper's
 * text; "R-n" are the readings listed in DESIGN.md §3.
 *
 * Problem (PAPER:163-216 1D, 394-459 2D, 860-895 3D):  A u = b on a structured grid of
 * n_0 x n_1 x n_2 interior nodes (x fastest), 2d+1-point stencil
 *     (A u)_p = a_P,p u_p - sum_{q nbr of p} c_pq u_q,   a_P,p = sum_q c_pq + beta,
 * Dirichlet data folded into b (so every node outside the domain has value 0).
 * c_pq is the coefficient of the face between p and q (all 1 for SW_COEF_POISSON).
 *
 * Decomposition: the grid is cut into boxes of
 * tile[0] x tile[1] x tile[2] nodes (tile must divide n).  In sweep k box r starts at
 * the corner with start bits s_a = c_a(k mod 2^d) XOR (r_a mod 2) (bit a set = starts at
 * the max end of axis a), c = [LR, RL] (1D), [NE, SW, NW, SE] (2D), the 8-cycle
 * [(111),(000),(011),(100),(101),(010),(110),(001)] (3D) (R-4, R-5).  Direction index
 * of a box = sum_a s_a << a; omega arrays are indexed by it (1D: 0 = LR, 1 = RL;
 * 2D: 0 = SW, 1 = SE, 2 = NW, 3 = NE).
 *
 * Multi-GPU: the slowest used axis (y in 2D, z in 3D) is split into
 * contiguous slabs of whole tile rows, one per rank (one process per GPU).  Every per-node
 * array on the device carries 2 ghost layers on each side of every axis; the ghost layers of
 * the slab axis hold the neighbouring ranks' values.  With a communicator (sw_comm, passed to
 * sw_decompose) the library refreshes them itself -- "halo points ... renewed (via
 * communication) prior to a new iteration" -- by NCCL point-to-point over
 * NVLink, overlapped with the sweep of the interior tile rows, and
 * sums the PCG reductions over ranks on the device.  Without one, the caller refreshes them
 * through sw_ghost_view() and drives the staged calls.
 *
 * Conventions.  Every call returns sw_status; nothing aborts the process; on error
 * sw_last_error() returns a thread-local message.  The library owns all device memory
 * it allocates; host inputs are copied.  All work is ordered on the cudaStream_t given
 * (NULL = legacy default stream); only sw_residual_norm, sw_pcg_solve and
 * sw_check_status synchronise.  Arrays passed in are fp64, x fastest ("numpy C order
 * with shape (n2, n1, n0)").
 */
#ifndef SWEEP_H
#define SWEEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sw_grid sw_grid; /* opaque */
typedef struct sw_comm sw_comm; /* opaque: the ranks of one slab decomposition */
typedef struct CUstream_st *sw_stream_t; /* == cudaStream_t */

typedef enum {
    SW_OK = 0,
    SW_EINVAL = 1,     /* bad argument (sizes, tile, omega outside (0,2), coefficient <= 0, ...) */
    SW_ESINGULAR = 2,  /* a coupled system had |pivot| < 1e-14 or an ILU pivot D~ <= 0 */
    SW_ENOCONV = 3,    /* PCG hit maxit (outputs still valid) */
    SW_ECUDA = 4,      /* CUDA runtime error */
    SW_ENCCL = 5,      /* communicator error (NCCL, or a host transport callback returned non-zero) */
    SW_ENOMEM = 6,     /* device allocation failed */
    SW_ESTATE = 7      /* call out of order (e.g. ilu_apply before ilu0_factor) */
} sw_status;

typedef enum { SW_COEF_POISSON = 0, SW_COEF_FACES = 1 } sw_coef;
typedef enum { SW_PC_NONE = 0, SW_PC_SSOR = 1, SW_PC_ILU0 = 2, SW_PC_MG = 3 } sw_precond;
/* SYMMETRIC: P = (D~+L) D~^-1 (D~+L)^T;  PAPER: P = (D~+L) D~^-1 (D~+U), U = A_E(k0) (R-C) */
typedef enum { SW_PAIR_SYMMETRIC = 0, SW_PAIR_PAPER = 1 } sw_pairing;
typedef enum {
    SW_X = 0, SW_B = 1, SW_R = 2, SW_Z = 3, SW_P = 4, SW_Q = 5, SW_INVD = 6, SW_Y = 7,
    SW_W1 = 8, SW_W2 = 9 /* work vectors of the m-step preconditioner (multi-rank drivers) */
} sw_vector;

/* Create a grid of n[0..dim-1] GLOBAL interior nodes.  kind = SW_COEF_POISSON (unit
 * faces) or SW_COEF_FACES (coefficients supplied by sw_set_faces / sw_set_coefficients_k
 * after sw_decompose).  beta >= 0.  Selects cuda_device.  No device memory is allocated
 * until sw_decompose.  *out is NULL on error. */
sw_status sw_create_grid(int dim, const int64_t n[3], sw_coef kind, double beta, int cuda_device, sw_grid **out);

/* ---- communicators ----------------------------------------
 * NCCL: rank 0 calls sw_comm_unique_id and the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed); every rank then calls sw_comm_init_nccl (collective, blocking).  NCCL is
 * loaded at run time (the libnccl.so.2 already in the process, e.g. torch's, else the system
 * one); SW_ENCCL if none can be loaded.  One rank per GPU.
 * HOST: a transport of the caller's (tests: several processes or threads sharing one GPU, over
 * gloo or shared memory).  The library stages the layers through pinned host memory, after a
 * stream synchronisation, and calls
 *   exchange(ctx, send_lo, recv_lo, bytes_lo, send_hi, recv_hi, bytes_hi): send send_lo to rank-1
 *       and receive its layers into recv_lo, likewise with rank+1 (bytes 0: no such neighbour);
 *   allgather(ctx, send, recv, bytes): recv = the nranks send buffers in rank order;
 * each returns 0 on success (else SW_ENCCL).  Host pointers, valid only during the call.
 * A communicator may serve several grids of the same ranks (one call at a time). */
typedef int (*sw_exchange_fn)(void *ctx, const void *send_lo, void *recv_lo, size_t bytes_lo, const void *send_hi,
                              void *recv_hi, size_t bytes_hi);
typedef int (*sw_allgather_fn)(void *ctx, const void *send, void *recv, size_t bytes);
sw_status sw_comm_unique_id(unsigned char id[128]);
sw_status sw_comm_init_nccl(const unsigned char id[128], int rank, int nranks, int cuda_device, sw_comm **out);
sw_status sw_comm_init_host(int rank, int nranks, sw_exchange_fn exchange, sw_allgather_fn allgather, void *ctx,
                            sw_comm **out);
sw_status sw_comm_destroy(sw_comm *c);

/* Fix the box shape (tile[a] must divide n[a]) and this rank's slab: rank r of nranks
 * owns tile rows [r*R/nranks, (r+1)*R/nranks) of the slowest axis (R = n_slow/tile_slow,
 * nranks must divide R).  Allocates the device arrays (2 iterate buffers, b, faces, ILU
 * and PCG work vectors) for the local slab plus 2 ghost layers per side of every axis,
 * all zero.  comm: NULL for one rank, or for several ranks whose ghost layers the caller
 * refreshes (the staged calls); else a communicator of the same rank / nranks (borrowed; it
 * must outlive the grid), which makes sw_sor_sweep, sw_residual_norm, sw_ilu0_factor,
 * sw_ilu_apply, sw_ssor_apply and sw_pcg_solve multi-rank operations. */
sw_status sw_decompose(sw_grid *g, const int tile[3], int rank, int nranks, sw_comm *comm);

/* Local slab geometry: n_local[3] (x,y,z), slab offset (global index of the first local
 * node along the slab axis), padded dims pad[3] of every device array and the element
 * offset of local node (0,0,0) in it.  Device arrays are x-fastest with strides
 * (1, pad[0], pad[0]*pad[1]). */
sw_status sw_local_shape(const sw_grid *g, int64_t n_local[3], int64_t *slab_offset, int64_t pad[3],
                         int64_t *origin);

/* Copy a per-node vector in / out.  src/dst hold the LOCAL slab interior (n_local
 * nodes, x fastest); *_is_device selects host or device memory.  sw_set_vector(SW_X)
 * sets the current iterate; SW_B the right-hand side.  Ghost layers are not touched
 * (refresh them with sw_ghost_view after setting, when nranks > 1). */
sw_status sw_set_vector(sw_grid *g, sw_vector which, const double *src, int src_is_device, sw_stream_t s);
sw_status sw_get_vector(const sw_grid *g, sw_vector which, double *dst, int dst_is_device, sw_stream_t s);

/* Device pointer of the padded array `which` (the current iterate for SW_X) so callers
 * can exchange ghost layers.  Borrowed; valid until sw_destroy / the next sweep swaps
 * the iterate buffers. */
sw_status sw_ghost_view(sw_grid *g, sw_vector which, double **dev_ptr);

/* Face coefficients.  face_host[a] is the array of faces normal to axis a for the
 * local slab extended by 2 node layers on each side of the slab axis: shape n_local
 * with n_a + 1 along axis a, and n_slow_local + 4 (+1 if a is the slab axis) along the
 * slab axis; entry [c] is the face between node c - e_a and node c (c in slab-local
 * coordinates, slab axis shifted by 2).  Every face must be > 0 except those outside the
 * physical domain, which are ignored.  (PAPER:189-197, 429-448.) */
sw_status sw_set_faces(sw_grid *g, const double *const face_host[3], sw_stream_t s);

/* Assemble faces on the device from node diffusivities:
 *   face_a(p,q) = scale[a] * ((2 k_p) k_q) / (k_p + k_q).
 * k_host covers the local slab with a one-node ring on the non-slab axes (n_a + 2 nodes,
 * index 0 = coordinate -1) and two extra layers on each side of the slab axis
 * (n_slow_local + 4 layers, index 0 = coordinate -2); entries outside the physical
 * domain's node ring are ignored.  k > 0. */
sw_status sw_set_coefficients_k(sw_grid *g, const double *k_host, const double scale[3], sw_stream_t s);

/* nsweeps decomposed SOR sweeps (PAPER:326-346 1D, 524-693 2D, 860-895 3D) starting at
 * phase *phase_inout; on return *phase_inout += nsweeps.  omega holds 1 value (all
 * directions) or 2^dim values indexed by direction bits, each in (0, 2).  Each sweep
 * solves (D/Omega + A_I(k)) u+ = b + (D/Omega - D) u - A_E(k) u exactly, i.e. every box
 * is relaxed from its start corner with the coupled 2x2 / 4x4 / 8x8 systems at faces
 * where two boxes start.  Multi-rank with a communicator: before its first
 * sweep the call refreshes the 2 ghost layers of the iterate if sw_set_vector(SW_X) made them
 * stale; each sweep then runs the slab's boundary tile rows first, hands the 2 new boundary
 * layers to the neighbours on a high-priority stream (NCCL send/recv) while the interior tile
 * rows run, and waits for them before the next sweep.  The result is
 * bitwise independent of nranks.  Without a communicator and nranks > 1: nsweeps = 1 per
 * call, the caller refreshes the SW_X ghost layers before each call. */
sw_status sw_sor_sweep(sw_grid *g, const double *omega, int n_omega, int nsweeps, int64_t *phase_inout,
                       sw_stream_t s);

/* ||b - A x||_2 / ||b||_2 of the current iterate (synchronises; over all ranks with a
 * communicator, single rank otherwise). */
sw_status sw_residual_norm(sw_grid *g, double *rel_out, sw_stream_t s);

/* D-ILU(0) factor at phase k0 (R-C): D~_p = a_P,p - sum_{q implicit for p, same box}
 * c_pq^2 / D~_q, stored as 1/D~ in SW_INVD.  Tile-local (with a communicator the 1-layer
 * ghost of 1/D~ is exchanged after it).  SW_ESINGULAR (reported at the next synchronising call
 * or sw_check_status) if some D~ <= 0. */
sw_status sw_ilu0_factor(sw_grid *g, int64_t phase, sw_stream_t s);

/* z = P^-1 r for the D-ILU(0) of sw_ilu0_factor.  r_dev / z_dev are device pointers to
 * PADDED arrays of the layout reported by sw_local_shape (e.g. from sw_ghost_view);
 * Borrowed.  With a communicator the library refreshes the ghost layers of r and of the
 * intermediate arrays between the stages itself; without one and nranks > 1 use the staged
 * form below (the caller refreshes them). */
sw_status sw_ilu_apply(sw_grid *g, const double *r_dev, double *z_dev, sw_pairing pairing, sw_stream_t s);

/* Same for the SSOR / SGS preconditioner z = w(2-w)(D + w L^T)^-1 D (D + w L)^-1 r at the
 * factor phase. */
sw_status sw_ssor_apply(sw_grid *g, double omega, const double *r_dev, double *z_dev, sw_pairing pairing,
                        sw_stream_t s);

/* Number m of preconditioner steps applied by sw_ilu_apply, sw_ssor_apply and sw_pcg_solve
 * (default 1), the "few iterations of SOR ... during each step of preconditioning" of
 * z_1 = P^-1 r, z_{j+1} = z_j + P^-1 (r - theta A z_j), i.e. m
 * Richardson steps of length theta on P^-1 A from zero, scaled by 1/theta (m = 1 is P^-1 r for
 * any theta).  With the SYMMETRIC pairing the operator is symmetric, and positive definite iff
 * theta * lambda_max(P^-1 A) < 2.  The decomposed SGS / D-ILU(0) preconditioners have
 * lambda_max(P^-1 A) = 2 (the start-face pairs; DESIGN R-C), so use theta < 1 (0.5 recommended)
 * for even m.  Single rank, or multi-rank with a communicator (the staged form below applies
 * one step).  SW_EINVAL unless
 * 1 <= m <= 64 and 0 < theta <= 1. */
sw_status sw_set_precond_steps(sw_grid *g, int m, double theta);

/* Geometric multigrid preconditioner (the decomposed sweep as the smoother
 * inside multigrid).  Builds `levels` - 1 coarse grids by halving the
 * node count per axis (every level must have even counts): piecewise-constant aggregation of
 * the fine nodes of a coarse node, restriction R = P^T and the Galerkin operator R A P, which is again a
 * face-coefficient operator (coarse face = sum of the 2^(d-1) fine faces it covers, beta_c =
 * 2^d beta; DESIGN R-19).  Coarse boxes: the fine box shape, shrunk to divide the level.
 * The symmetric V-cycle (sw_mg_apply, and SW_PC_MG in sw_pcg_solve): nu Richardson steps of length
 * theta on P^-1 A from zero, P the decomposed SGS (SYMMETRIC pairing), i.e. theta times the m-step
 * operator of sw_set_precond_steps, before and after the coarse correction, which is added scaled by coarse_scale (the usual
 * over-correction of piecewise-constant interpolation; any value > 0 keeps the V-cycle symmetric
 * positive definite); on the coarsest level nu_coarse steps.  With a communicator every level is
 * decomposed over the same ranks (each level's tile rows must split evenly, else SW_EINVAL), the
 * coarse faces of the neighbours' layers are exchanged once and the cycle exchanges ghost layers
 * before every residual; without one, single rank.  SW_EINVAL for levels
 * outside [2, 16], nu outside [1, 64], nu_coarse outside [1, 1024], theta outside (0, 1],
 * coarse_scale outside (0, 4] or an odd count on a level to be coarsened.  `axes` (bit a = axis a)
 * selects the coarsened axes of every level, 0 = all: for anisotropic problems (config 5's
 * 1 : 0.1 : 0.01) semi-coarsening of the strongly coupled axes only; a coarse node then aggregates
 * 2^k fine nodes, k the number of coarsened axes, and beta_c = 2^k beta. */
sw_status sw_mg_setup(sw_grid *g, int levels, int nu, double theta, int nu_coarse, double coarse_scale, int axes);

/* z = B r, one V-cycle from zero (padded device arrays as for sw_ilu_apply; borrowed). */
sw_status sw_mg_apply(sw_grid *g, const double *r_dev, double *z_dev, sw_stream_t s);

/* Cycle index gamma of the multigrid preconditioner: 1 = V-cycle (default), 2 = W-cycle (each level
 * above the coarsest corrects twice: x_c = C r_c, then x_c += C (r_c - A_c x_c), C the level's
 * cycle).  2 C - C A_c C is symmetric, so the W-cycle stays a valid CG preconditioner whenever the
 * coarse cycle converges.  Takes effect from the next sw_mg_apply / SW_PC_MG solve.  SW_EINVAL for
 * gamma outside {1, 2}. */
sw_status sw_mg_set_cycle(sw_grid *g, int gamma);

/* Preconditioned CG from x0 = 0 on the right-hand side SW_B until ||r||/||b|| < rtol
 * (recursive residual) or maxit; result in SW_X.  precond SW_PC_ILU0 factors at phase 0
 * first.  SW_ENOCONV: iters/relres still valid.  beta = (r+.z+)/(r.z), or the flexible
 * (Polak-Ribiere) beta = z+.(r+ - r)/(r.z) that the nonsymmetric PAPER pairing needs
 * (SURVEY §8(c) C-PCG; sw_set_pcg_flexible).  alpha, beta and the stop test stay on the
 * device: one rank runs iterations 2.. as one CUDA graph with a conditional WHILE node and
 * synchronises once per solve.  With a communicator (SW_PC_NONE / SSOR / ILU0): every reduction is each rank's
 * double-double partial, all-gathered on the device and summed in rank order, so all ranks take
 * identical steps; ghost layers are exchanged inside the iteration (r and the preconditioner's
 * intermediate layers, then z, from which each rank forms the neighbours' direction values
 * itself).  Iteration counts agree with the single-rank solve to +-1.  SW_PC_MG works over ranks
 * too (sw_mg_setup with a communicator). */
sw_status sw_pcg_solve(sw_grid *g, sw_precond precond, double omega, sw_pairing pairing, double rtol, int maxit,
                       int *iters_out, double *relres_out, sw_stream_t s);

/* Which beta sw_pcg_solve uses: -1 (default) the flexible one exactly when the preconditioner is
 * ILU(0) or SSOR with SW_PAIR_PAPER, 0 always the standard one, 1 always the flexible one (one
 * extra copy of r and one extra dot product per iteration).  SW_EINVAL for other modes. */
sw_status sw_set_pcg_flexible(sw_grid *g, int mode);

/* Staged preconditioner application, for drivers that run one PCG over several ranks (the
 * sw_*_apply calls above are the single-rank composition of all stages).  Stage 0 solves the
 * forward factor (r -> the library's SW_Y array); stage 1 the backward factor (PAPER: the
 * coupled solve at the reversed corner; SYMMETRIC: the pass over nodes outside coupled sets);
 * stages 2 .. dim+1 (SYMMETRIC only) the coupled sets of degree 1 .. dim (R-C).  Between
 * stages the caller refreshes the ghost layers of the slab axis: r (1 layer) before stage 0, Y
 * (1 layer) before stage 1 for PAPER, Y (1) and z (2 layers) before every stage >= 2; 1/D~ (1)
 * once after sw_ilu0_factor.  sw_precond_stages returns the number of stages (0 on NULL). */
int sw_precond_stages(const sw_grid *g, sw_pairing pairing);
sw_status sw_ilu_apply_stage(sw_grid *g, int stage, const double *r_dev, double *z_dev, sw_pairing pairing,
                             sw_stream_t s);
sw_status sw_ssor_apply_stage(sw_grid *g, int stage, double omega, const double *r_dev, double *z_dev,
                              sw_pairing pairing, sw_stream_t s);

/* PCG vector primitives on PADDED device arrays of the local slab (layout of sw_local_shape);
 * each reduction is a fixed-order double-double sum over the local slab written as (hi, lo) to
 * the 2-double DEVICE array *_dd (a multi-rank driver sums the ranks' pairs in rank order).
 *   sw_apply_A: y = A x (ghost layers of x must be current), dot = x.y
 *   sw_dot:     dot = a.b
 *   sw_axpy2:   x += alpha p, r -= alpha q, rr = r.r
 *   sw_xpby:    p = z + beta p                                                            */
sw_status sw_apply_A(sw_grid *g, const double *x_dev, double *y_dev, double *dot_dd, sw_stream_t s);
sw_status sw_dot(sw_grid *g, const double *a_dev, const double *b_dev, double *dot_dd, sw_stream_t s);
sw_status sw_axpy2(sw_grid *g, double alpha, double *x_dev, double *r_dev, const double *p_dev, const double *q_dev,
                   double *rr_dd, sw_stream_t s);
sw_status sw_xpby(sw_grid *g, const double *z_dev, double beta, double *p_dev, sw_stream_t s);

/* out = a x + b y on the local slab's interior nodes, products and sum rounded separately (the
 * m-step preconditioner's r - theta A z and z + dz, sw_set_precond_steps, for drivers that apply
 * it over several ranks).  Device pointers to padded arrays; out may alias x or y. */
sw_status sw_axpby(sw_grid *g, double a, const double *x_dev, double b, const double *y_dev, double *out_dev,
                   sw_stream_t s);

/* ---- nine-point molecule ("extension ... for nine-point or higher
 * order central stencils is straightforward ... the size of local systems ... increased").  2D:
 * (A u)_p = a_P u_p - sum over the 8 neighbours c_pq u_q with the grid's axis faces (unit for
 * SW_COEF_POISSON) and two diagonal coefficient arrays over the cell corners c (0..n per axis,
 * x fastest, (n0 + 1) (n1 + 1) values each, GLOBAL arrays on every rank):
 *   dd[c] couples (c_x - 1, c_y - 1) and c;  da[c] couples (c_x - 1, c_y) and (c_x, c_y - 1);
 * a_P = ((W + E) + (S + N)) + ((SW + NE) + (SE + NW)) + beta.  After sw_set_diagonals the grid's
 * sw_sor_sweep is the nine-point decomposed sweep (DESIGN R-N3: a neighbour is new iff it lies on
 * the start side of the node's box along every axis where they differ; the coupled set at a start
 * corner becomes a dense 4 x 4); boxes of at most 64 x 64; multi-rank as the five-point sweep.  The
 * preconditioner, residual and PCG calls stay five-point only (SW_ESTATE on such a grid).
 * SW_EINVAL for dim != 2 or a negative / non-finite coefficient. */
sw_status sw_set_diagonals(sw_grid *g, const double *dd_host, const double *da_host, sw_stream_t s);

/* ---- eikonal equation |grad u| = f by decomposed fast sweeping (PAPER:2593-2599
 * names the application, its supplementary paper is not available).  2D, boxes of at most 64 x 64,
 * any number of ranks (the same slab decomposition and communicator as the SOR sweep).  The local
 * update is the Godunov upwind rule of fast sweeping (Zhao 2005; DESIGN R-E1):
 *   a = min(u_W, u_E), b = min(u_S, u_N) (+inf outside the domain), fh = f_p h,
 *   ubar = min(a,b) + fh if |a - b| >= fh, else ((a + b) + sqrt(2 fh^2 - (a - b)^2)) / 2,
 *   u_p <- min(u_p, ubar);
 * each box sweeps from its start corner on the SOR schedule (new values on the start side, old on
 * the end side, R-E2), the coupled nodes at start-start faces (pairs, the 4-node corner) solved
 * exactly by ordered fixing (R-E3).  The iterate is SW_X: set it with sw_set_vector (+inf
 * everywhere, 0 at the sources) before the first sweep; sources keep 0.
 * sw_set_slowness: f over the local slab (x fastest), finite and > 0 (SW_EINVAL otherwise), grid
 *   spacing h > 0; copied (host pointer); with a communicator the 2 ghost layers are exchanged.
 * sw_eikonal_sweep: nsweeps passes from phase *phase_inout (then += nsweeps).
 * sw_eikonal_changes: number of nodes (over all ranks with a communicator) the last pass changed
 *   (0 = converged: the discrete viscosity solution); synchronises. */
sw_status sw_set_slowness(sw_grid *g, const double *f_host, double h, sw_stream_t s);
sw_status sw_eikonal_sweep(sw_grid *g, int nsweeps, int64_t *phase_inout, sw_stream_t s);
sw_status sw_eikonal_changes(sw_grid *g, int64_t *changed_out, sw_stream_t s);

/* Synchronise `s` and report a deferred device-side error (singular coupled system). */
sw_status sw_check_status(sw_grid *g, sw_stream_t s);

/* Number of kernel launches this grid has issued (for the bench's gpu_launches). */
int64_t sw_launch_count(const sw_grid *g);

sw_status sw_destroy(sw_grid *g);
const char *sw_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
