/*
 * pgrid.h -- C ABI of the B200-native topology-based power-grid transient
 * solver (arxiv 1409.7166, "An Efficient Topology-Based Algorithm for Transient
 * Analysis of Power Grid"; PAPER.md).  Library: paper_1409_7166_b200/lib/libpgb200.so
 *
 * Method (§II-A Eq. (2) and §IV Eqs. (12)-(15), Algorithm 1): at every
 * backward-Euler step solve (C/h + G + hL) x(t+h) = rhs directly on the netlist
 * graph by nodal relaxation -- never assembling G.  Each node is updated from
 * its neighbours' voltages, branch conductances, pad conductance to Vdd,
 * capacitor history C_i/h x_i(t) and its PWL current load (Eq. (13)), with SOR
 * relaxation omega (Eq. (15)).  Inductors use the backward-Euler companion
 * model (Eq. (10)): conductance h/L (series R-L: 1/(R + L/h)) plus a history
 * current updated after every step.
 *
 * Conventions (all entry points):
 *  - Return 0 (PG_OK) on success or a negative PG_E* code; pg_last_error()
 *    then returns a thread-local, NUL-terminated description.  No entry point
 *    aborts the process; on error the grid object is left unchanged (create
 *    functions set *out = NULL).
 *  - `mem` says where caller buffers live: PG_MEM_HOST (pageable or pinned host
 *    memory) or PG_MEM_DEVICE (CUDA device memory of the current device).
 *    Inputs are COPIED into library-owned device memory; the caller keeps
 *    ownership of every buffer it passes and may free it after the call.
 *  - Node index of a mesh node (layer l, row y, column x) is
 *    (l * ny + y) * nx + x ("natural layout"); layer 0 is the bottom (device)
 *    layer, layer `layers-1` the top (pad) layer.
 *  - All values are SI: siemens, farads, henries, amperes, volts, seconds.
 *  - Work is enqueued on the grid's stream (pg_set_stream; default: the legacy
 *    default stream) and every entry point returns after its results are
 *    complete in the caller's buffers.
 *  - A pg_grid is not thread-safe; distinct grids may be used concurrently.
 */
#ifndef PGRID_H
#define PGRID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_API __attribute__((visibility("default")))

typedef struct pg_grid pg_grid;

enum { PG_MEM_HOST = 0, PG_MEM_DEVICE = 1 };

enum {
  PG_OK = 0,
  PG_EINVAL = -1,    /* bad argument (sizes, indices, nonpositive values, omega outside (0,2)) */
  PG_ECUDA = -2,     /* CUDA runtime / launch error (message carries cudaGetErrorString) */
  PG_ENOCONV = -3,   /* a time step hit max_sweeps without meeting tol (results still written) */
  PG_ENOMEM = -4,    /* device allocation failed */
  PG_ESTATE = -5,    /* call not valid for this grid (e.g. RLC data on a CSR grid) */
  PG_ENONFINITE = -6 /* an iterate became NaN / Inf (e.g. from non-finite device inputs); results invalid */
};

enum {
  PG_METHOD_RBSOR = 0,  /* red-black ordered Gauss-Seidel / SOR (Eq. (13)+(15) in red-black numbering) */
  PG_METHOD_JACOBI = 1  /* weighted Jacobi (comparison baseline) */
};

/* Layered-mesh grid (structure-of-arrays store).  PAPER.md §II-A: "C is a
 * diagonal matrix whose (i,i) element is the capacitance between node i and
 * ground ... G0 is ... the conductance between node i and source"; Fig. 2
 * node model (R and L branches to neighbours).
 *   gx[n]  conductance (S) of the in-layer segment (l,y,x)-(l,y,x+1); entries
 *          with x = nx-1 must be 0.  >= 0.
 *   gy[n]  conductance of (l,y,x)-(l,y+1,x); entries with y = ny-1 must be 0.
 *   gz[n]  conductance 1/R of the via (l,y,x)-(l+1,y,x); layer layers-1 must be 0.
 *   lz[n]  via series inductance (H, >= 0) or NULL (RC grid).  A via with
 *          lz > 0 is a series R-L branch (R = 1/gz).
 *   cap[n] node-to-ground capacitance (F, >= 0).
 *   pad_node[n_pads], pad_g[n_pads]: pad branches from node to the Vdd source
 *          node, conductance 1/R (> 0); pad_l[n_pads] series inductance or NULL.
 *          A node may carry several pads.
 *   n = layers * ny * nx.  1 <= layers <= 256, ny, nx >= 1.  Meshes of up to
 *   8 layers are swept by the streaming strip kernels; taller stacks by the
 *   per-colour sweep (option "colour"; no slab groups).
 * Every node must have a path to a pad (Lemma 1 / topological assumption 3);
 * this is not checked here (an isolated node without capacitance makes the
 * diagonal zero and is reported as PG_EINVAL by pg_transient).            */
PG_API int pg_create_mesh(int32_t layers, int32_t ny, int32_t nx,
                          const double *gx, const double *gy, const double *gz,
                          const double *lz, const double *cap, int64_t n_pads,
                          const int64_t *pad_node, const double *pad_g,
                          const double *pad_l, double vdd, int mem, pg_grid **out);

/* Irregular RC grid given as a branch list (CSR store built natively:
 * parallel branches kept, self-loops and zero-conductance branches dropped,
 * nodes 2-coloured by BFS parity when the graph is bipartite, greedily
 * multi-coloured otherwise; the sweep visits the colours in order -- Eq. (13)
 * under that numbering).  Bipartite graphs are built on the device;
 * other graphs (and every graph when the environment variable
 * PGB200_CSR_HOST is set) by the host builder, which gives the same store.
 * Invalid branches (endpoint outside [0, n), conductance negative or not
 * finite; pg_last_error() names the first such branch) or capacitances
 * (negative or not finite) return PG_EINVAL.
 *   bu[m], bv[m]: branch end nodes in [0, n); bg[m]: conductance (>= 0).
 *   cap[n], pads as in pg_create_mesh (RC pads only).  n >= 1.          */
PG_API int pg_create_csr(int64_t n, int64_t m, const int64_t *bu, const int64_t *bv,
                         const double *bg, const double *cap, int64_t n_pads,
                         const int64_t *pad_node, const double *pad_g, double vdd,
                         int mem, pg_grid **out);

/* PWL current loads (§II-A "modeled as piecewise linear ideal current
 * sources"; load convention: current drawn from the node to ground).  Source k
 * sits on node[k] with breakpoints t[ptr[k]..ptr[k+1]) (strictly increasing,
 * seconds) and values i[...] (A); linear between breakpoints, first/last value
 * held outside.  ptr has n_src+1 entries, ptr[0] = 0, every source >= 1 point.
 * Replaces any previous set.  n_src = 0 clears the loads.                    */
PG_API int pg_set_sources(pg_grid *g, int64_t n_src, const int64_t *node,
                          const int64_t *ptr, const double *t, const double *i, int mem);

/* Initial condition x(0) (n values; Algorithm 1 input "initial capacitor
 * voltages").  Default after create: every node at vdd, inductor currents 0
 * (the exact DC operating point of an unloaded grid).  Inductor currents are
 * reset to 0 by this call.  The values (host or device memory) are checked on
 * the device first: a NaN or infinite value returns PG_EINVAL and leaves the
 * grid's state unchanged.                                                   */
PG_API int pg_set_voltages(pg_grid *g, const double *v, int mem);

/* Voltages after the last completed pg_transient step (or x(0)); n values. */
PG_API int pg_get_voltages(pg_grid *g, double *v, int mem);

/* Enqueue all work of this grid on `stream` (a cudaStream_t, may be NULL). */
PG_API int pg_set_stream(pg_grid *g, void *stream);

/* Tuning knobs (key, value); unknown keys -> PG_EINVAL.
 *   "fuse"   F, sweeps fused per launch of the temporally blocked mesh sweep,
 *            1..4, or 0 (default: 2); Jacobi and CSR sweeps run 1 per launch
 *   "lag"    wavefront lag D (rows) between fused sweep levels: 3 (default) or 4
 *   "batch"  sweep launches enqueued between host convergence polls, >= 1
 *   "resident" 1 (default): red-black SOR on a single mesh that fits one
 *            thread-block cluster (<= 16 CTAs x 512 threads, one thread per
 *            (layer, row, column pair): L * ceil(NX/2) <= 512 and
 *            ceil(NY / floor(512 / (L * ceil(NX/2)))) <= 16, e.g. 2 x 64 x 64)
 *            runs all sweeps of a time step in one cluster launch with V in
 *            shared memory (convergence tested after every sweep, so
 *            pg_stats.sweeps_per_launch = 1); 0: the streaming sweep
 *   "pipe"   1 (default): full launches of F = 2 mesh sweeps run the
 *            warp-specialised two-level pipeline kernel (k_rb_sweep2); 0: the
 *            generic temporally blocked kernel for every F (same results)
 *   "pdl"    0 (default): off; 1: consecutive sweep launches of a single
 *            grid use programmatic dependent launch (the next launch's
 *            prologue and constant-row loads overlap the previous launch's
 *            tail; mesh pipeline kernel and the staged CSR colour launches,
 *            whose first tiles' bulk copies are then requested before the
 *            dependency wait) -- same results, measured slower on configs
 *            1, 2 and 4
 *   "l2keep" / "l2first" L2 eviction policy of the pipeline kernel, 6-bit
 *            masks over (gx, gy, gz_eff, b, 1/d, V): l2keep bits 0-4 read that
 *            constant array with evict_last, bit 5 writes V with evict_last;
 *            l2first reads the arrays (bit 5: V) with evict_first; others
 *            evict_normal.  -1 (default, auto): meshes with a per-launch
 *            footprint (56 B per element) below twice the L2 use l2keep = 32,
 *            l2first = 63 (stream the reads, keep the freshly written V for
 *            the next launch), larger meshes 0 / 0
 *   "l2promo" L2 promotion of the sweep's TMA loads in bytes: 0, 64, 128,
 *            256 (default 128: +0.6-1.3 % over 256 on configs 1, 3, 4,
 *            profiles/r2_l2promo_ab.txt)
 *   "graph"  1 (default): replay full batches of sweep launches from a captured
 *            CUDA graph (single grids, and slab groups whose exchange is
 *            capturable or fused into the sweep); 0: plain launches
 *   "rows"   rows per CTA of the mesh sweep (0: auto)
 *   "width"  column pairs per strip of the mesh sweep: 32 (one warp per layer
 *            row) or 64 (two warps; halves the x-halo share, needs 2x shared
 *            memory); 0 = auto
 *   "stages" shared-memory ring stages S of the mesh sweep (0: auto =
 *            D (F-1) + 6); a (F, S, D) variant that is not compiled falls
 *            back to the default S, then to smaller F
 *   "colour" 1: mesh sweeps run colour by colour, two launches of
 *            k_rb_colour_mesh per sweep (one thread per node of the colour;
 *            same iterates as the streaming sweep bit for bit,
 *            pg_stats.sweeps_per_launch = 1); 0 (default): only meshes taller
 *            than 8 layers use it
 *   "csr_stage" 1 (default): CSR grids run the staged multi-colour sweep
 *            (k_csr_sweep_staged: every 256-row tile's row pointers, b, 1/d,
 *            columns and values bulk-copied into shared memory, one stage per
 *            CTA, 8 CTAs per SM) when every tile fits its stage (at most
 *            1536 entries per 256 rows of one colour); 0, or a tile that does
 *            not fit: one thread per row (k_csr_sweep), same iterates bit
 *            for bit
 *   "timing" 1: an event pair around every time step's sweep launches
 *            (stats.sweep_ms, stats.sweep_launches), read after the call: no
 *            extra synchronisation, graphs and PDL stay on                  */
PG_API int pg_set_option(pg_grid *g, const char *key, int64_t value);

typedef struct {
  int64_t steps_done;      /* time steps completed */
  int64_t sweeps_total;    /* relaxation sweeps performed (sum over steps) */
  int64_t sweeps_max;      /* max sweeps in one step */
  int64_t failed_step;     /* first step that hit max_sweeps (0: none) */
  int64_t kernel_launches; /* kernels launched by this call */
  double last_delta;       /* max |dV| of the final sweep of the last step (V) */
  double device_ms;        /* device time of the call (CUDA events) */
  double sweep_ms;         /* device time of the sweep launches that ran (option "timing") */
  int64_t sweep_launches;  /* sweep-kernel launches that did work (option "timing") */
  int64_t sweeps_per_launch; /* F: sweeps fused per sweep launch (convergence tested every F sweeps) */
} pg_stats;

/* Algorithm 1: backward-Euler transient from x(0) at t = 0 for `steps` steps
 * of length h (> 0).  Each step: fused RHS kernel (PWL loads at t+h, C/h x(t),
 * pad and inductor history) -> relaxation sweeps from V(s-1) until
 * max_i |V_i^(k) - V_i^(k-1)| < tol (Algorithm 1 line 8, infinity norm) or
 * max_sweeps -> inductor companion-current update.  The RHS kernel and one
 * pass after the last step check the iterates for NaN / Inf (PG_ENONFINITE).
 * tol <= 0 runs exactly
 * max_sweeps sweeps per step.  omega in (0, 2) (Eq. (15); 1 = Gauss-Seidel).
 * method: PG_METHOD_RBSOR or PG_METHOD_JACOBI.  When the fused sweep kernel
 * checks convergence every F sweeps (option "fuse"), a step may run up to
 * F-1 sweeps past the first sweep below tol.
 * Probes: probe_out[(s) * n_probe + p] = V(s h) at node probe_node[p] for
 * s = 0..steps (probe_out holds (steps+1)*n_probe doubles in `mem`);
 * n_probe = 0 disables recording.  sweeps_out (nullable, HOST, steps+1
 * int64) receives per-step sweep counts.  stats (nullable, host) is filled
 * on success and on PG_ENOCONV.                                             */
PG_API int pg_transient(pg_grid *g, double h, int64_t steps, double tol, double omega,
                        int method, int64_t max_sweeps, int64_t n_probe,
                        const int64_t *probe_node, double *probe_out, int mem,
                        int64_t *sweeps_out, pg_stats *stats);

/* Algorithm 1 continued: `steps` more backward-Euler steps from the grid's
 * current state -- the voltages and inductor currents left by the previous
 * pg_transient / pg_transient_continue call (steps s0+1 .. s0+steps at
 * t = s h, s0 = the steps taken since x(0)), or by pg_set_voltages / pg_dc
 * (s0 = 0: the state is x(0) at t = 0; after pg_dc it is the DC operating
 * point).  A transient cut into consecutive calls gives the same results
 * as one call over all its steps (Algorithm 1 line 2 loop; the time
 * loop only carries V and the inductor currents).  h must equal the h of the
 * steps taken so far (PG_EINVAL otherwise).  Probes record V(s0 h) at row 0
 * and V((s0+k) h) at row k.  Other arguments and results as pg_transient.   */
PG_API int pg_transient_continue(pg_grid *g, double h, int64_t steps, double tol, double omega,
                                 int method, int64_t max_sweeps, int64_t n_probe,
                                 const int64_t *probe_node, double *probe_out, int mem,
                                 int64_t *sweeps_out, pg_stats *stats);

/* ---- Multi-GPU: slab partition of a mesh -------------------
 * A global layers x NY x nx mesh is cut into blocks of rows ("slabs"), one per
 * rank.  Rank r's slab grid is an ordinary mesh grid (pg_create_mesh) over the
 * global rows [max(0, Y0 - G), min(NY, Y1 + G)): its owned rows [Y0, Y1) plus G
 * ghost rows of each neighbour, built from the global arrays' rows (gy of the
 * last local row set to 0) with the pads and loads of those rows.  The
 * red-black sweep is exact on the owned rows when G >= 2 F (F = option
 * "fuse"): every sweep launch recomputes 2F rows of halo from the ghost rows
 * (Eq. (13) in the global red-black numbering, R12).       */

/* Mark local rows [y_begin, y_end) as owned (updated, written, counted in the
 * convergence norm); y0_parity = parity of the global index of local row 0.
 * Mesh grids only (PG_ESTATE otherwise).  A slab grid is advanced only by
 * pg_group_transient.                                                       */
PG_API int pg_set_slab(pg_grid *g, int32_t y_begin, int32_t y_end, int32_t y0_parity);

typedef struct pg_group pg_group;

/* A fresh NCCL unique id (128 bytes written to id128) for pg_group_nccl; call
 * on one rank and broadcast it.  NCCL is loaded at run time (libnccl.so.2, the
 * copy already in the process if any); PG_ESTATE if it cannot be loaded.    */
PG_API int pg_nccl_unique_id(void *id128);

/* Join this process's slab (rank `rank` of `nranks`, ranks ordered by rows,
 * one GPU each, current device) into an NCCL group with `ghost` rows per side.
 * Collective: every rank calls it with the same id.  The slab must own
 * [ghost, ny - ghost) except at the global edges (rank 0 owns from local row 0,
 * the last rank up to its last row).                                        */
PG_API int pg_group_nccl(pg_grid *slab, const void *id128, int32_t nranks, int32_t rank,
                         int32_t ghost, pg_group **out);

/* Single-process group of n slab grids on the current device, ordered by rows
 * and sharing one stream: the n-rank protocol with device-to-device copies in
 * place of NCCL (emulates n ranks on one GPU; same kernels and ordering).   */
PG_API int pg_group_local(int32_t n, pg_grid *const *slabs, int32_t ghost, pg_group **out);

/* Algorithm 1 on all slabs in lockstep (method: red-black SOR).  After every
 * sweep launch the launch's convergence norm max|dV| is max-reduced over all
 * slabs (ncclAllReduce of one 8-byte word) and each slab's `ghost` boundary
 * rows are sent to its neighbours' ghost rows (ncclSend/ncclRecv of packed
 * rows), so every rank takes the same stopping decision and the owned rows
 * equal the single-grid iterates.  Arguments as pg_transient (no probes;
 * voltages via pg_get_voltages on each slab, owned rows); sweeps_out / stats
 * describe this process's first slab (identical on all ranks).  Collective.  */
/* Peer-memory slab exchange: the sweep kernel of every slab
 * stores its boundary rows straight into the neighbours' receive buffers
 * (double-buffered by launch epoch), max-reduces its convergence norm into
 * every slab's norm ring with remote atomics and bumps every slab's arrival
 * counter; the next launch waits on its local counter -- no separate
 * collective per launch.  Needs the two-sweep pipeline kernel for every launch
 * (options fuse = 0 / 2, pipe = 1; max_sweeps even) and ghost >= 4; at most
 * 8 slabs.  All slabs must run the same transients.  A wait that exceeds ~4 s
 * (a missing peer) makes pg_group_transient return PG_ECUDA.
 *
 * Arguments and ownership: slabs / slab are grids marked with pg_set_slab
 * (rank r of nranks, `ghost` rows of each neighbour, the layout of
 * pg_group_local); the group keeps pointers to them (destroy the group before
 * the grids) and owns its receive buffers and mapped peer memory
 * (pg_group_destroy releases them).  A slab grid of a group cannot be swept on
 * its own (pg_transient / pg_dc return PG_EINVAL).
 *
 * pg_group_local_p2p: n slabs on the current device in one process (their
 *   "peers" are each other's buffers; the launches are ordered on one stream).
 * pg_group_p2p_create / _export / _connect: one slab per process and GPU;
 *   export this rank's record into blob (cap bytes available; *len receives
 *   the record size; blob may be NULL to query it; the record holds the CUDA
 *   IPC handles of the receive buffers and control block), gather the records
 *   of all ranks concatenated in rank order (e.g. torch.distributed
 *   all_gather), pass them with blob_len = the record size to connect, then
 *   barrier before the first transient.  Errors: PG_EINVAL for bad ranks,
 *   ghost rows, options or inconsistent records; PG_ECUDA when a CUDA call
 *   (IPC mapping) fails. */
PG_API int pg_group_local_p2p(int32_t n, pg_grid *const *slabs, int32_t ghost, pg_group **out);
PG_API int pg_group_p2p_create(pg_grid *slab, int32_t nranks, int32_t rank, int32_t ghost, pg_group **out);
PG_API int pg_group_p2p_export(pg_group *grp, void *blob, int64_t cap, int64_t *len);
PG_API int pg_group_p2p_connect(pg_group *grp, const void *blobs, int64_t blob_len);

PG_API int pg_group_transient(pg_group *grp, double h, int64_t steps, double tol, double omega,
                              int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats);

/* Self-test of a connected CUDA-IPC peer group (no kernel waits on another
 * rank, so it may run with all ranks on one GPU): phase 0 writes this rank's
 * mark (0x5EED0000 + rank) into its control block and, through the mapped
 * peer pointers, into element 0 of the neighbours' receive buffers; after a
 * host barrier over all ranks, phase 1 reads every rank's mark through the
 * mapped control blocks into out[0..nranks) and the marks the neighbours
 * stored into this rank's lower / upper receive buffers into out[nranks],
 * out[nranks+1] (-1 without that neighbour).  Call before the first
 * transient (the first transient reseeds the receive buffers).          */
PG_API int pg_group_p2p_selftest(pg_group *grp, int32_t phase, int64_t *out);

/* pg_group_transient continued from every slab's current state (as
 * pg_transient_continue for a single grid).  Collective.                  */
PG_API int pg_group_transient_continue(pg_group *grp, double h, int64_t steps, double tol, double omega,
                                       int64_t max_sweeps, int64_t *sweeps_out, pg_stats *stats);

/* Free the group's buffers and communicator (the slab grids stay).  NULL ok. */
PG_API void pg_group_destroy(pg_group *grp);

/* DC analysis (§II-A "In DC analysis, A = G", Eq. (3)): solve
 * G v = G0 Vdd - i(t) by the same relaxation (Eq. (13)/(15) with C/h = 0:
 * capacitors open; a series R-L branch conducts 1/R, its inductor shorted), the
 * loads evaluated at time t, starting from x(0) (pg_set_voltages; default Vdd).
 * The result is read with pg_get_voltages; inductor currents are left at the
 * DC branch currents.  Every node needs a conductive path to a pad (else
 * PG_EINVAL: zero diagonal).  Convergence needs omega close to 2 on large
 * grids (no C/h term on the diagonal).  Other arguments as pg_transient.   */
PG_API int pg_dc(pg_grid *g, double t, double tol, double omega, int method, int64_t max_sweeps,
                 pg_stats *stats);

/* Relaxation factor for Eq. (15) by Young's theory (§IV-D defers the
 * choice of omega to [Young]): `sweeps` Jacobi sweeps of the homogeneous
 * system (C/h + G + hL) e = 0 from x(0); the spectral radius rho of the Jacobi
 * iteration matrix J is estimated by the Rayleigh quotient of J^2 at the
 * second-to-last iterate, rho^2 ~ ||e_N||_D^2 / ||e_{N-1}||_D^2 (D = diagonal of
 * the system; D^{1/2} J D^{-1/2} is symmetric), and for the red-black
 * (2-cyclic, consistently ordered) numbering the optimal SOR factor is
 * 2 / (1 + sqrt(1 - rho^2)) (clamped to 1.999).  The estimate approaches rho
 * from below as `sweeps` grows.  Leaves the grid's state as after creation /
 * pg_set_voltages.                                                        */
PG_API int pg_estimate_omega(pg_grid *g, double h, int64_t sweeps, double *rho, double *omega_opt);

/* Relaxation factor tuned on the grid's own transient: omega_b from
 * pg_estimate_omega (2000 sweeps), then n_cand candidates omega_b + k d_omega
 * (k = 0 .. n_cand-1, capped at 1.999; Young: overestimating omega_b costs
 * little, underestimating it a lot) each run for the first `steps` time steps
 * from x(0) to tol; *omega_out = the candidate with the fewest sweeps
 * (sweeps_out, nullable host int64[n_cand], receives every candidate's total;
 * INT64_MAX if it hit 1e6 sweeps in a step).  Leaves the grid at x(0) with
 * zero inductor currents.  1 <= n_cand <= 64, d_omega >= 0, tol > 0.      */
PG_API int pg_tune_omega(pg_grid *g, double h, int64_t steps, double tol, int64_t n_cand, double d_omega,
                         double *omega_out, int64_t *sweeps_out);

/* Number of nodes / dimensions (layers, ny, nx are 0 for CSR grids). */
PG_API int pg_info(const pg_grid *g, int64_t *n, int32_t *layers, int32_t *ny, int32_t *nx,
                   int32_t *n_colors);

/* Free all device memory of the grid.  NULL is a no-op.  The grid's blocks
 * return to the library's per-device memory pools, which keep up to
 * PGB200_POOL_GIB (default 48) GiB of freed per-node arrays and 1 GiB of
 * smaller blocks mapped for the next grid (re-mapping a config-4-sized grid
 * costs ~0.4-1 s per create); pg_release_memory hands them back. */
PG_API void pg_destroy(pg_grid *g);

/* Return the freed blocks the library's memory pools hold on `device`
 * (-1: every device the library has used) to the CUDA driver, so that other
 * allocators of the process (cudaMalloc, PyTorch) can use that memory.  Live
 * grids keep their memory.  Synchronises the device(s).  Returns PG_OK, or
 * PG_EINVAL for a device index outside [-1, 63]. */
PG_API int pg_release_memory(int32_t device);

/* Description of the last error on this thread ("" if none). */
PG_API const char *pg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PGRID_H */
