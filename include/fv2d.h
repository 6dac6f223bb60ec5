/*
 * fv2d.h -- C ABI of libfv2d.so, the B200 (sm_100a) hot path of the first-order
 * finite-volume scheme of arXiv:1701.05431 (Essadki et al., "A task-driven
 * implementation of a simple numerical solver for hyperbolic conservation laws").
 *
 * Problem statement followed by this interface (PAPER.md = P:, SPEC.md = S:):
 *   dW/dt + div F(W) = S(W), W in R^nVar                      (eq:conservation_law)
 *   Nx x Ny Cartesian cells on [x0,x1] x [y0,y1]
 *   W* = W - dt/dx (F~_{i+1/2} - F~_{i-1/2}) - dt/dy (...)    (eq:VF_scheme)
 *   F~ = Lax-Friedrichs with directional sigma
 *   dt * max |lambda| <= min(dx, dy), fixed dt checked         (eq:CFL_cond)
 *   W^{n+1} = W* + dt S(W*)                                   (eq:SourceTerm)
 * Systems: scalar advection (nVar 1, BASELINE configs[0]), Euler (nVar 4,
 * eq:Euler P:626-636, S = 0), evaporating spray (nVar 6, eq:Essadki P:938-999,
 * source with the NDF reconstruction of S:401-419).  Arithmetic is IEEE
 * binary64 in the canonical evaluation order of DESIGN.md §3.1 with no FMA
 * contraction, so transport results are bitwise those of a plain CPU loop.
 *
 * Conventions
 *  - Every call returns an fv2d_status; nothing throws, nothing aborts.
 *  - A context is thread-compatible, not thread-safe: one thread at a time.
 *  - Host arrays are owned by the caller; the library copies in/out.  Device
 *    buffers, the NCCL communicator and device scalars are owned by the context.
 *  - Stepping is asynchronous on the context's CUDA stream.  Numerical errors
 *    (CFL violation, non-admissible state, reconstruction failure) are latched
 *    on the device; once latched every later step is a no-op and the readable
 *    state is W^k of the failing step k (ping-pong buffers are never half
 *    written).  They are reported by fv2d_synchronize / fv2d_get_state /
 *    fv2d_compute_dt and described by fv2d_last_error.
 *  - Layouts: FV2D_AOS is the paper's Cell array: double
 *    W[ny][nx][nvar] (x fastest, variable innermost).  FV2D_SOA is
 *    double W[nvar][ny][nx].  With nranks > 1 every host array holds this
 *    rank's block only: with y-slabs (nranks_x <= 1) rows
 *    [rank*ny/nranks, (rank+1)*ny/nranks) of all nx columns; with 2-D blocks
 *    (nranks_x = PX > 1, PY = nranks/PX, rank = ry*PX + rx) rows
 *    [ry*ny/PY, (ry+1)*ny/PY) x columns [rx*nx/PX, (rx+1)*nx/PX), so nx and ny
 *    in the shapes above read as the block's width and height.
 */
#ifndef FV2D_H
#define FV2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FV2D_VERSION_MAJOR 1
#define FV2D_VERSION_MINOR 0

typedef enum {
  FV2D_OK = 0,
  FV2D_E_ARG = 1,       /* invalid argument / configuration (usage error, S:612 code 1) */
  FV2D_E_CFL = 2,       /* fixed dt violates eq:CFL_cond at the start of a step */
  FV2D_E_NONFINITE = 3, /* non-admissible or non-finite state (rho<=0, p<=0, NaN, inf) */
  FV2D_E_RECON = 4,     /* spray NDF reconstruction failed to converge */
  FV2D_E_CUDA = 5,      /* CUDA runtime error (message in fv2d_last_error) */
  FV2D_E_NCCL = 6,      /* NCCL error */
  FV2D_E_STATE = 7      /* call not valid in the context's current state (e.g. no state set) */
} fv2d_status;

typedef enum { FV2D_ADVECTION = 0, FV2D_EULER = 1, FV2D_SPRAY = 2 } fv2d_system;

/* Boundary conditions per axis.  Periodic is the paper's domain (R/Z)^2.
 * Dirichlet: the ghost cell is the constant state cfg.dirichlet.
 * Wall: the ghost is the mirror of the boundary cell with the normal momentum
 * negated (Euler, spray); not defined for advection (FV2D_E_ARG). */
typedef enum { FV2D_BC_PERIODIC = 0, FV2D_BC_DIRICHLET = 1, FV2D_BC_WALL = 2 } fv2d_bc;

typedef enum { FV2D_AOS = 0, FV2D_SOA = 1 } fv2d_layout;

/* Kernel / schedule options (cfg.flags). */
#define FV2D_FLAG_NAIVE 0x1u        /* paper's GPU mapping: one thread per cell,
                                        every neighbour re-derived, every face computed twice.
                                        Same bits, ~2.5x the FP64 work; kept as a baseline. */
#define FV2D_FLAG_SPLIT_SOURCE 0x2u /* spray: source as a separate pass after transport
                                        (the only mode; accepted for compatibility) */
#define FV2D_FLAG_ONE_CELL 0x4u     /* fused kernel with one cell per lane instead of the
                                        default two-cells-per-lane kernel (same bits) */
#define FV2D_FLAG_FUSE_SOURCE 0x10u /* reserved (removed): a one-pass spray step (flux + update +
                                        source per cell) was built and measured slower than the
                                        split source pass on B200 (2.38 vs 1.96 ms at 4096^2; the
                                        source is issue-bound and the transport's instructions land
                                        on that pipe).  fv2d_create returns
                                        FV2D_E_ARG if it is set. */
#define FV2D_FLAG_GRAPH 0x20u      /* replay each step from a CUDA graph captured once per
                                        ping-pong parity (re-captured when dt/mode change);
                                        single-process contexts only */
#define FV2D_FLAG_PEER_HALO 0x40u  /* nranks > 1 without NCCL: the step kernel stores its
                                        boundary rows straight into the neighbours' ghost rows
                                        over peer memory (NVLink), and the CFL max-all-reduce is
                                        done with system-scope atomics and an arrival counter in
                                        peer memory.  Connect with fv2d_peer_connect (CUDA IPC,
                                        one process per GPU) or fv2d_peer_connect_local (ranks of
                                        one process) before fv2d_set_state. */
#define FV2D_FLAG_NCCL_LOOPBACK 0x8u /* take the NCCL halo/all-reduce path even with
                                        nranks == 1 (self send/recv; needs an id from
                                        fv2d_nccl_unique_id); exercises the multi-GPU
                                        plumbing on one device */
#define FV2D_FLAG_PEER_SPLIT 0x100u  /* peer-memory path with the CFL all-reduce and the finalize
                                        as two small kernels after the step kernel instead of
                                        inside its last CTA (the default: one kernel per step) */
#define FV2D_FLAG_GHOST_COLUMNS 0x80u /* store x-ghost columns and route the x-neighbour data
                                        through them exactly as for 2-D rank blocks
                                        (nranks_x > 1, where this is implied), even with
                                        one block along x: that block is its own west/east
                                        neighbour when x is periodic.  Same bits; with
                                        FV2D_FLAG_NCCL_LOOPBACK it exercises the NCCL column
                                        exchange (pack, send/recv, unpack) on one device */

typedef struct {
  int32_t nx, ny;          /* global mesh, >= 1; ny % (nranks*nslabs) == 0 */
  int32_t nvar;            /* must equal the system's nVar (1, 4, 6) */
  int32_t system;          /* fv2d_system */
  int32_t bc_x, bc_y;      /* fv2d_bc */
  double x0, x1, y0, y1;   /* domain; dx = (x1-x0)/nx, dy = (y1-y0)/ny */
  double param[8];         /* advection: a_x, a_y | euler: gamma | spray: K, theta */
  double dirichlet[6];     /* constant ghost state for FV2D_BC_DIRICHLET */
  int32_t rank, nranks;    /* y-slab decomposition across processes (1 GPU each) */
  int32_t nslabs;          /* y-slabs per process on the same device (>= 1); their
                              ghost rows are exchanged exactly like the ranks' */
  int32_t device;          /* CUDA device ordinal */
  uint32_t flags;          /* FV2D_FLAG_* */
  int32_t tiles_x, tiles_y; /* 0/1: one launch per step.  > 1: each step is launched as
                              tiles_x x tiles_y separate sub-launches over the slab (the
                              paper's NPartX x NPartY task decomposition, P:215-220;
                              granularity study P:741-754).  Same bits. */
  int32_t nranks_x;        /* 0/1: y-slabs.  PX > 1: the ranks form a PX x (nranks/PX) grid of
                              2-D blocks (the paper's NPartX x NPartY decomposition with
                              its four overlaps): rank = ry*PX + rx owns
                              columns [rx*nx/PX, ...) of rows [ry*ny/PY, ...); each block
                              also stores its east/west ghost columns, written by the
                              neighbours' step kernels (FV2D_FLAG_PEER_HALO) or exchanged
                              by NCCL.  Requires nx % PX == 0, nx/PX >= 2, nslabs == 1. */
  int32_t reserved[4];     /* must be 0 */
} fv2d_config;

typedef struct fv2d_ctx fv2d_ctx;

typedef struct {
  int64_t steps;           /* steps issued (including no-op steps after a latched error) */
  int64_t kernel_launches; /* kernels launched by this context so far */
  int64_t newton_iters;    /* spray: Newton iterations summed over cells and steps, if counted */
  double dt;               /* current device dt (adaptive mode), 0 if unset */
  double step_kernel_ms;   /* with profiling on: summed device time of the step kernels
                              (CUDA events recorded on the context stream around each
                              step-kernel launch), since profiling was enabled */
  int64_t step_kernels_timed; /* number of step-kernel launches in step_kernel_ms */
  double source_kernel_ms;    /* with profiling on: summed device time of the split spray
                                 source kernels of steps (not captured in a CUDA graph) */
  int64_t source_kernels_timed;
  int32_t sms;             /* multiprocessors of the context's device */
  int32_t resident_ctas;   /* resident CTAs of the marching step kernel (SMs x occupancy API),
                              the launch-shape cost model's wave size */
  int32_t strip_rows;      /* rows per CTA strip chosen for a full-slab launch */
  int32_t reserved0;
} fv2d_stats;

/* Library version; never fails. */
fv2d_status fv2d_version(int32_t* major, int32_t* minor);

/* Default-initialised config: periodic unit square, Euler gamma = 1.4, 1 rank, 1 slab. */
fv2d_status fv2d_config_default(fv2d_config* cfg, int32_t nx, int32_t ny, int32_t system);

/* NCCL unique id for nranks > 1 (call on rank 0, broadcast the 128 bytes, e.g.
 * with torch.distributed).  FV2D_E_NCCL if libnccl.so.2 cannot be loaded. */
fv2d_status fv2d_nccl_unique_id(uint8_t id[128]);

/* Create a context: validates cfg, selects cfg.device, allocates the two
 * ping-pong SoA buffers of this rank's slab(s) (plus ghost rows and a staging
 * buffer), and for nranks > 1 initialises an NCCL communicator from nccl_id
 * (collective over all ranks).  cuda_stream: a cudaStream_t to run on (NULL =
 * the legacy default stream); it must outlive the context. */
fv2d_status fv2d_create(const fv2d_config* cfg, const uint8_t* nccl_id, void* cuda_stream,
                        fv2d_ctx** out);

/* Release every resource of ctx (NULL is accepted). */
fv2d_status fv2d_destroy(fv2d_ctx* ctx);

/* Initial condition W^0: copy this rank's slab from a host array in
 * `layout`, fill the ghost rows (halo exchange for nranks > 1), reset the step
 * counter, the latched error and the adaptive dt.  Synchronous. */
fv2d_status fv2d_set_state(fv2d_ctx* ctx, const double* host, fv2d_layout layout);

/* Same from a device array (SoA [nvar][ny_local][nx], tight pitch); asynchronous. */
fv2d_status fv2d_set_state_device(fv2d_ctx* ctx, const double* dev, fv2d_layout layout);

/* Copy the current state W^k of this rank's slab to a host array.  Synchronous.
 * Returns the latched error, if any (the copied state is then W^k of the
 * failing step). */
fv2d_status fv2d_get_state(fv2d_ctx* ctx, double* host, fv2d_layout layout);

/* CFL reduction (eq:CFL_cond): smax = max over all cells (all ranks) of
 * max(|lambda|_x, |lambda|_y) of the current state; dt = (cfl*min(dx,dy))/smax.
 * Also installs dt as the adaptive time step.  Synchronous.  smax/dt may be NULL. */
fv2d_status fv2d_compute_dt(fv2d_ctx* ctx, double cfl, double* dt, double* smax);

/* Check a fixed dt against eq:CFL_cond on the current state without stepping:
 * FV2D_E_CFL if dt*smax > min(dx,dy).  Synchronous.  smax may be NULL. */
fv2d_status fv2d_check_dt(fv2d_ctx* ctx, double dt, double* smax);

/* nsteps steps with the paper's constant dt: each step checks
 * dt*smax(W^n) <= min(dx,dy) (fused into the step pass) and computes W^{n+1}
 * = transport (eq:VF_scheme) + source (eq:SourceTerm, spray only).  On a CFL
 * violation at step k the error is latched and the state stays W^k.
 * Asynchronous (no host synchronisation).  FV2D_E_ARG if dt <= 0 or nsteps < 0. */
fv2d_status fv2d_step(fv2d_ctx* ctx, double dt, int32_t nsteps);

/* nsteps steps with dt_n = (cfl*min(dx,dy))/smax(W^n) (BASELINE north_star
 * "CFL time-step reduction"); smax(W^{n+1}) is reduced in the epilogue of step
 * n.  dt_log (nsteps doubles, may be NULL) receives every dt used; passing a
 * non-NULL dt_log synchronises.  FV2D_E_ARG if cfl <= 0 or cfl > 1. */
fv2d_status fv2d_step_adaptive(fv2d_ctx* ctx, double cfl, int32_t nsteps, double* dt_log);

/* One standalone splitting step W <- W + dt S(W) (eq:SourceTerm) on the
 * current state; identity for S = 0 systems.  Asynchronous. */
fv2d_status fv2d_apply_source(fv2d_ctx* ctx, double dt);

/* Wait for all work of ctx; return the latched numerical error, if any. */
fv2d_status fv2d_synchronize(fv2d_ctx* ctx);

/* Zero-copy view of the current device state of local slab `slab` (layout
 * "row-interleaved SoA"): element (v, j, i) is at
 * d_ptr[j*row_stride + v*pitch + i] for j in [-1, ny_slab] (rows -1 and ny_slab
 * are the ghost rows).  Valid until the next step. */
fv2d_status fv2d_device_state(fv2d_ctx* ctx, int32_t slab, double** d_ptr, int64_t* pitch,
                              int64_t* row_stride, int32_t* ny_slab);

/* Description of the last error: message (NUL-terminated, truncated to n), the
 * step index, the global cell index j*nx+i (lowest index among offending cells)
 * and the offending value (speed for E_CFL).  Any output pointer may be NULL. */
fv2d_status fv2d_last_error(fv2d_ctx* ctx, char* buf, size_t n, int64_t* step, int64_t* cell,
                            double* value);

/* Counters; with profiling on, synchronises and folds the pending kernel events
 * into step_kernel_ms. */
fv2d_status fv2d_get_stats(fv2d_ctx* ctx, fv2d_stats* out);

/* Host-resident stepping: W^0 = host_in (as fv2d_set_state), nsteps steps of
 * the constant dt checked every step (as fv2d_step), host_out = the result (as
 * fv2d_get_state); synchronous.  Same bits as those three calls.  For a
 * single-rank, single-slab context (y-slab layout; the spray with its split
 * source pass run per band) with layout FV2D_AOS the first step is pipelined
 * over row bands: band b is copied host->device and converted while band b-1
 * is stepped and band b-2 is converted back and copied device->host, so the two copy
 * directions and the kernels overlap (the bands next to the periodic/wall
 * y-boundary are stepped last, after the ghost rows are filled).  Other
 * contexts run the three calls in sequence.  host_out may equal host_in.
 * Use fv2d_host_alloc (pinned) memory for overlapped copies.  On a latched
 * error the state, and host_out, hold W^k of the failing step k (the output
 * bands already copied are overwritten with W^k). */
fv2d_status fv2d_step_host(fv2d_ctx* ctx, const double* host_in, double* host_out, fv2d_layout layout, double dt,
                           int32_t nsteps);

/* Asynchronous output (the paper's gatherForOutput -> switch -> outputToDisk
 * pipeline, which writes a snapshot without a global barrier):
 * enqueue a copy of the current state W^k of this rank's slab into `host`
 * (layout as fv2d_get_state; use fv2d_host_alloc memory for a truly
 * asynchronous copy) and return at once.  On a side stream the state is
 * converted into a device staging buffer and copied to the host while later
 * steps run; only the step that would overwrite W^k's buffer waits for the
 * conversion.  `host` must stay valid until fv2d_snapshot_wait returns.
 * Snapshots are taken in call order; stepping results are unchanged (bitwise). */
fv2d_status fv2d_snapshot(fv2d_ctx* ctx, double* host, fv2d_layout layout);

/* Block until every enqueued snapshot has landed in host memory. */
fv2d_status fv2d_snapshot_wait(fv2d_ctx* ctx);

/* Peer-memory multi-GPU path (FV2D_FLAG_PEER_HALO).  fv2d_peer_export writes this
 * rank's FV2D_PEER_HANDLE_BYTES of CUDA IPC handles (both state buffers and the
 * collective sync block); gather them from every rank (rank-major) and pass the
 * nranks * FV2D_PEER_HANDLE_BYTES bytes to fv2d_peer_connect on every rank.
 * fv2d_peer_connect_local does the same for contexts of one process (group[r]
 * = the context of rank r; the ranks must then be driven from separate host
 * threads and streams, like separate processes).  Collective calls
 * (set_state, compute_dt, check_dt, step*, apply_source) must be made by all
 * ranks in the same order, as with NCCL; a rank that never arrives makes the
 * others latch FV2D_E_NCCL after ~20 s instead of hanging. */
#define FV2D_PEER_HANDLE_BYTES 192
fv2d_status fv2d_peer_export(fv2d_ctx* ctx, uint8_t* handles);
fv2d_status fv2d_peer_connect(fv2d_ctx* ctx, const uint8_t* all_handles);
fv2d_status fv2d_peer_connect_local(fv2d_ctx* ctx, fv2d_ctx* const* group);

/* Page-locked host memory for snapshots / state transfers (cudaHostAlloc). */
fv2d_status fv2d_host_alloc(size_t bytes, void** ptr);
fv2d_status fv2d_host_free(void* ptr);

/* enable != 0: record a CUDA event pair around every step-kernel launch (for the
 * roofline measurement of the dominant kernel); resets the accumulated time. */
fv2d_status fv2d_set_profiling(fv2d_ctx* ctx, int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* FV2D_H */
