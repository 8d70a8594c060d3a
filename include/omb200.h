/*
 * omb200.h -- C ABI of the B200 hydro-step library (libomb200.so).
 *
 * Plain C: device pointers, sizes and a CUDA stream handle passed as void*.
 * No torch or Python types.  Every call is stream-ordered and asynchronous;
 * nothing here synchronises the host.  Return value 0 = success, negative =
 * error (message via omb_last_error()).
 *
 * Each entry point replaces one interface of the reference (octomini):
 *   omb_primitives   <- kernels.primitives         pkg/src/octomini/kernels.py:36, _kernels/reference.py:30-45
 *   omb_reconstruct  <- kernels.reconstruct        kernels.py:37, _kernels/_core.pyx:41-156
 *   omb_fluxes       <- kernels.fluxes             kernels.py:38, _kernels/_core.pyx:223-347
 *   omb_stage        <- HydroStepper._stage        hydro/step.py:106-144 (ghost fill -> reconstruct ->
 *                       fluxes -> update, fused; the CFL-abort test of :132-139 is done by the
 *                       caller on the amax this call accumulates)
 *   omb_cfl          <- HydroStepper.cfl_dt        hydro/step.py:81-92
 *   omb_gather       <- mesh.ghosts.fill_leaf_ghosts (same-level + physical BCs), ghosts.py:115-150
 */
#ifndef OMB200_H
#define OMB200_H

#ifdef __cplusplus
extern "C" {
#endif

#define OMB_ABI_VERSION 7

/* per-leaf topology / geometry record (device array, one per leaf) */
typedef struct {
    int nbr[27];   /* batch index of the same-level neighbour at offset (i,j,k), index (i+1)*9+(j+1)*3+(k+1); -1 none */
    int offmask;   /* bit 2a: the -a face is a physical wall; bit 2a+1: the +a face */
    double ox, oy, oz;  /* first interior cell centre (SubGrid.origin) */
    double dx, inv_dx;  /* cell width and the host-computed 1.0/dx */
    int flags;     /* bit 0: export face fluxes to flux[slot]; bit 1: update deferred to omb_reflux_update;
                    * 8^3 blocks of a 16^3/32^3 leaf: bit 2+2a / 3+2a: the positivity-fallback count on axis a
                    * starts at 3 / ends at 10 (not 2 / 11); bits 8+5a: the block's cell offset in its leaf */
    int slot;      /* flux export slot (OMB_FLUX_SLOT doubles: FX (6,9,8,8), FY (6,8,9,8), FZ (6,8,8,9)) */
} OmbLeafInfo;

#define OMB_FLUX_SLOT (3 * 6 * 9 * 8 * 8)
#define OMB_AMR_TASK_INTS 16

/* one RK3 stage over all runs of the batch (state layout [6][fstride], leaf-major 8^3 blocks, z fastest) */
typedef struct {
    const double *ucur;   /* stage input, also the halo source */
    const double *u0;     /* RK3 step-start snapshot */
    double *unext;        /* stage output (must not alias ucur) */
    const double *grav;   /* [4][fstride] gx,gy,gz,dphi_dt or NULL */
    long long fstride;    /* doubles between fields (>= nleaves*512) */
    const OmbLeafInfo *info;
    const int *run_off;   /* [nruns+1] offsets into run_leaf */
    const int *run_leaf;  /* leaf indices of each run (1..4 leaves), consecutive along +x at one level */
    int nruns;
    const double *dt;     /* device scalar */
    double a, b;          /* stage weights (SSP_RK3_STAGES) */
    double gamma, gm1, eta, inv_gamma, omega;   /* gm1 = gamma-1.0, inv_gamma = 1.0/gamma (host-rounded) */
    double floor_rho, floor_tau, floor_vmax;
    int bc;               /* 0 outflow, 1 reflecting, 2 periodic */
    int new_mode, override_center, contact;
    unsigned long long *amax_bits;  /* device: running max of the signal speed (bits of a non-negative double) */
    unsigned long long *fallback;   /* device: running positivity-fallback count */
    double *flux;         /* face-flux export slots (AMR coarse/fine faces), may be NULL if no leaf exports */
    /* multi-GPU, NVLink peer reads (replaces the halo exchange of ghosts.py:115-150 across ranks):
     * halo[k] = address of the field-0 block of the leaf in halo slot nown + k inside its OWNER's
     * stage-input buffer (CUDA IPC peer memory, same fstride on every rank); NULL: halo slots local */
    const double *const *halo;
    int nown;
    /* passive-scalar pass (species; SURVEY.md 0.2 -- a scalar follows tau's path: PPM, KT flux,
     * Simpson faces, RK update, no sources / dual energy / floors): scalar != 0 runs the stage on
     * ucur = (rho, sx, sy, sz, p, X) built by omb_scalar_input, reads X's step-start state from
     * s_u0 and writes only X's stage output to s_next ([fstride] each); unext is not written */
    int scalar;
    const double *s_u0;
    double *s_next;
} OmbStageDesc;

/* AMR ghost regions: each task fills, in the interior of a VIRTUAL leaf (batch index >= number of real
 * leaves), the cells the stage kernel's gather reads for one coarse/fine neighbour region of a real leaf:
 * minmod prolongation of the coarse leaf (task[0] = 0) or 8-cell restriction of the fine children (1).
 * int task[16]: role, rd[3], virtual leaf, coarse: src, m0[3], m1[3], foff[3] | fine: child[8] */
typedef struct {
    double *u;            /* state [6][fstride] (real + virtual leaves) */
    long long fstride;
    const int *tasks;     /* [ntasks][16] */
    int ntasks;
} OmbAmrDesc;

/* reflux + deferred update of coarse leaves on coarse/fine faces */
typedef struct {
    OmbStageDesc stage;   /* same arguments as the stage just run */
    const int *leaf;      /* [nleaves] batch index of each reflux leaf */
    const int *off;       /* [nleaves+1] CSR offsets into tasks */
    const int *tasks;     /* [.][6]: axis, side, fine child's flux slot, k_t1, k_t2, unused */
    int nleaves;
} OmbRefluxDesc;

typedef struct {
    const double *u;      /* state [6][fstride] */
    long long fstride;
    int nleaves;
    const double *dx;     /* [nleaves] */
    double gamma, gm1, eta, cfl;
    double *ratio;        /* scratch [nleaves] */
    int *bad;             /* scratch [nleaves] */
    double *out;          /* [2]: worst = min dx/speed, dt = cfl*worst */
    int *bad_leaf;        /* [1]: first leaf (batch order) with a non-finite speed, -1 none */
    double *dt_dev;       /* optional: receives dt */
} OmbCflDesc;

int omb_abi_version(void);
const char *omb_last_error(void);
int omb_stage_smem_bytes(void);
/* multi-GPU NVLink halo reads: allocate (zeroed) device memory with its CUDA IPC handle (64 bytes), and
 * open a peer's handle in the current device's context (lazy peer access) */
int omb_ipc_alloc(long long bytes, void **ptr, void *handle64);
int omb_ipc_open(const void *handle64, void **ptr);
/* enable kernels of the current device to read peer_device's memory (multi-GPU NVLink halo reads) */
int omb_enable_peer_access(int peer_device);

int omb_primitives(const double *u, int m, double gamma, double eta, double *prim, void *stream);
int omb_reconstruct(const double *prim, int m, int new_mode, int contact_on, double gamma,
                    double *lo, double *hi, unsigned long long *fallback, void *stream);
int omb_fluxes(const double *lo, const double *hi, int n, double gamma, int new_mode, int override_center,
               double *fx, double *fy, double *fz, unsigned long long *amax_bits, void *stream);
int omb_stage(const OmbStageDesc *desc, void *stream);
/* coarse/fine ghost regions (ghosts.py:62-112, transfer.py:13-64) before a stage */
int omb_amr_ghosts(const OmbAmrDesc *desc, void *stream);
/* reflux (step.py:206-241) + update (step.py:243-288) of the deferred coarse leaves after a stage */
int omb_reflux_update(const OmbRefluxDesc *desc, void *stream);
int omb_cfl(const OmbCflDesc *desc, void *stream);
/* multi-GPU halo exchange (replaces the cross-rank part of fill_leaf_ghosts, ghosts.py:115-150):
 * pack whole leaves idx[0..n) of a [6][fstride] state into a leaf-major [n][6][512] message, and
 * unpack such a message into leaf slots first..first+n of a state */
int omb_pack_leaves(const double *u, long long fstride, const int *idx, int n, double *out, void *stream);
int omb_unpack_leaves(const double *in, int n, double *u, long long fstride, int first, void *stream);
/* self-test: counts (into bad[0]) quotients where the kernels' reciprocal-based divisions (div_by,
 * the straight-line KT form, div_nz) differ from IEEE; bad[1..5] = first mismatch (a, b, a/b, div_by, KT form)
 * as bit patterns, bad[7] = claimed flag.  bad must hold 8 zeroed counters. */
int omb_selftest_div(unsigned long long seed, long long n, unsigned long long *bad, void *stream);
/* scalar flux surface (hydro/flux.py:12-94; the reference's test oracle for the point flux):
 * omb_kt_flux  <- flux.kt_flux(left, right, axis, eos) for n point pairs; states [n][7] =
 *   (rho, vx, vy, vz, p, eint, tau) as PrimitiveState holds them; out [n][6].  A pair with a
 *   non-finite rho/v/p gets NaNs and atomically lowers *bad (init n) to its index: the caller raises
 *   NumericsError like flux.py:56-58.
 * omb_face_flux <- flux.face_flux(point_fluxes, new_mode) for n faces; pts [n][9][6], out [n][6] */
int omb_kt_flux(const double *left, const double *right, int n, int axis, double gamma, double *out, int *bad,
                void *stream);
/* omb_physical_flux <- flux.physical_flux(state, axis) (flux.py:40-47) for n states [n][7] */
int omb_physical_flux(const double *states, int n, int axis, double *out, void *stream);
int omb_face_flux(const double *pts, int n, int new_mode, double *out, void *stream);
/* passive scalars: the input of a scalar pass, dst [6][fstride] = (rho, sx, sy, sz, p, X) from the stage
 * input u (p as the stage's primitive conversion computes it, reference.py:30-45).  Leaves [0, n_all) get
 * fields 0-4 (n_all counts the AMR virtual leaves, filled by omb_amr_ghosts before); leaves [0, n_x) get
 * X from x (skip with x = NULL; run omb_amr_ghosts on dst, then this again with x = NULL, for AMR) */
int omb_scalar_input(const double *u, long long fstride, int n_all, const double *x, int n_x, double gamma,
                     double gm1, double eta, double *dst, void *stream);
/* self-check of the device pow (csrc/omb_pow.cuh, glibc's algorithm and tables): out[i] = pow(x[i], y[i]),
 * to be compared bitwise with the host libm's pow -- the reference's tau goes through glibc pow
 * (reference.py:39, hydro/eos.py:50-61) */
int omb_selftest_pow(const double *x, const double *y, long long n, double *out, void *stream);
/* host (CPU) packing between per-leaf padded arrays (6, n+6, n+6, n+6) -- SubGrid.u, tree.py:47-61 --
 * and the [6][L][n^3] device layout; multithreaded, used around H2D/D2H copies.  m = the padded edge
 * of the host arrays: n + 6 for whole leaves; for the 8^3 blocks of 16^3 / 32^3 leaves (n = 8) the
 * leaf's edge (22 / 38), leaf_u[i] pointing at the block's corner inside its leaf's array (ABI 7 added
 * m to the five host-transfer calls) */
int omb_host_pack(const double *const *leaf_u, int L, int n, int m, long long fstride, double *out);
int omb_host_unpack(const double *in, int L, int n, int m, long long fstride, double *const *leaf_u);
/* the same fused with the host<->device copy of a [6][fstride] device state (the e2e path of
 * HydroStepper's host state of record, step.py:94-102): leaves cut into nchunks chunks, host threads
 * pack chunk c into the pinned buffer while chunk c-1 is copied (upload), or unpack chunk c while
 * chunk c+1 is in flight (download).  upload returns with copies still queued on `stream`;
 * download returns with the host arrays written. */
/* host threads used by omb_host_pack/unpack/upload/download (0 = all cores, capped at 16) */
int omb_set_host_threads(int n);
int omb_host_upload(const double *const *leaf_u, int L, int n, int m, long long fstride, double *pinned,
                    double *dev, int nchunks, void *stream);
int omb_host_download(const double *dev, double *pinned, int L, int n, int m, long long fstride,
                      double *const *leaf_u, int nchunks, void *stream);
/* the download overlapped with the launch parts of the stage producing it: chunk c = leaves
 * [bounds[c], bounds[c+1]) is copied on copy_stream after the cudaEvent_t ready[c] fires, then unpacked
 * by the host threads; returns with the host arrays written */
int omb_host_download_after(const double *dev, double *pinned, int n, int m, long long fstride,
                            double *const *leaf_u, int nchunks, const int *bounds, void *const *ready,
                            void *copy_stream);
/* zero-copy host transfers (n = 8): leaf_u is a DEVICE array of L pointers to padded (6, 14, 14, 14)
 * arrays in mapped pinned host memory (the stepper re-homes SubGrid.u into one pinned slab).  The GPU
 * reads / writes them over PCIe in whole 64 B lines: per (field, x), rows y = 3..10 with all z, widened
 * to the 15 lines they touch; the ghost z of those rows and the widening's edge doubles go to / come
 * from `stash` (L * 2688 doubles of device memory), so the host ghost cells are written back unchanged.  Both are asynchronous on `stream`. */
int omb_host_gather(const double *const *leaf_u, int L, long long fstride, double *dev, double *stash, void *stream);
int omb_host_scatter(const double *dev, const double *stash, int L, long long fstride, double *const *leaf_u,
                     void *stream);
/* multi-GPU AMR: gather rows idx[0..n) of length `row` into a contiguous message / scatter them back
 * (the exported face-flux slots the reflux of step.py:206-241 reads across ranks) */
int omb_gather_rows(const double *src, long long row, const int *idx, int n, double *out, void *stream);
int omb_scatter_rows(const double *in, long long row, const int *idx, int n, double *dst, void *stream);
/* device-side diagnostics / IO: per-leaf field sums for conservation_totals
 * (problems/diagnostics.py:9-30; fixed summation order), and the checkpoint payload order
 * (mesh/checkpoint.py:34-55: per leaf, 6 fields, x fastest) */
int omb_leaf_sums(const double *u, long long fstride, int L, double *out, void *stream);
int omb_disk_order(const double *u, long long fstride, int L, double *out, void *stream);
/* FP64 DFMA throughput probe (roofline denominator): blocks*256*8*iters DFMAs */
int omb_fp64_peak(double *scratch, int blocks, int iters, void *stream);
/* padded (6,14,14,14) conserved block of one leaf as the ghost fill would produce it */
int omb_gather(const double *u, long long fstride, const OmbLeafInfo *info, int leaf, int bc,
               double *out, void *stream);
/* the same for n consecutive leaves first..first+n-1 (n <= 65535), out [n][6][14][14][14]: the
 * stage state with its ghosts filled, as HydroStepper._stage hands it to a host gravity solver
 * (hydro/step.py:106-113, mesh/ghosts.py:115-157; AMR regions need omb_amr_ghosts first) */
int omb_gather_leaves(const double *u, long long fstride, const OmbLeafInfo *info, int first, int n, int bc,
                      double *out, void *stream);

/* ---- FMM gravity (gravity/solver.py:50-164; _core.pyx:372-608; multipole.py) ----------------------
 * Order-3 Cartesian FMM over the entity table (octree nodes + each leaf's block hierarchy down to cells).
 * omb_fmm_traverse (HOST): the dual-tree traversal of build_interactions (_core.pyx:372-459): pairs
 *   (pa, pb) in discovery order with their lattice keys; returns the count, or -(count) if cap was
 *   too small.  center [nent][3], width [nent], children [nent][8] (-1 for cells), is_cell [nent].
 * Device passes (stream-ordered): masses rho*dx^3 into the cell entities' M0 (M = [nent][20]);
 *   upward per level (parents [np] of that level); M2L per target entity with its contributions
 *   in the reference's order (off [ntarget+1] into contrib: source | group << 40 | cell-cell << 62 | flip << 63,
 *   D [G][2][20] kernel derivatives and their parity flip; cellcell non-NULL when the lists hold
 *   cell-cell contributions -- the kernels read the kind from bit 62 of each word, which
 *   omb_fmm_build sets); downward per level;
 *   fields phi / gx / gy / gz [nleaf][512] of the cell entities (cell_base [nleaf]). */
long long omb_fmm_traverse(const double *center, const double *width, const long long *children,
                           const unsigned char *is_cell, long long nent, long long root, double theta,
                           long long *pa, long long *pb, long long *pk, long long cap);
/* grouping + per-target contribution lists (HOST, O(pairs)) of a traversal: see omb_fmm.cu */
long long omb_fmm_build(const long long *pa, const long long *pb, const long long *pk, long long np, long long nent,
                        long long *group_first, unsigned char *group_flags, long long gcap, long long *off,
                        unsigned long long *contrib);
/* theta = 0 (direct_traversal_eval, _core.pyx:611-690): per-target lists in traversal order (HOST), and the
 * direct cell-cell sums into phi / g of the cells (device) */
int omb_fmm_build_direct(const long long *pa, const long long *pb, long long np, long long nent, long long *off,
                         unsigned long long *contrib);
int omb_fmm_direct(const long long *off, const unsigned long long *contrib, const double *center, const double *M,
                   const long long *cell_base, int nleaf, double *phi, double *gx, double *gy, double *gz,
                   void *stream);
int omb_fmm_masses(const double *rho, const long long *cell_base, int nleaf, const double *dx3, double *M,
                   void *stream);
int omb_fmm_upward(const long long *parents, int np, const long long *children, const double *center, double *M,
                   void *stream);
int omb_fmm_m2l(const long long *off, const unsigned long long *contrib, const double *D,
                const unsigned char *cellcell, const double *M, double *L, long long ntarget,
                const long long *targets, const long long *subset /* NULL: all ntarget targets */, void *stream);
/* one of the two M2L passes (part 0: L0..L3, part 1: L4..L19) over its own CSR lists; cellcell = NULL
 * declares a list without cell-cell contributions (part 1 needs none of them: the solver passes it the
 * subsequence of the other contributions, same order, so the result is unchanged bit for bit) */
int omb_fmm_m2l_part(int part, const long long *off, const unsigned long long *contrib, const double *D,
                     const unsigned char *cellcell, const double *M, double *L, long long ntarget,
                     const long long *targets, const long long *subset, double *m0 /* NULL, or nentities doubles:
                     part 0 first copies the monopoles there and reads cell-cell masses from it */,
                     long long nentities, void *stream);
/* pass 0 of two solves over the same lists at once (the stage's density and rho_dot solves): each
 * word and D row read once; m0ab (2 * nentities doubles) receives the two monopoles interleaved per
 * entity; the next pointer is unused (may be NULL) */
int omb_fmm_m2l0_pair(const long long *off, const unsigned long long *contrib, const double *D,
                      const unsigned char *cellcell, const double *Ma, const double *Mb, double *La, double *Lb,
                      long long ntarget, const long long *targets, const long long *subset, double *m0ab,
                      double *unused, long long nentities, void *stream);
int omb_fmm_downward(const long long *parents, int np, const long long *children, const double *center, double *L,
                     void *stream);
int omb_fmm_fields(const double *L, const long long *cell_base, int nleaf, double *phi, double *gx, double *gy,
                   double *gz, void *stream);
/* rho_dot = -div(momentum) (gravity/solver.py:156-168) of the batch's first nleaf leaves of a [6][fstride]
 * state, the neighbour cells gathered like the stage kernel's halo (info = the batch's OmbLeafInfo;
 * halo / nown as OmbStageDesc: peer reads of other GPUs' leaves, or NULL) */
int omb_fmm_rhodot(const double *u, long long fstride, const OmbLeafInfo *info, int bc, int nleaf,
                   const double *const *halo, int nown, double *out, void *stream);
const char *omb_fmm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
