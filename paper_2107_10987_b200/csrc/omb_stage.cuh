// omb_stage.cuh -- the fused RK stage for one RUN of n=8 leaves (a run is
// R >= 1 same-level leaves adjacent along +x, processed as one x-stream).
//
// One CTA per run.  The CTA streams the padded x-planes of the run through
// shared memory and, per plane X, does what the reference does per leaf in
// hydro/step.py:106-144:
//
//   P0  gather plane X+2 (interior + 3-wide halo from neighbour leaves,
//       physical BCs applied exactly as mesh/ghosts.py:115-150) and convert
//       to primitives (reference.py:30-45) into a 5-plane ring
//   P1A/B  for the 9 lines with d.x = 1: PPM monotonised lo/hi on plane X
//       (_core.pyx:61-155) and the central-upwind flux (_core.pyx:180-220)
//       of every interface between planes X-1 and X, for every face axis
//       that uses it -- computed ONCE (the reference evaluates each 1-4x)
//   P2A/B  combine the point fluxes into x-face fluxes with the Simpson rule
//       in the reference's deviation form and summation order
//       (_core.pyx:310-346) and into boundary point values for y/z faces
//   P3/P4  in-plane lines (1, 2, 7, 8): lo/hi and their fluxes
//   P5  finish the y/z faces of plane X-1, start those of plane X -- run in
//       the NEXT plane's P0 phase, beside the conversion
//   P6  conservative update of plane X-2 + sources + dual-energy + floors
//       (step.py:243-288), on the last 64 threads: fluxes/sources/RK during
//       P2A, dual energy/floors/store during P3
// i.e. 7 barriers per plane: P0+P5 | P1A | P2A+P6a | P1B | P2B | P3+P6b | P4.
//
// lo/hi and point fluxes never leave shared memory.  Every phase is a loop
// over independent items separated by barriers; values a thread carries
// across a barrier live in `Hold`.  The kernel is latency-bound per phase
// (one item chain per thread, 16 warps per SM), so items are cut so that the
// longest chain of a phase is short: independent parts of an item go to
// threads that would idle, or one thread carries two independent chains
// instead of two rounds (profiles/README.md).  The same code is compiled for
// the host by the CPU emulation harness (tests/native), which runs each phase
// for every thread index in turn in the kernel's barrier order.
#pragma once
#include "omb_math.cuh"

namespace omb {

constexpr int N = 8, M = 14, PL = M * M;  // padded plane = 196 cells
constexpr int NP = 100;                   // lo/hi positions per plane: [2,12)^2
constexpr int NFACEX = 64;                // x-faces per boundary: [3,11)^2
constexpr int NYF = 72;                   // y-face slots: y in [2,10], z in [3,10]
constexpr int NZF = 72;                   // z-face slots: y in [3,10], z in [2,10]
constexpr int NCOR = 81;                  // corners (a,b) in [2,10]^2

// lines with d.x = 1, in line order; group A = 0..4, group B = 5..8
OMB_HD int dl_line(int dl) { return dl < 5 ? (dl == 0 ? 0 : dl + 2) : dl + 4; }
// in-plane lines 1, 2, 7, 8
OMB_HD int ip_line(int ip) { return ip < 2 ? ip + 1 : ip + 5; }

OMB_HD int pos10(int y, int z) { return (y - 2) * 10 + (z - 2); }

// The items of the reconstruction phases -- (line, position) of a plane --
// come from tables (omb_items.cuh, gen_phase_items.py): ordered by cost (KT
// with 3, 2, 1 axes, then reconstruction only, then the rho/p-only positions
// whose lo/hi feed no flux but count in the reference's positivity fallback),
// then half-warp by half-warp so the 8-byte shared-memory accesses through
// the prim ring (row pitch 14) and the lo/hi / point-flux slots (pitch 10) hit
// distinct banks.  Entry: bits 0-6 pos10, 7-10 the line's index in the phase,
// 11 FULL (all six fields; else rho and p only), 12 KT (the interface from
// the previous plane into this position feeds a face).
}  // namespace omb
#include "omb_items.cuh"
namespace omb {
#ifdef __CUDACC__
static __device__ const unsigned short d_items[OMB_ITEMS_TOTAL] = OMB_ITEMS_ALL;
#endif
static const unsigned short h_items[OMB_ITEMS_TOTAL] = OMB_ITEMS_ALL;
OMB_HD unsigned item_entry(int off, int it) {
#ifdef __CUDA_ARCH__
  return __ldg(&d_items[off + it]);
#else
  return h_items[off + it];
#endif
}
OMB_HD int yslot(int y, int z) { return (y - 2) * 8 + (z - 3); }
OMB_HD int zslot(int y, int z) { return (y - 3) * 9 + (z - 2); }
OMB_HD int cslot(int a, int b) { return (a - 2) * 9 + (b - 2); }
OMB_HD int xface(int y, int z) { return (y - 3) * 8 + (z - 3); }

// RAW channels (point flux of one line for one axis), group A then B
//   A: 0:(0,x) 1:(3,x) 2:(3,y) 3:(4,x) 4:(4,y) 5:(5,x) 6:(5,z) 7:(6,x) 8:(6,z)
//   B: ch = 3*(l-9) + axis
OMB_HD int chA(int l, int axis) {
  switch (l) {
    case 0: return 0;
    case 3: return axis == 0 ? 1 : 2;
    case 4: return axis == 0 ? 3 : 4;
    case 5: return axis == 0 ? 5 : 6;
    default: return axis == 0 ? 7 : 8;  // 6
  }
}
OMB_HD int chB(int l, int axis) { return 3 * (l - 9) + axis; }

// shared-memory layout (doubles)
struct Smem {
  static constexpr int PR = 0;                       // [5][6][14][14] prim ring
  static constexpr int HI = PR + 5 * NF * PL;        // [9][6][100] hi of d.x=1 lines, previous plane
  static constexpr int RAW = HI + 9 * NF * NP;       // union region
  // RAW union members
  static constexpr int RAWA = RAW;                   // [9][6][100]
  static constexpr int RAWB = RAW;                   // [12][6][100]
  static constexpr int LHI = RAW;                    // [4][2][6][100] in-plane lo/hi
  static constexpr int IPCY = RAW + 4 * 2 * NF * NP; // [6][72]
  static constexpr int IPCZ = IPCY + NF * NYF;       // [6][72]
  static constexpr int IPR = IPCZ + NF * NZF;        // [2 lines][2 axes][6][81]
  static constexpr int RAW_END_IP = IPR + 2 * 2 * NF * NCOR;
  static constexpr int RAW_END_B = RAW + 12 * NF * NP;
  static constexpr int RAW_SIZE = (RAW_END_IP > RAW_END_B ? RAW_END_IP : RAW_END_B) - RAW;
  static constexpr int EDEV = RAW + RAW_SIZE;        // [6][64] x-face edge deviation sums
  static constexpr int FX = EDEV + NF * NFACEX;      // [3 ring][6][64] x-face fluxes (centre, then final)
  static constexpr int BYE = FX + 3 * NF * NFACEX;   // [6][72]
  static constexpr int BZE = BYE + NF * NYF;         // [6][72]
  static constexpr int BV = BZE + NF * NZF;          // [2][6][81]
  static constexpr int FP = BV + 2 * NF * NCOR;      // [2][4][6][72]
  static constexpr int FYZ = FP + 2 * 4 * NF * NYF;  // [2][6][72]
  static constexpr int SG0 = FYZ + 2 * NF * NYF;    // [6][196] staged conserved plane (next P0)
  static constexpr int SG6 = SG0 + NF * PL;          // [16][64] staged cur(6) u0(6) grav(4) (next P6)
  static constexpr int LINFO = SG6 + 16 * NFACEX;    // the run's LeafInfo copies [4] (+ leaf ids [4])
  static constexpr int FLIPS = LINFO + 4 * 20 + 2;  // [196] bytes: wall-mirror flips of the SG0 plane
  static constexpr int TOTAL = FLIPS + (PL + 7) / 8;
  static constexpr int BYTES = TOTAL * 8;
};
static_assert(Smem::BYTES <= 232448, "stage shared memory exceeds 227 KB");
static_assert(Smem::RAW_SIZE >= 4 * NF * PL, "prologue staging of planes 0..3 uses the RAW union");

// 8-byte global -> shared asynchronous copy (cp.async / LDGSTS on the GPU,
// an immediate copy in the host emulation), completed by async_wait_all()
// followed by a barrier.
// The host emulation (tests/native/emu_stage.cpp, OMB_EMU_ASYNC) defers each
// copy to the simulated thread's matching wait, like the hardware, so a read
// of staged data before its wait + barrier shows up as a parity failure.
#if !defined(__CUDA_ARCH__) && defined(OMB_EMU_ASYNC)
void omb_emu_async_copy(double* dst, const double* src);
void omb_emu_async_commit();
void omb_emu_async_wait(int keep);
#endif
OMB_HD void async_copy8(double* dst_smem, const double* src) {
#ifdef __CUDA_ARCH__
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src) : "memory");
#elif defined(OMB_EMU_ASYNC)
  omb_emu_async_copy(dst_smem, src);
#else
  *dst_smem = *src;
#endif
}
OMB_HD void async_commit() {
#ifdef __CUDA_ARCH__
  asm volatile("cp.async.commit_group;\n" ::: "memory");
#elif defined(OMB_EMU_ASYNC)
  omb_emu_async_commit();
#endif
}
OMB_HD void async_wait_all() {
#ifdef __CUDA_ARCH__
  asm volatile("cp.async.wait_all;\n" ::: "memory");
#elif defined(OMB_EMU_ASYNC)
  omb_emu_async_wait(0);
#endif
}
// wait until at most the most recently committed group is still in flight
OMB_HD void async_wait_prev() {
#ifdef __CUDA_ARCH__
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
#elif defined(OMB_EMU_ASYNC)
  omb_emu_async_wait(1);
#endif
}

struct LeafInfo {
  int nbr[27];    // batch index of the same-level (or virtual AMR) neighbour per offset, -1 none
  int offmask;    // bit 2a: -a side is a physical wall, bit 2a+1: +a side
  double ox, oy, oz, dx, inv_dx;
  int flags;      // bit 0: export face fluxes to flux[slot]; bit 1: update deferred (reflux);
                  // 16^3/32^3 blocks (blocks.py): bits 2-7 fallback-count range, 8-22 cell offsets
  int slot;
};
constexpr int FLUX_SLOT = 3 * NF * 9 * 8 * 8;  // FX (6,9,8,8) | FY (6,8,9,8) | FZ (6,8,8,9)
constexpr int FXO = 0, FYO = NF * 9 * 64, FZO = 2 * NF * 9 * 64;

static_assert(sizeof(LeafInfo) == 20 * 8, "LeafInfo is 160 bytes (Smem::LINFO)");

// item rounds of every phase: the CUDA kernel runs 512 threads and no phase has more than 500
// items, so each thread takes at most one -- the second round exists only for the host emulation's
// smaller thread counts (256, 384).  (Compiling the second round into the kernel cost 12 B of
// spills and 4-5 %: profiles/r02/ab11_one_round.txt.)
#if defined(__CUDA_ARCH__)
constexpr int ITEM_ROUNDS = 1;
#else
constexpr int ITEM_ROUNDS = 2;
#endif
struct StageArgs {
  const double* ucur;   // [6][L][512] stage input (halo source)
  const double* u0;     // [6][L][512] RK3 u0 snapshot
  double* unext;        // [6][L][512] stage output
  const double* grav;   // [4][L][512] gx gy gz dphi_dt or null
  long long fstride;    // field stride in doubles (>= L*512)
  const LeafInfo* info;
  const int* run_off;   // [nruns+1]
  const int* run_leaf;  // leaves of all runs, consecutive along +x
  const double* dt;     // device scalar
  double a, b;
  double gamma, gm1, eta, inv_gamma, omega;
  double inv_gm1;       // RN(1/gm1), host-computed
  double floor_rho, floor_tau, floor_vmax;
  int bc;               // 0 outflow, 1 reflecting, 2 periodic
  int new_mode, quad, contact;  // quad = new_mode && !override
  unsigned long long* amax_bits;  // per-stage accumulators
  unsigned long long* fallback;
  double* flux;                   // face-flux export slots (AMR), or null
  const double* const* halo;      // multi-GPU: halo slot k's block in its owner's buffer, or null
  int nown;                       // first halo slot
  int scalar;                     // passive-scalar pass: ucur = (rho, s, p, X); X alone is updated
  const double* s_u0;             // scalar pass: X at the step start
  double* s_next;                 // scalar pass: X's stage output
};

// conserved state of padded cell c (local coords in [0,14)^3) of a leaf, as
// mesh/ghosts.py:115-150 fills it for same-level neighbours and physical
// boundaries: region per axis, off-domain axes remapped (mirror for
// reflecting walls with the normal momentum negated, clamp for outflow).
OMB_HD long long gather_addr(const LeafInfo& LI, int bc, int cx, int cy, int cz, int& flipmask) {
  int c[3] = {cx, cy, cz};
  int rd[3], idx[3];
  flipmask = 0;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    int rr = c[a] < 3 ? -1 : (c[a] >= 3 + N ? 1 : 0);
    bool off = rr != 0 && ((LI.offmask >> (2 * a + (rr > 0))) & 1);
    if (off) {
      rd[a] = 0;
      if (bc == 1) {
        idx[a] = rr > 0 ? (N - 1) - (c[a] - 3 - N) : 2 - c[a];
        flipmask |= 1 << a;
      } else {
        idx[a] = rr > 0 ? N - 1 : 0;
      }
    } else {
      rd[a] = rr;
      idx[a] = rr > 0 ? c[a] - 3 - N : (rr < 0 ? c[a] + N - 3 : c[a] - 3);
    }
  }
  int src = LI.nbr[(rd[0] + 1) * 9 + (rd[1] + 1) * 3 + (rd[2] + 1)];
  return (long long)src * 512 + (idx[0] * 64 + idx[1] * 8 + idx[2]);
}

OMB_HD void gather_cell(const double* U, long long fstride, const LeafInfo& LI, int bc, int cx, int cy, int cz,
                        double* u) {
  int flipmask;
  long long base = gather_addr(LI, bc, cx, cy, cz, flipmask);
#pragma unroll
  for (int v = 0; v < NF; v++) u[v] = U[v * fstride + base];
#pragma unroll
  for (int a = 0; a < 3; a++)
    if ((flipmask >> a) & 1) u[1 + a] = -u[1 + a];
}

// values a thread carries across the barrier after P1 (<= 2 items per
// thread: P1 has <= 500 items and the kernel runs >= 256 threads)
struct Hold {
  double h0[NF], h1[NF];
  int s0, s1;
};

struct Stage {
  double* S;
  StageArgs A;
  int run, R, X;
  int ring[5];  // shared-memory offsets of planes X-2 .. X+2 in the prim ring
  const int* leaves;      // the run's leaves (global memory; staged into lids)
  const LeafInfo* LIs;    // shared-memory copies of the run's LeafInfo
  const int* lids;        // shared-memory copies of the run's leaf indices
  // thread-carried reductions
  double amax;
  long long fb;
  // this thread's item of P1A / P1B / P3 (the same every plane), loaded once per CTA: the
  // per-phase table loads sat at the head of each phase's chain (c3 +2.1 %, ab12_preload.txt)
  unsigned item_p1a, item_p1b, item_p3;

  OMB_HD void load_items(int tid) {
    int na = A.new_mode ? OMB_ITEMS_P1A_NEW_N : OMB_ITEMS_P1A_OLD_N;
    int oa = A.new_mode ? OMB_ITEMS_P1A_NEW_OFF : OMB_ITEMS_P1A_OLD_OFF;
    int n3 = A.new_mode ? OMB_ITEMS_P3_NEW_N : OMB_ITEMS_P3_OLD_N;
    int o3 = A.new_mode ? OMB_ITEMS_P3_NEW_OFF : OMB_ITEMS_P3_OLD_OFF;
    item_p1a = tid < na ? item_entry(oa, tid) : 0u;
    item_p1b = tid < OMB_ITEMS_P1B_NEW_N ? item_entry(OMB_ITEMS_P1B_NEW_OFF, tid) : 0u;
    item_p3 = tid < n3 ? item_entry(o3, tid) : 0u;
  }

  OMB_HD double& sm(int off) { return S[off]; }
  OMB_HD double* prp(int x, int v) { return S + Smem::PR + ((x % 5) * NF + v) * PL; }
  OMB_HD void set_plane(int x) {
    X = x;
#pragma unroll
    for (int k = 0; k < 5; k++) ring[k] = Smem::PR + (((x + 3 + k) % 5) * NF) * PL;  // (x-2+k) mod 5
  }
  OMB_HD const double* ringp(int k, int v) const { return S + ring[k] + v * PL; }

  // copy the run's leaf descriptors into shared memory (read every plane;
  // global copies would keep missing the small L1 left beside 230 KB of
  // shared memory).  A barrier must follow.
  OMB_HD void stage_run_info(int tid, int nthr) {
    int* dst = (int*)(S + Smem::LINFO);
    for (int i = tid; i < R * 40; i += nthr) dst[i] = ((const int*)&A.info[leaves[i / 40]])[i % 40];
    if (tid < R) ((int*)(S + Smem::LINFO + 80))[tid] = leaves[tid];
  }
  OMB_HD void bind_run_info() {
    LIs = (const LeafInfo*)(S + Smem::LINFO);
    lids = (const int*)(S + Smem::LINFO + 80);
  }

  // flux export slot of this run's leaf (exporting leaves always run alone)
  OMB_HD double* export_slot() const {
    if (R != 1 || A.flux == nullptr) return nullptr;
    const LeafInfo& LI = LIs[0];
    return (LI.flags & 1) ? A.flux + (long long)LI.slot * FLUX_SLOT : nullptr;
  }

  // how many leaves of the run count position (X, y, z) in the reference's positivity-fallback
  // count: [2,12)^3 per leaf (_core.pyx:143-155); a block of a 16^3 / 32^3 leaf (blocks.py) counts
  // only its share of its leaf's range (flags bits 2-7: the range starts at 3 / ends at 10)
#ifdef __CUDA_ARCH__
  __device__ __noinline__  // only the rare fallback branch calls it: keep its registers out of mono6
#else
  inline
#endif
  int mult(int X, int c0) const {  // c0 = y * M + z (recovered from the stencil address)
    int y = c0 / M, z = c0 % M;
    int c = 0;
    for (int r = 0; r < R; r++) {
      int f = LIs[r].flags;
      bool in = X >= 8 * r + 2 + ((f >> 2) & 1) && X <= 8 * r + 11 - ((f >> 3) & 1) &&
                y >= 2 + ((f >> 4) & 1) && y <= 11 - ((f >> 5) & 1) && z >= 2 + ((f >> 6) & 1) &&
                z <= 11 - ((f >> 7) & 1);
      c += in;
    }
    return c;
  }
  OMB_HD bool interior(int X) const { return X >= 3 && X < 8 * R + 3; }

  // ---- P0: gather + primitives of padded plane X into the ring -----------
  OMB_HD void view_of(int X, int& r, int& lx) const {  // run-local leaf r, padded x in it
    if (X < 3) { r = 0; lx = X; }
    else if (X >= 8 * R + 3) { r = R - 1; lx = X - 8 * (R - 1); }
    else { r = (X - 3) >> 3; lx = 3 + ((X - 3) & 7); }
  }

  OMB_HD void load_plane(int X, int tid, int nthr) {  // synchronous (prologue)
    int r, lx;
    view_of(X, r, lx);
    const LeafInfo& LI = LIs[r];
    for (int it = tid; it < PL; it += nthr) {
      double u[NF], w[NF];
      gather_cell(A.ucur, A.fstride, LI, A.bc, lx, it / M, it % M, u);
      if (A.scalar) prim_cell_scalar(u, w);
      else prim_cell(u, A.gamma, A.gm1, A.eta, w);
#pragma unroll
      for (int v = 0; v < NF; v++) prp(X, v)[it] = w[v];
    }
  }

  // issue the asynchronous gather of padded plane Xn into SG0 (or `stage`)
  OMB_HD void prefetch_plane(int Xn, int tid, int nthr, int stage = Smem::SG0) {
    int r, lx;
    view_of(Xn, r, lx);
    const LeafInfo& LI = LIs[r];
    for (int it = tid; it < PL; it += nthr) {
      int fm;
      long long base = gather_addr(LI, A.bc, lx, it / M, it % M, fm);
      int src = (int)(base >> 9);
      // a neighbour leaf owned by another GPU is read from its owner's buffer over NVLink
      const double* p = (A.halo != nullptr && src >= A.nown) ? A.halo[src - A.nown] + (base & 511) : A.ucur + base;
#pragma unroll
      for (int v = 0; v < NF; v++) async_copy8(S + stage + v * PL + it, p + v * A.fstride);
      if (stage == Smem::SG0) ((unsigned char*)(S + Smem::FLIPS))[it] = (unsigned char)fm;  // for P0
    }
  }

  // P0: primitives of the staged plane Xn into the ring (wall flips recorded
  // by the prefetch for the SG0 plane, re-derived for the prologue's planes)
  OMB_HD void convert_plane(int Xn, int tid, int nthr, int stage = Smem::SG0) {
    int r, lx;
    view_of(Xn, r, lx);
    const LeafInfo& LI = LIs[r];
    for (int it = tid; it < PL; it += nthr) {
      int fm;
      if (stage == Smem::SG0) fm = ((const unsigned char*)(S + Smem::FLIPS))[it];  // recorded by the prefetch
      else gather_addr(LI, A.bc, lx, it / M, it % M, fm);
      double u[NF], w[NF];
#pragma unroll
      for (int v = 0; v < NF; v++) u[v] = S[stage + v * PL + it];
#pragma unroll
      for (int a = 0; a < 3; a++)
        if ((fm >> a) & 1) u[1 + a] = -u[1 + a];
      if (A.scalar) prim_cell_scalar(u, w);
      else prim_cell(u, A.gamma, A.gm1, A.eta, w);
#pragma unroll
      for (int v = 0; v < NF; v++) prp(Xn, v)[it] = w[v];
    }
  }

  // issue the asynchronous loads of cur, u0 (and gravity) of plane Xc's cells into SG6
  OMB_HD void prefetch_update(int Xc, int tid, int nthr) {
    int r = (Xc - 3) >> 3, lx = (Xc - 3) & 7;
    long long base = (long long)lids[r] * 512 + lx * 64;
    bool grav = A.grav != nullptr;
    for (int it = tid; it < NFACEX; it += nthr) {
      long long cell = base + it;  // (y-3)*8 + (z-3) == it
#pragma unroll
      for (int v = 0; v < NF; v++) {
        async_copy8(S + Smem::SG6 + v * NFACEX + it, A.ucur + v * A.fstride + cell);
        const double* u0 = (A.scalar && v == NF - 1) ? A.s_u0 + cell : A.u0 + v * A.fstride + cell;
        async_copy8(S + Smem::SG6 + (NF + v) * NFACEX + it, u0);
      }
      if (grav)
#pragma unroll
        for (int k = 0; k < 4; k++) async_copy8(S + Smem::SG6 + (2 * NF + k) * NFACEX + it, A.grav + k * A.fstride + cell);
    }
  }

  // monotonised lo/hi of 6 fields at (X, y, z) along line l, with contact
  // steepening and the positivity fallback (_core.pyx:61-155 for one cell)
  // full = false: only rho and p (fields 0, 4) are reconstructed -- enough
  // for the fallback count when nothing consumes this cell's lo/hi
  OMB_HD void mono6(int l, int X, int y, int z, double* lo, double* hi, bool full = true) {
    int dx = ldx(l), dy = ldy(l), dz = ldz(l);
    int c0 = y * M + z, dd = dy * M + dz;
    int ad[5];
#pragma unroll
    for (int k = 0; k < 5; k++) ad[k] = (dx ? ring[k] : ring[2]) + c0 + (k - 2) * dd;
    double rr[5] = {0, 0, 0, 0, 0}, pm1 = 0, pp1 = 0;
    // two fields at a time -- (rho, p), (vx, vy), (vz, tau): their loads and interface values
    // straight-line, so the two chains interleave; the flat shortcut per pair (A/B on one box:
    // c3 +1.4 %, c2 -0.3 %; with select-based monotonisation too: c3 +1.3 %, c2 -2.5 %)
#pragma unroll
    for (int pi = 0; pi < 3; pi++) {
      const int va = pi == 0 ? 0 : (pi == 1 ? 1 : 3), vb = pi == 0 ? 4 : (pi == 1 ? 2 : 5);
      if (!full && pi > 0) {
        lo[va] = hi[va] = lo[vb] = hi[vb] = 0.0;
        continue;
      }
      double sa[5], sb[5];
#pragma unroll
      for (int k = 0; k < 5; k++) {
        sa[k] = S[ad[k] + va * PL];
        sb[k] = S[ad[k] + vb * PL];
      }
      bool fa = sa[0] == sa[2] && sa[1] == sa[2] && sa[3] == sa[2] && sa[4] == sa[2];
      bool fb = sb[0] == sb[2] && sb[1] == sb[2] && sb[3] == sb[2] && sb[4] == sb[2];
      if (fa && fb) {
        lo[va] = hi[va] = sa[2];
        lo[vb] = hi[vb] = sb[2];
      } else {  // a flat stencil through the full path gives lo = hi = a as well (clamp, extremum)
        double la = iface(sa[0], sa[1], sa[2], sa[3]), ha = iface(sa[1], sa[2], sa[3], sa[4]);
        double lb = iface(sb[0], sb[1], sb[2], sb[3]), hb = iface(sb[1], sb[2], sb[3], sb[4]);
        mono(sa[2], la, ha);
        mono(sb[2], lb, hb);
        lo[va] = la;
        hi[va] = ha;
        lo[vb] = lb;
        hi[vb] = hb;
      }
      if (pi == 0) {
#pragma unroll
        for (int k = 0; k < 5; k++) rr[k] = sa[k];
        pm1 = sb[1];
        pp1 = sb[3];
      }
    }
    if (A.contact) contact_steepen(rr, pm1, pp1, A.gamma, lo[0], hi[0]);
    if (lo[0] <= 0.0 || lo[4] <= 0.0) {
      fb += mult(X, ad[2] - ring[2]);
#pragma unroll
      for (int v = 0; v < NF; v++) lo[v] = S[ad[2] + v * PL];
    }
    if (hi[0] <= 0.0 || hi[4] <= 0.0) {
      fb += mult(X, ad[2] - ring[2]);
#pragma unroll
      for (int v = 0; v < NF; v++) hi[v] = S[ad[2] + v * PL];
    }
  }

  OMB_HD void kt_into(const KtState& sP, const KtState& sQ, int l, int axis, double* dst, int stride) {
    int d = axis == 0 ? ldx(l) : (axis == 1 ? ldy(l) : ldz(l));
    // the canonical line direction runs against the face normal: the stored
    // lo/hi states swap roles (_core.pyx:299-306)
    bool flip = d < 0;
    double sp = kt_axis(sP, sQ, axis, flip, dst, stride);
    if (sp > amax) amax = sp;
  }

  // ---- P1: boundary lines (d.x = 1) of group g on plane X ----------------
  OMB_HD void boundary_lines(int g, int tid, int nthr, Hold& h) {
    int dl0 = g == 0 ? 0 : 5;
    int toff = g == 0 ? (A.new_mode ? OMB_ITEMS_P1A_NEW_OFF : OMB_ITEMS_P1A_OLD_OFF) : OMB_ITEMS_P1B_NEW_OFF;
    int nitems = g == 0 ? (A.new_mode ? OMB_ITEMS_P1A_NEW_N : OMB_ITEMS_P1A_OLD_N) : OMB_ITEMS_P1B_NEW_N;
    h.s0 = h.s1 = -1;
#pragma unroll 1
    for (int k = 0; k < ITEM_ROUNDS; k++) {
      int it = tid + k * nthr;
      if (it >= nitems) break;
      unsigned e = k == 0 ? (g == 0 ? item_p1a : item_p1b) : item_entry(toff, it);
      int pos = e & 127, dl = dl0 + ((e >> 7) & 15);
      int l = dl_line(dl);
      int y = 2 + pos / 10, z = 2 + pos % 10;
      double lo[NF], hi[NF];
      mono6(l, X, y, z, lo, hi, (e >> 11) & 1);
      if (k == 0) {
#pragma unroll
        for (int v = 0; v < NF; v++) h.h0[v] = hi[v];
        h.s0 = dl * NF * NP + pos;
      } else {
#pragma unroll
        for (int v = 0; v < NF; v++) h.h1[v] = hi[v];
        h.s1 = dl * NF * NP + pos;
      }
      // the interface (X-1, P) -> (X, pos), P = pos - d, feeds a face of an interior cell
      bool kt = X >= 3 && (A.quad || l == 0) && ((e >> 12) & 1);
      if (!kt) continue;
      int pp = pos - ldy(l) * 10 - ldz(l);
      double hp[NF];
#pragma unroll
      for (int v = 0; v < NF; v++) hp[v] = S[Smem::HI + (dl * NF + v) * NP + pp];
      KtState sP, sQ;
      kt_state(hp, A.gamma, A.gm1, A.inv_gm1, sP);
      kt_state(lo, A.gamma, A.gm1, A.inv_gm1, sQ);
      // axes served by this line: x always; y for lines 3,4; z for 5,6; all for 9..12
      int ax_second = (l == 3 || l == 4) ? 1 : 2;
      int nax = l == 0 ? 1 : (l >= 9 ? 3 : 2);
#pragma unroll
      for (int q = 0; q < 3; q++) {
        if (q >= nax) break;
        int ax = q == 0 ? 0 : (l >= 9 ? q : ax_second);
        double* dst = g == 0 ? S + Smem::RAWA + (chA(l, ax) * NF) * NP + pp : S + Smem::RAWB + (chB(l, ax) * NF) * NP + pp;
        kt_into(sP, sQ, l, ax, dst, NP);
      }
    }
  }

  OMB_HD void store_hi(const Hold& h) {
    if (h.s0 >= 0) {
#pragma unroll
      for (int v = 0; v < NF; v++) S[Smem::HI + h.s0 + v * NP] = h.h0[v];
    }
    if (h.s1 >= 0) {
#pragma unroll
      for (int v = 0; v < NF; v++) S[Smem::HI + h.s1 + v * NP] = h.h1[v];
    }
  }

  OMB_HD double rawA(int l, int ax, int v, int y, int z) { return S[Smem::RAWA + (chA(l, ax) * NF + v) * NP + pos10(y, z)]; }
  OMB_HD double rawB(int l, int ax, int v, int y, int z) { return S[Smem::RAWB + (chB(l, ax) * NF + v) * NP + pos10(y, z)]; }
  OMB_HD double vertex(int ax, int v, int a, int b) {
    return vert_acc(rawB(9, ax, v, a, b), rawB(10, ax, v, a, b + 1), rawB(11, ax, v, a + 1, b),
                    rawB(12, ax, v, a + 1, b + 1));
  }

  // ---- P2A: x-face centre + edges, boundary edge points for y/z faces -----
  // One item per (field, slot): the x face (slots < 64) and the y/z boundary
  // edge points of that slot -- 432 items, one round, independent chains.
  OMB_HD void combine_A(int tid, int nthr) {
    double* FXc = S + Smem::FX + (X % 3) * NF * NFACEX;
    int ntot = A.quad ? NF * NYF : NF * NFACEX;
    for (int it = tid; it < ntot; it += nthr) {
      // per field: the 64 x-faces / y / z boundary edges of 8 x 8 blocks as paired-row half-warps
      // (bank-free through the pitch-10 point-flux slots), the 8 leftover edges of each after
      int v, r, yb, zb, yc, zc, f = NFACEX;
      if (it < NF * NFACEX) {
        v = it >> 6;
        r = it & 63;
        int yy = (r >> 4) + 4 * ((r >> 3) & 1), zz = r & 7;
        f = yy * 8 + zz;  // x-face (3 + yy, 3 + zz)
        yb = 2 + yy; zb = 3 + zz; yc = 3 + yy; zc = 2 + zz;
      } else {
        v = (it - NF * NFACEX) >> 3;
        r = (it - NF * NFACEX) & 7;
        yb = 10; zb = 3 + r; yc = 3 + r; zc = 10;
      }
      if (f < NFACEX) {
        int y = 3 + f / 8, z = 3 + f % 8;
        double C = rawA(0, 0, v, y, z);
        FXc[v * NFACEX + f] = C;
        if (!A.quad) {
          if (double* ex = export_slot()) ex[FXO + (v * 9 + (X - 3)) * 64 + f] = C;
        } else {
          double e0 = edge_acc(rawA(5, 0, v, y, z - 1), rawA(6, 0, v, y, z));
          double e1 = edge_acc(rawA(5, 0, v, y, z), rawA(6, 0, v, y, z + 1));
          double e2 = edge_acc(rawA(3, 0, v, y - 1, z), rawA(4, 0, v, y, z));
          double e3 = edge_acc(rawA(3, 0, v, y, z), rawA(4, 0, v, y + 1, z));
          S[Smem::EDEV + v * NFACEX + f] = (pdev_edge(e0, C) + pdev_edge(e1, C)) + (pdev_edge(e2, C) + pdev_edge(e3, C));
        }
      }
      if (A.quad) {  // y-edge point (yb, zb) of y faces, z-edge point (yc, zc) of z faces
        S[Smem::BYE + v * NYF + yslot(yb, zb)] = edge_acc(rawA(3, 1, v, yb, zb), rawA(4, 1, v, yb + 1, zb));
        S[Smem::BZE + v * NZF + zslot(yc, zc)] = edge_acc(rawA(5, 2, v, yc, zc), rawA(6, 2, v, yc, zc + 1));
      }
    }
  }

  // ---- P2B: x-face vertices -> final x flux; vertex points for y/z -------
  // One item per (field, corner): both y/z vertex points of the corner and
  // (corners < 64) the final x face -- 486 items, one round.
  OMB_HD void combine_B(int tid, int nthr) {
    double* FXc = S + Smem::FX + (X % 3) * NF * NFACEX;
    for (int it = tid; it < NF * NCOR; it += nthr) {
      // per field: the x-faces and an 8 x 8 block of corners as paired-row half-warps, then the
      // 17 corners left (a = 10 or b = 10)
      int v, c, f = NFACEX;
      if (it < NF * NFACEX) {
        v = it >> 6;
        int r = it & 63, yy = (r >> 4) + 4 * ((r >> 3) & 1), zz = r & 7;
        f = yy * 8 + zz;
        c = yy * 9 + zz;  // corner (2 + yy, 2 + zz)
      } else {
        v = (it - NF * NFACEX) / 17;
        int r = (it - NF * NFACEX) % 17;
        c = r < 9 ? 8 * 9 + r : (r - 9) * 9 + 8;
      }
      if (f < NFACEX) {
        int y = 3 + f / 8, z = 3 + f % 8;
        double C = FXc[v * NFACEX + f];
        double edev = S[Smem::EDEV + v * NFACEX + f];
        double vdev = (pdev_vert(vertex(0, v, y - 1, z - 1), C) + pdev_vert(vertex(0, v, y - 1, z), C)) +
                      (pdev_vert(vertex(0, v, y, z - 1), C) + pdev_vert(vertex(0, v, y, z), C));
        double Fv = face_final(C, edev, vdev);
        FXc[v * NFACEX + f] = Fv;
        if (double* ex = export_slot()) ex[FXO + (v * 9 + (X - 3)) * 64 + f] = Fv;
      }
#pragma unroll
      for (int ax = 0; ax < 2; ax++)
        S[Smem::BV + (ax * NF + v) * NCOR + c] = vertex(1 + ax, v, 2 + c / 9, 2 + c % 9);
    }
  }

  // ---- P3: in-plane lines 1, 2, 7, 8 on plane X --------------------------
  OMB_HD void inplane_lines(int tid, int nthr) {
    int toff = A.new_mode ? OMB_ITEMS_P3_NEW_OFF : OMB_ITEMS_P3_OLD_OFF;
    int nitems = A.new_mode ? OMB_ITEMS_P3_NEW_N : OMB_ITEMS_P3_OLD_N;
#pragma unroll 1
    for (int it = tid; it < nitems && it < tid + ITEM_ROUNDS * nthr; it += nthr) {
      unsigned e = it == tid ? item_p3 : item_entry(toff, it);
      int pos = e & 127, ip = (e >> 7) & 15, l = ip_line(ip);
      int y = 2 + pos / 10, z = 2 + pos % 10;
      double lo[NF], hi[NF];
      mono6(l, X, y, z, lo, hi, (e >> 11) & 1);
#pragma unroll
      for (int v = 0; v < NF; v++) {
        S[Smem::LHI + ((ip * 2 + 0) * NF + v) * NP + pos] = lo[v];
        S[Smem::LHI + ((ip * 2 + 1) * NF + v) * NP + pos] = hi[v];
      }
    }
  }

  OMB_HD void lhi_state(int ip, int side, int y, int z, KtState& s) {
    double w[NF];
#pragma unroll
    for (int v = 0; v < NF; v++) w[v] = S[Smem::LHI + ((ip * 2 + side) * NF + v) * NP + pos10(y, z)];
    kt_state(w, A.gamma, A.gm1, A.inv_gm1, s);
  }

  // ---- P4: in-plane fluxes (y/z face centres, y/z edge points) -----------
  // The two axes of an edge point go to two threads (each recomputes the two
  // states): 468 single-axis items, one round on 512 threads.
  OMB_HD void inplane_fluxes(int tid, int nthr) {
    int ntot = NYF + NZF + (A.quad ? 4 * NCOR : 0);
    for (int it = tid; it < ntot; it += nthr) {
      int ip, py, pz, qy, qz, l, ax0, nax, stride;
      double* dst;
      // bank-free order: 8 x 8 blocks as half-warps of (8 z of row y, row y + 4) -- the lo/hi slot
      // pitch 10 puts them 8 doubles apart mod 16 -- then the rows / columns left over
      if (it < 64 || (it >= 128 && it < 136)) {  // y-face centre (y in [2,10], z in [3,10])
        py = it < 64 ? 2 + (it >> 4) + 4 * ((it >> 3) & 1) : 10;
        pz = 3 + (it & 7);
        int sy = (py - 2) * 8 + (pz - 3);
        ip = 0; l = 1; qy = py + 1; qz = pz;
        ax0 = 1; nax = 1; dst = S + Smem::IPCY + sy; stride = NYF;
      } else if (it < 144) {  // z-face centre (y in [3,10], z in [2,10])
        int r = it - 64;
        if (it < 128) { py = 3 + (r >> 4) + 4 * ((r >> 3) & 1); pz = 2 + (r & 7); }
        else { py = 3 + (it - 136); pz = 10; }
        int s2 = (py - 3) * 9 + (pz - 2);
        ip = 1; l = 2; qy = py; qz = pz + 1;
        ax0 = 2; nax = 1; dst = S + Smem::IPCZ + s2; stride = NZF;
      } else {  // edge points: each (axis k, line li) group's 8 x 8 block, then the 4 x 17 left
        int j = it - 144, grp, a, b;
        if (j < 256) {
          grp = j >> 6;
          int r = j & 63;
          a = 2 + (r >> 4) + 4 * ((r >> 3) & 1);
          b = 2 + (r & 7);
        } else {
          grp = (j - 256) / 17;
          int r = (j - 256) % 17;
          a = r < 9 ? 10 : 2 + (r - 9);
          b = r < 9 ? 2 + r : 10;
        }
        int k = grp >> 1, li = grp & 1, c = (a - 2) * 9 + (b - 2);
        l = li == 0 ? 7 : 8;
        ip = li + 2;
        py = a; pz = li == 0 ? b : b + 1;
        qy = py + 1; qz = pz + ldz(l);
        ax0 = 1 + k; nax = 1; dst = S + Smem::IPR + ((li * 2 + k) * NF) * NCOR + c; stride = NCOR;
      }
      KtState sP, sQ;
      lhi_state(ip, 1, py, pz, sP);
      lhi_state(ip, 0, qy, qz, sQ);
#pragma unroll 1
      for (int k = 0; k < nax; k++) kt_into(sP, sQ, l, ax0 + k, dst + k * NF * NCOR, stride);
    }
  }

  OMB_HD double ipr(int li, int axi, int v, int a, int b) { return S[Smem::IPR + ((li * 2 + axi) * NF + v) * NCOR + cslot(a, b)]; }
  OMB_HD double bv(int axi, int v, int a, int b) { return S[Smem::BV + (axi * NF + v) * NCOR + cslot(a, b)]; }

  // ---- P5: finish y/z faces of plane X-1, start those of plane X ---------
  // (thread tid takes items from (tid - first) mod nthr on: P0 runs this
  // beside the conversion, which occupies threads [0, first))
  OMB_HD void faces_yz(int tid, int nthr, int first = 0) {
    bool fin = interior(X - 1), start = interior(X);
    bool q = A.quad;
    // (threads below `first` take the last items: tried instead, only threads from `first` on
    // with two items on some -- 3 % slower, profiles/r02/ab8_faces_split.txt)
    int t0 = tid - first, step = nthr;
    if (t0 < 0) t0 += nthr;
    // one item = the y face and the z face of slot (v, s): 432 items, one
    // round on 512 threads, two independent chains per thread
    for (int it = t0; it < NF * NYF; it += step)
#pragma unroll
    for (int zf = 0; zf < 2; zf++) {
      int v = it / NYF, s = it % NYF;  // NYF == NZF
      int y, z;
      if (!zf) { y = 2 + s / 8; z = 3 + s % 8; }
      else { y = 3 + s / 9; z = 2 + s % 9; }
      double* fp = S + Smem::FP + (zf * 4 * NF) * NYF;
      double edge_b = q ? S[(zf ? Smem::BZE : Smem::BYE) + v * NYF + s] : 0.0;
      // corners of this face on the boundary plane X-1/2 (and in-plane edges)
      int ca0, cb0, ca1, cb1;  // first / second corner (V0,V1 or V2,V3 order)
      if (!zf) { ca0 = y; cb0 = z - 1; ca1 = y; cb1 = z; }
      else { ca0 = y - 1; cb0 = z; ca1 = y; cb1 = z; }
      if (fin) {
        double C = fp[(0 * NF + v) * NYF + s];
        double F = C;
        if (q) {
          double S01 = fp[(1 * NF + v) * NYF + s], pd2 = fp[(2 * NF + v) * NYF + s];
          double T01 = fp[(3 * NF + v) * NYF + s];
          double pd3 = pdev_edge(edge_b, C);
          double pv2 = pdev_vert(bv(zf, v, ca0, cb0), C), pv3 = pdev_vert(bv(zf, v, ca1, cb1), C);
          F = face_final(C, S01 + (pd2 + pd3), T01 + (pv2 + pv3));
        }
        S[Smem::FYZ + (zf * NF + v) * NYF + s] = F;
        if (double* ex = export_slot()) {
          int xi = X - 1 - 3;  // cell plane being finalised
          if (!zf) ex[FYO + ((v * 8 + xi) * 9 + (y - 2)) * 8 + (z - 3)] = F;
          else ex[FZO + ((v * 8 + xi) * 8 + (y - 3)) * 9 + (z - 2)] = F;
        }
      }
      if (start) {
        double C = S[(zf ? Smem::IPCZ : Smem::IPCY) + v * NYF + s];
        fp[(0 * NF + v) * NYF + s] = C;
        if (q) {
          double e0 = edge_acc(ipr(0, zf, v, ca0, cb0), ipr(1, zf, v, ca0, cb0));
          double e1 = edge_acc(ipr(0, zf, v, ca1, cb1), ipr(1, zf, v, ca1, cb1));
          fp[(1 * NF + v) * NYF + s] = pdev_edge(e0, C) + pdev_edge(e1, C);
          fp[(2 * NF + v) * NYF + s] = pdev_edge(edge_b, C);
          fp[(3 * NF + v) * NYF + s] = pdev_vert(bv(zf, v, ca0, cb0), C) + pdev_vert(bv(zf, v, ca1, cb1), C);
        }
      }
    }
  }

  // ---- P6: update the cells of plane X-1 ---------------------------------
  // The update split in two so each half hides beside a phase's own items:
  // part A (fluxes, sources, RK combination) leaves the 6 combined values in
  // SG6's `cur` rows (consumed by then); part B (dual energy, floors) stores.
  OMB_HD UpdateParams update_params() const {
    UpdateParams P;
    P.dt = *A.dt; P.a = A.a; P.b = A.b;
    P.gamma = A.gamma; P.eta = A.eta; P.inv_gamma = A.inv_gamma; P.omega = A.omega;
    P.floor_rho = A.floor_rho; P.floor_tau = A.floor_tau; P.floor_vmax = A.floor_vmax;
    P.has_grav = A.grav != nullptr;
    P.has_src = (A.omega != 0.0) || P.has_grav;
    return P;
  }
  OMB_HD void update_plane_a(int tid, int nthr) {
    int Xc = X - 1;
    int r = (Xc - 3) >> 3, lx = (Xc - 3) & 7;
    const LeafInfo& LI = LIs[r];
    if (LI.flags & 2) return;
    const double* FXlo = S + Smem::FX + (Xc % 3) * NF * NFACEX;
    const double* FXhi = S + Smem::FX + (X % 3) * NF * NFACEX;
    const UpdateParams P = update_params();
    for (int it = tid; it < NFACEX; it += nthr) {
      int y = 3 + it / 8, z = 3 + it % 8;
      double u[NF], u0[NF], rr[NF], nw[NF], g[4] = {0, 0, 0, 0};
#pragma unroll
      for (int v = 0; v < NF; v++) {
        u[v] = S[Smem::SG6 + v * NFACEX + it];
        u0[v] = S[Smem::SG6 + (NF + v) * NFACEX + it];
        double dfx = FXhi[v * NFACEX + it] - FXlo[v * NFACEX + it];
        double dfy = S[Smem::FYZ + v * NYF + yslot(y, z)] - S[Smem::FYZ + v * NYF + yslot(y - 1, z)];
        double dfz = S[Smem::FYZ + (NF + v) * NYF + zslot(y, z)] - S[Smem::FYZ + (NF + v) * NYF + zslot(y, z - 1)];
        double t = 0.0 - dfx * LI.inv_dx;
        t = t - dfy * LI.inv_dx;
        t = t - dfz * LI.inv_dx;
        rr[v] = t;
      }
      if (P.has_grav)
#pragma unroll
        for (int k = 0; k < 4; k++) g[k] = S[Smem::SG6 + (2 * NF + k) * NFACEX + it];
      double xc = LI.ox + LI.dx * (double)(lx + ((LI.flags >> 8) & 31));  // origin + dx * i of the leaf
      double yc = LI.oy + LI.dx * (double)(y - 3 + ((LI.flags >> 13) & 31));
      update_cell_rk(P, u, u0, rr, xc, yc, g, nw);
#pragma unroll
      for (int v = 0; v < NF; v++) S[Smem::SG6 + v * NFACEX + it] = nw[v];
    }
  }
  OMB_HD void update_plane_b(int tid, int nthr) {
    int Xc = X - 1;
    int r = (Xc - 3) >> 3, lx = (Xc - 3) & 7;
    int leaf = lids[r];
    const LeafInfo& LI = LIs[r];
    if (LI.flags & 2) return;
    const UpdateParams P = update_params();
    for (int it = tid; it < NFACEX; it += nthr) {
      long long cell = (long long)leaf * 512 + lx * 64 + it;  // (y-3)*8 + (z-3) == it
      double nw[NF], out[NF];
#pragma unroll
      for (int v = 0; v < NF; v++) nw[v] = S[Smem::SG6 + v * NFACEX + it];
      if (A.scalar) {  // the passive scalar: no dual energy, no floors
        A.s_next[cell] = nw[NF - 1];
        continue;
      }
      update_cell_fin(P, nw, out);
#pragma unroll
      for (int v = 0; v < NF; v++) A.unext[v * A.fstride + cell] = out[v];
    }
  }

  OMB_HD void update_plane(int tid, int nthr) {
    int Xc = X - 1;
    int r = (Xc - 3) >> 3, lx = (Xc - 3) & 7;
    int leaf = lids[r];
    const LeafInfo& LI = LIs[r];
    if (LI.flags & 2) return;  // coarse leaf on a coarse/fine face: omb_reflux_update does it
    const double* FXlo = S + Smem::FX + (Xc % 3) * NF * NFACEX;
    const double* FXhi = S + Smem::FX + (X % 3) * NF * NFACEX;
    UpdateParams P;
    P.dt = *A.dt; P.a = A.a; P.b = A.b;
    P.gamma = A.gamma; P.eta = A.eta; P.inv_gamma = A.inv_gamma; P.omega = A.omega;
    P.floor_rho = A.floor_rho; P.floor_tau = A.floor_tau; P.floor_vmax = A.floor_vmax;
    P.has_grav = A.grav != nullptr;
    P.has_src = (A.omega != 0.0) || P.has_grav;
    for (int it = tid; it < NFACEX; it += nthr) {
      if (it < 0) continue;
      int y = 3 + it / 8, z = 3 + it % 8;
      long long cell = (long long)leaf * 512 + lx * 64 + (y - 3) * 8 + (z - 3);
      double u[NF], u0[NF], rr[NF], out[NF], g[4] = {0, 0, 0, 0};
#pragma unroll
      for (int v = 0; v < NF; v++) {
        u[v] = S[Smem::SG6 + v * NFACEX + it];
        u0[v] = S[Smem::SG6 + (NF + v) * NFACEX + it];
        double dfx = FXhi[v * NFACEX + it] - FXlo[v * NFACEX + it];
        double dfy = S[Smem::FYZ + v * NYF + yslot(y, z)] - S[Smem::FYZ + v * NYF + yslot(y - 1, z)];
        double dfz = S[Smem::FYZ + (NF + v) * NYF + zslot(y, z)] - S[Smem::FYZ + (NF + v) * NYF + zslot(y, z - 1)];
        double t = 0.0 - dfx * LI.inv_dx;
        t = t - dfy * LI.inv_dx;
        t = t - dfz * LI.inv_dx;
        rr[v] = t;
      }
      if (P.has_grav)
#pragma unroll
        for (int k = 0; k < 4; k++) g[k] = S[Smem::SG6 + (2 * NF + k) * NFACEX + it];
      double xc = LI.ox + LI.dx * (double)(lx + ((LI.flags >> 8) & 31));  // origin + dx * i of the leaf
      double yc = LI.oy + LI.dx * (double)(y - 3 + ((LI.flags >> 13) & 31));
      if (A.scalar) {
        update_cell_rk(P, u, u0, rr, xc, yc, g, out);
        A.s_next[cell] = out[NF - 1];
        continue;
      }
      update_cell(P, u, u0, rr, xc, yc, g, out);
#pragma unroll
      for (int v = 0; v < NF; v++) A.unext[v * A.fstride + cell] = out[v];
    }
  }

};

// ---------------------------------------------------------------------------
// AMR ghost regions (mesh/ghosts.py:62-112, mesh/transfer.py:13-64)
// ---------------------------------------------------------------------------
// minmod of the forward / backward differences (transfer.py:13-35); b is the
// coarse row inside the clipped sub-block [0, nb): edge cells see the
// linear-extrapolation pad, so their slope is one-sided
OMB_HD double amr_minmod(double a, double b) {
  double pick = fabs(a) < fabs(b) ? a : b;
  return a * b > 0.0 ? pick : 0.0;
}
OMB_HD double amr_slope(double bm, double b0, double bp, int j, int nb) {
  if (nb == 1) return 0.0;
  double fwd, bwd;
  if (j == 0) {
    bwd = b0 - (2.0 * b0 - bp);  // padded lo = 2*b[0] - b[1]
    fwd = bp - b0;
  } else if (j == nb - 1) {
    fwd = (2.0 * b0 - bm) - b0;  // padded hi = 2*b[nb-1] - b[nb-2]
    bwd = b0 - bm;
  } else {
    fwd = bp - b0;
    bwd = b0 - bm;
  }
  return amr_minmod(fwd, bwd);
}

// value (field v) of block cell (b0,b1,b2) of AMR task t, reading interiors of U
OMB_HD double amr_cell(const double* U, long long fstride, const int* t, int v, const int* b) {
  const double* Uv = U + v * fstride;
  if (t[0] == 0) {  // coarse neighbour: prolong the clipped coarse sub-block
    const double* C = Uv + (long long)t[5] * 512;
    int j[3], p[3], nb[3], cg[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      int fi = t[12 + a] + b[a];  // index in the prolonged sub-block
      j[a] = fi >> 1;
      p[a] = fi & 1;
      nb[a] = t[9 + a] - t[6 + a];
      cg[a] = t[6 + a] + j[a];
    }
    auto at = [&](int x, int y, int z) { return C[x * 64 + y * 8 + z]; };
    double c0 = at(cg[0], cg[1], cg[2]);
    double sx = amr_slope(j[0] > 0 ? at(cg[0] - 1, cg[1], cg[2]) : 0.0, c0,
                          j[0] < nb[0] - 1 ? at(cg[0] + 1, cg[1], cg[2]) : 0.0, j[0], nb[0]);
    double sy = amr_slope(j[1] > 0 ? at(cg[0], cg[1] - 1, cg[2]) : 0.0, c0,
                          j[1] < nb[1] - 1 ? at(cg[0], cg[1] + 1, cg[2]) : 0.0, j[1], nb[1]);
    double sz = amr_slope(j[2] > 0 ? at(cg[0], cg[1], cg[2] - 1) : 0.0, c0,
                          j[2] < nb[2] - 1 ? at(cg[0], cg[1], cg[2] + 1) : 0.0, j[2], nb[2]);
    return ((c0 + sx * (p[0] ? 0.25 : -0.25)) + sy * (p[1] ? 0.25 : -0.25)) + sz * (p[2] ? 0.25 : -0.25);
  }
  // fine neighbours: restriction of the covering child's 2x2x2 cells
  int c[3], k[3], f[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    c[a] = b[a] + (t[1 + a] == -1 ? N - 3 : 0);  // coarse cell within the region's pos block
    k[a] = c[a] >= N / 2 ? 1 : 0;
    f[a] = 2 * c[a] - k[a] * N;
  }
  // the covering child: a select over the 8 (a runtime index into t would send the caller's
  // register copy of the task to local memory)
  const int ci = k[0] + 2 * k[1] + 4 * k[2];
  int child = t[5];
#pragma unroll
  for (int j = 1; j < 8; j++) child = ci == j ? t[5 + j] : child;
  const double* F = Uv + (long long)child * 512;
  auto at = [&](int x, int y, int z) { return F[(f[0] + x) * 64 + (f[1] + y) * 8 + (f[2] + z)]; };
  return 0.125 * (((at(0, 0, 0) + at(1, 0, 0)) + (at(0, 1, 0) + at(1, 1, 0))) +
                  ((at(0, 0, 1) + at(1, 0, 1)) + (at(0, 1, 1) + at(1, 1, 1))));
}

// reflux substitution of one task into this leaf's flux set F (step.py:222-241):
// the coarse face block gets 0.25*((f00+f10)+(f01+f11)) of the fine child's face fluxes
OMB_HD int flux_index(int ax, int v, int fi, int s1, int s2) {
  if (ax == 0) return FXO + ((v * 9 + fi) * 8 + s1) * 8 + s2;
  if (ax == 1) return FYO + ((v * 8 + s1) * 9 + fi) * 8 + s2;
  return FZO + ((v * 8 + s1) * 8 + s2) * 9 + fi;
}
OMB_HD void reflux_apply(double* F, const double* flux, const int* rt, int tid, int nthr) {
  int ax = rt[0], side = rt[1], k1 = rt[3], k2 = rt[4];
  const double* fine = flux + (long long)rt[2] * FLUX_SLOT;
  int cface = side > 0 ? N : 0, fface = side > 0 ? 0 : N;
  for (int i = tid; i < NF * 16; i += nthr) {
    int v = i / 16, a = (i / 4) % 4, b = i % 4;
    double f00 = fine[flux_index(ax, v, fface, 2 * a, 2 * b)], f10 = fine[flux_index(ax, v, fface, 2 * a + 1, 2 * b)];
    double f01 = fine[flux_index(ax, v, fface, 2 * a, 2 * b + 1)];
    double f11 = fine[flux_index(ax, v, fface, 2 * a + 1, 2 * b + 1)];
    F[flux_index(ax, v, cface, k1 * 4 + a, k2 * 4 + b)] = 0.25 * ((f00 + f10) + (f01 + f11));
  }
}

// update of all 512 cells of `leaf` from its (refluxed) flux set F (step.py:243-288)
OMB_HD void update_leaf(const StageArgs& A, int leaf, const double* F, int tid, int nthr) {
  const LeafInfo& LI = A.info[leaf];
  UpdateParams P;
  P.dt = *A.dt; P.a = A.a; P.b = A.b;
  P.gamma = A.gamma; P.eta = A.eta; P.inv_gamma = A.inv_gamma; P.omega = A.omega;
  P.floor_rho = A.floor_rho; P.floor_tau = A.floor_tau; P.floor_vmax = A.floor_vmax;
  P.has_grav = A.grav != nullptr;
  P.has_src = (A.omega != 0.0) || P.has_grav;
  for (int c = tid; c < 512; c += nthr) {
    int x = c / 64, y = (c / 8) % 8, z = c % 8;
    long long cell = (long long)leaf * 512 + c;
    double u[NF], u0[NF], rr[NF], out[NF], g[4] = {0, 0, 0, 0};
#pragma unroll
    for (int v = 0; v < NF; v++) {
      u[v] = A.ucur[v * A.fstride + cell];
      u0[v] = (A.scalar && v == NF - 1) ? A.s_u0[cell] : A.u0[v * A.fstride + cell];
      double dfx = F[flux_index(0, v, x + 1, y, z)] - F[flux_index(0, v, x, y, z)];
      double dfy = F[flux_index(1, v, y + 1, x, z)] - F[flux_index(1, v, y, x, z)];
      double dfz = F[flux_index(2, v, z + 1, x, y)] - F[flux_index(2, v, z, x, y)];
      double tt = 0.0 - dfx * LI.inv_dx;
      tt = tt - dfy * LI.inv_dx;
      tt = tt - dfz * LI.inv_dx;
      rr[v] = tt;
    }
    if (P.has_grav)
#pragma unroll
      for (int q = 0; q < 4; q++) g[q] = A.grav[q * A.fstride + cell];
    double xc = LI.ox + LI.dx * (double)(x + ((LI.flags >> 8) & 31));
    double yc = LI.oy + LI.dx * (double)(y + ((LI.flags >> 13) & 31));
    if (A.scalar) {
      update_cell_rk(P, u, u0, rr, xc, yc, g, out);
      A.s_next[cell] = out[NF - 1];
      continue;
    }
    update_cell(P, u, u0, rr, xc, yc, g, out);
#pragma unroll
    for (int v = 0; v < NF; v++) A.unext[v * A.fstride + cell] = out[v];
  }
}

// block cell count / decode and placement inside the virtual leaf
OMB_HD int amr_block_cells(const int* t) {
  int c = 1;
#pragma unroll
  for (int a = 0; a < 3; a++) c *= t[1 + a] ? 3 : N;
  return c;
}
OMB_HD void amr_decode(const int* t, int i, int* b, int& vcell) {
  int d[3];
#pragma unroll
  for (int a = 0; a < 3; a++) d[a] = t[1 + a] ? 3 : N;
  b[2] = i % d[2];
  b[1] = (i / d[2]) % d[1];
  b[0] = i / (d[2] * d[1]);
  int v[3];
#pragma unroll
  for (int a = 0; a < 3; a++) v[a] = b[a] + (t[1 + a] == -1 ? N - 3 : 0);
  vcell = v[0] * 64 + v[1] * 8 + v[2];
}

}  // namespace omb
