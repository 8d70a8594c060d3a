// omb_kernels.cu -- sm_100a kernels of the B200 hydro step and the C ABI
// (include/omb200.h).  Build: see paper_2107_10987_b200/build.py
// (nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false ...).
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <string>

#include "../../include/omb200.h"
#include "omb_math.cuh"
#include "omb_stage.cuh"

using namespace omb;

static_assert(sizeof(OmbLeafInfo) == sizeof(LeafInfo), "OmbLeafInfo layout");

static thread_local std::string g_err;
static int set_err(const char* what, cudaError_t e) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return -1;
}
static int set_err(const std::string& what) {
  g_err = what;
  return -2;
}
#define CK(call, what)                       \
  do {                                       \
    cudaError_t _e = (call);                 \
    if (_e != cudaSuccess) return set_err(what, _e); \
  } while (0)

// ---------------------------------------------------------------------------
// face quadrature tables (geometry.py:51-123) for the per-sub-grid flux shim
// ---------------------------------------------------------------------------
struct FaceTable {
  int kind[9], nrow[9], line[25], dp[25][3], flip[25];
};
__constant__ FaceTable c_ft[3];

static void build_face_tables(FaceTable* ft) {
  static const int D[13][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, -1, 0}, {1, 0, 1}, {1, 0, -1},
                               {0, 1, 1}, {0, 1, -1}, {1, 1, 1}, {1, 1, -1}, {1, -1, 1}, {1, -1, -1}};
  const double off[3] = {0.0, -0.5, 0.5};
  for (int a = 0; a < 3; a++) {
    int b = a == 0 ? 1 : 0, c = a == 2 ? 1 : 2;
    int npt = 0, nr = 0;
    for (int kind = 0; kind < 3; kind++)  // stable sort by kind of the (tb, tc) enumeration
      for (int ib = 0; ib < 3; ib++)
        for (int ic = 0; ic < 3; ic++) {
          double tb = off[ib], tc = off[ic];
          int k = (tb != 0.0) + (tc != 0.0);
          if (k != kind) continue;
          ft[a].kind[npt] = kind;
          int cnt = 0;
          for (int l = 0; l < 13; l++) {
            if (D[l][a] == 0 || (D[l][b] != 0) != (tb != 0.0) || (D[l][c] != 0) != (tc != 0.0)) continue;
            double pt[3];
            pt[a] = 0.5;
            pt[b] = tb;
            pt[c] = tc;
            ft[a].line[nr] = l;
            for (int q = 0; q < 3; q++) {
              double p = pt[q] - 0.5 * D[l][q];
              ft[a].dp[nr][q] = (int)(p < 0 ? p - 0.5 : p + 0.5);
            }
            ft[a].flip[nr] = D[l][a] < 0;
            nr++;
            cnt++;
          }
          ft[a].nrow[npt++] = cnt;
        }
  }
}

// one-time setup PER DEVICE (face tables in that device's constant bank, the
// stage/reflux kernels' shared-memory attributes): a bit per device, set under
// a mutex, read lock-free afterwards -- entry points may be called from many
// host threads and for several devices in one process (the reference calls its
// kernels from scheduler threads, _core.pyx:60,239).  Defined after the kernels.
static int lib_init();

// ---------------------------------------------------------------------------
// per-sub-grid shims (the reference's `kernels` module surface)
// ---------------------------------------------------------------------------
__global__ void k_primitives(const double* __restrict__ u, int m, double gamma, double gm1, double eta,
                             double* __restrict__ prim) {
  long long nc = (long long)m * m * m;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nc; c += (long long)gridDim.x * blockDim.x) {
    double uu[NF], w[NF];
    for (int v = 0; v < NF; v++) uu[v] = u[v * nc + c];
    prim_cell(uu, gamma, gm1, eta, w);
    for (int v = 0; v < NF; v++) prim[v * nc + c] = w[v];
  }
}

// one thread per (line, cell in [2,m-2)^3): lo/hi of 6 fields of one cell
__global__ void k_reconstruct(const double* __restrict__ prim, int m, int nlines, int contact, double gamma,
                              double* __restrict__ lo, double* __restrict__ hi, unsigned long long* fallback) {
  int core = m - 4;
  long long ncore = (long long)core * core * core;
  long long nc = (long long)m * m * m;
  long long total = ncore * nlines;
  unsigned long long fb = 0;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < total;
       it += (long long)gridDim.x * blockDim.x) {
    int l = (int)(it / ncore);
    long long r = it % ncore;
    int i = 2 + (int)(r / (core * core)), j = 2 + (int)((r / core) % core), k = 2 + (int)(r % core);
    int dx = ldx(l), dy = ldy(l), dz = ldz(l);
    long long o[5];
    for (int q = 0; q < 5; q++) o[q] = ((long long)(i + (q - 2) * dx) * m + (j + (q - 2) * dy)) * m + (k + (q - 2) * dz);
    double L[NF], H[NF], rr[5], pm1 = 0, pp1 = 0;
    for (int v = 0; v < NF; v++) {
      double s[5];
      for (int q = 0; q < 5; q++) s[q] = prim[v * nc + o[q]];
      double lv = iface(s[0], s[1], s[2], s[3]);
      double hv = iface(s[1], s[2], s[3], s[4]);
      mono(s[2], lv, hv);
      L[v] = lv;
      H[v] = hv;
      if (v == 0)
        for (int q = 0; q < 5; q++) rr[q] = s[q];
      if (v == 4) { pm1 = s[1]; pp1 = s[3]; }
    }
    if (contact) contact_steepen(rr, pm1, pp1, gamma, L[0], H[0]);
    if (L[0] <= 0.0 || L[4] <= 0.0) {
      fb++;
      for (int v = 0; v < NF; v++) L[v] = prim[v * nc + o[2]];
    }
    if (H[0] <= 0.0 || H[4] <= 0.0) {
      fb++;
      for (int v = 0; v < NF; v++) H[v] = prim[v * nc + o[2]];
    }
    long long base = (long long)l * NF * nc + o[2];
    for (int v = 0; v < NF; v++) {
      lo[base + v * nc] = L[v];
      hi[base + v * nc] = H[v];
    }
  }
  if (fb) atomicAdd(fallback, fb);
}

// one thread per face: the reference's 9-point / 25-row loop verbatim
__global__ void k_fluxes(const double* __restrict__ lo, const double* __restrict__ hi, int n, double gamma,
                         double gm1, int new_mode, int override_center, double* fx, double* fy, double* fz,
                         unsigned long long* amax_bits) {
  int m = n + 6;
  long long nc = (long long)m * m * m;
  int nface = (n + 1) * n * n;
  double amax = 0.0;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < 3 * nface; it += gridDim.x * blockDim.x) {
    int axis = it / nface, f = it % nface;
    int n0 = axis == 0 ? n + 1 : n, n1 = axis == 1 ? n + 1 : n, n2 = axis == 2 ? n + 1 : n;
    int i0 = f / (n1 * n2), i1 = (f / n2) % n1, i2 = f % n2;
    int low[3] = {axis == 0 ? 2 + i0 : 3 + i0, axis == 1 ? 2 + i1 : 3 + i1, axis == 2 ? 2 + i2 : 3 + i2};
    const FaceTable& T = c_ft[axis];
    double center[NF] = {0, 0, 0, 0, 0, 0}, pd[4][NF], edev[NF] = {0, 0, 0, 0, 0, 0}, vdev[NF] = {0, 0, 0, 0, 0, 0};
    int rr0 = 0, ei = 0, vi = 0;
    for (int pt = 0; pt < 9; pt++) {
      int kind = T.kind[pt], nrow = T.nrow[pt];
      if (kind != 0 && (!new_mode || override_center)) { rr0 += nrow; continue; }
      double acc[NF] = {0, 0, 0, 0, 0, 0}, pair[NF];
      for (int r = 0; r < nrow; r++) {
        int l = T.line[rr0 + r];
        int p[3] = {low[0] + T.dp[rr0 + r][0], low[1] + T.dp[rr0 + r][1], low[2] + T.dp[rr0 + r][2]};
        long long P = ((long long)p[0] * m + p[1]) * m + p[2];
        long long Q = ((long long)(p[0] + ldx(l)) * m + (p[1] + ldy(l))) * m + (p[2] + ldz(l));
        double wP[NF], wQ[NF];
        for (int v = 0; v < NF; v++) {
          wP[v] = hi[((long long)l * NF + v) * nc + P];
          wQ[v] = lo[((long long)l * NF + v) * nc + Q];
        }
        KtState sP, sQ;
        kt_state(wP, gamma, gm1, 1.0 / gm1, sP);
        kt_state(wQ, gamma, gm1, 1.0 / gm1, sQ);
        double fv[NF];
        double sp = kt_axis(sP, sQ, axis, T.flip[rr0 + r] != 0, fv);
        if (sp > amax) amax = sp;
        if (nrow == 4) {
          if (r == 0 || r == 2) {
            for (int v = 0; v < NF; v++) pair[v] = fv[v];
          } else {
            for (int v = 0; v < NF; v++) acc[v] += pair[v] + fv[v];
          }
        } else {
          for (int v = 0; v < NF; v++) acc[v] += fv[v];
        }
      }
      rr0 += nrow;
      if (kind == 0) {
        for (int v = 0; v < NF; v++) center[v] = acc[v];
      } else if (kind == 1) {
        for (int v = 0; v < NF; v++) pd[ei][v] = pdev_edge(acc[v], center[v]);
        if (++ei == 4)
          for (int v = 0; v < NF; v++) edev[v] = (pd[0][v] + pd[1][v]) + (pd[2][v] + pd[3][v]);
      } else {
        for (int v = 0; v < NF; v++) pd[vi][v] = pdev_vert(acc[v], center[v]);
        if (++vi == 4)
          for (int v = 0; v < NF; v++) vdev[v] = (pd[0][v] + pd[1][v]) + (pd[2][v] + pd[3][v]);
      }
    }
    double* F = axis == 0 ? fx : (axis == 1 ? fy : fz);
    long long fs = (long long)n0 * n1 * n2;
    for (int v = 0; v < NF; v++)
      F[v * fs + f] = (new_mode && !override_center) ? face_final(center[v], edev[v], vdev[v]) : center[v];
  }
  if (amax > 0.0) atomicMax(amax_bits, (unsigned long long)__double_as_longlong(amax));
}

// ---------------------------------------------------------------------------
// fused stage: one CTA per run
// ---------------------------------------------------------------------------
constexpr int STAGE_THREADS = 512;

__device__ __forceinline__ void block_reduce(double amax, long long fb, unsigned long long* amax_bits,
                                             unsigned long long* fallback) {
  __shared__ double s_max[STAGE_THREADS / 32];
  __shared__ long long s_fb[STAGE_THREADS / 32];
  for (int o = 16; o > 0; o >>= 1) {
    double t = __shfl_xor_sync(0xffffffffu, amax, o);
    amax = t > amax ? t : amax;
    fb += __shfl_xor_sync(0xffffffffu, fb, o);
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_max[w] = amax;
    s_fb[w] = fb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    long long f = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) {
      m = s_max[i] > m ? s_max[i] : m;
      f += s_fb[i];
    }
    if (m > 0.0) atomicMax(amax_bits, (unsigned long long)__double_as_longlong(m));
    if (f) atomicAdd(fallback, (unsigned long long)f);
  }
}

#ifdef OMB_PHASE_PROF
// profiling build only (profiles/phase_prof.py): thread 0 of every CTA adds
// the cycles between consecutive barrier exits to its phase's counter
__device__ unsigned long long g_phase_cycles[16];
#define PH(k)                                                        \
  do {                                                               \
    if (tid == 0) {                                                  \
      long long _t = clock64();                                      \
      atomicAdd(&g_phase_cycles[k], (unsigned long long)(_t - _t0)); \
      _t0 = _t;                                                      \
    }                                                                \
  } while (0)
#else
#define PH(k) \
  do {        \
  } while (0)
#endif

// SC: the passive-scalar pass (a separate instantiation, so the hydro stage
// carries none of its branches: A.scalar is a compile-time constant below)
template <int NT, int SC>
__global__ void __launch_bounds__(NT, 1) k_stage(StageArgs A) {
  static_assert(NT >= 2 * NFACEX, "P6 runs on the last 64 threads of the last P1 group");
  static_assert(ITEM_ROUNDS == 2 || NT >= OMB_ITEMS_P1A_NEW_N, "one round of reconstruction items needs >= 500 threads");
  extern __shared__ double S[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  Stage st;
  st.S = S;
  st.A = A;
  st.A.scalar = SC;
  st.run = blockIdx.x;
  int off = A.run_off[blockIdx.x];
  st.R = A.run_off[blockIdx.x + 1] - off;
  st.leaves = A.run_leaf + off;
  st.amax = 0.0;
  st.fb = 0;
  st.bind_run_info();
  st.stage_run_info(tid, nthr);
  st.load_items(tid);
  __syncthreads();
  Hold h;
  const int R = st.R;
#ifdef OMB_PHASE_PROF
  long long _t0 = clock64();
#endif
  // prologue: planes 0..3 staged in the (still unused) RAW union and plane 4
  // in SG0, all loads in flight at once; then planes 0..3 converted
  for (int X = 0; X < 4; X++) st.prefetch_plane(X, tid, nthr, Smem::RAW + X * NF * PL);
  st.prefetch_plane(4, tid, nthr);
  async_commit();
  async_wait_all();
  __syncthreads();
  for (int X = 0; X < 4; X++) st.convert_plane(X, tid, nthr, Smem::RAW + X * NF * PL);
  __syncthreads();
  PH(0);
  const int ngroups = A.new_mode ? 2 : 1;
  for (int X = 2; X < 8 * R + 4; X++) {
    st.set_plane(X);
    // P0: primitives of plane X+2 (threads [0, 196)); beside it P5 of plane
    // X-1 -- its y/z faces (the next phase overwrites the in-plane fluxes they
    // read) -- and the staging of the next update's inputs (SG6)
    if (X + 2 < 8 * R + 6) st.convert_plane(X + 2, tid, nthr);
    if (X - 1 >= 3) {
      st.set_plane(X - 1);
      st.faces_yz(tid, nthr, PL);
      st.set_plane(X);
    }
    // (512 threads: [116, 196) convert a cell and have no face item)
    constexpr int T6 = NF * NYF - (512 - PL);
    if (st.interior(X - 2) && tid >= T6 && tid < T6 + NFACEX) st.prefetch_update(X - 2, tid - T6, NFACEX);
    async_commit();
    __syncthreads();
    PH(1);
    if (X + 3 < 8 * R + 6) st.prefetch_plane(X + 3, tid, nthr);  // stage next P0 (cp.async)
    async_commit();
    // P6 = the update of plane X-2 (its x fluxes sit in the 3-slot FX ring,
    // its y/z fluxes in FYZ since this plane's P0, its inputs staged in SG6),
    // in two halves on the last 64 threads: fluxes + sources + RK beside P2A
    // (432 items), dual energy + floors + store beside P3 (<= 400 items)
    const bool p6 = X >= 3 && st.interior(X - 2);
#pragma unroll 1
    for (int g = 0; g < ngroups; g++) {
      st.boundary_lines(g, tid, nthr, h);  // P1
      // the update inputs staged in this plane's P0 (SG6) land before P6 part A
      // (this plane's SG0 group, committed last, may still be in flight)
      if (g == 0) async_wait_prev();
      __syncthreads();
      PH(2 + 2 * g);
      st.store_hi(h);
      if (X >= 3) {  // P2
        if (g == 0) st.combine_A(tid, nthr);
        else if (A.quad) st.combine_B(tid, nthr);
      }
      if (g == 0 && p6 && tid >= nthr - NFACEX) {  // P6 part A on the threads P2A leaves idle
        st.set_plane(X - 1);
        st.update_plane_a(tid - (nthr - NFACEX), NFACEX);
        st.set_plane(X);
      }
      __syncthreads();
      PH(3 + 2 * g);
    }
    st.inplane_lines(tid, nthr);  // P3 (<= 400 items)
    if (p6 && tid >= nthr - NFACEX) {  // P6 part B on the last 64 threads
      st.set_plane(X - 1);
      st.update_plane_b(tid - (nthr - NFACEX), NFACEX);
      st.set_plane(X);
    }
    __syncthreads();
    PH(6);
    if (st.interior(X)) st.inplane_fluxes(tid, nthr);  // P4 (<= 468 items)
    async_wait_all();  // SG0 for the next P0
    __syncthreads();
    PH(7);
  }
  // P5 of the last plane, and the last update's inputs
  st.set_plane(8 * R + 3);
  st.faces_yz(tid, nthr);
  if (tid < NFACEX) st.prefetch_update(8 * R + 2, tid, NFACEX);
  async_commit();
  async_wait_all();
  __syncthreads();
  PH(8);
  // P6 of the last plane
  st.set_plane(8 * R + 3);
  st.update_plane(tid, nthr);
  PH(9);
  block_reduce(st.amax, st.fb, A.amax_bits, A.fallback);
}

// ---------------------------------------------------------------------------
// CFL: per-leaf speed, then a single-CTA min reduction
// ---------------------------------------------------------------------------
__global__ void k_cfl_leaf(const double* __restrict__ U, long long fstride, const double* __restrict__ dxs,
                           double gamma, double gm1, double eta, double* ratio, int* bad) {
  int leaf = blockIdx.x;
  double best = 0.0;
  bool nan = false, first = true;
  for (int c = threadIdx.x; c < 512; c += blockDim.x) {
    double u[NF];
    for (int v = 0; v < NF; v++) u[v] = U[v * fstride + (long long)leaf * 512 + c];
    double s = speed_cell(u, gamma, gm1, eta);
    if (s != s) nan = true;
    else if (first || s > best) best = s;
    first = false;
  }
  __shared__ double sb[32];
  __shared__ int sn[32];
  for (int o = 16; o > 0; o >>= 1) {
    double t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
    nan |= __shfl_xor_sync(0xffffffffu, (int)nan, o) != 0;
  }
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = best;
    sn[threadIdx.x >> 5] = nan;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = sb[0];
    int anynan = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) {
      m = sb[i] > m ? sb[i] : m;
      anynan |= sn[i];
    }
    // np.max propagates NaN; np.isfinite(speed) rejects NaN and inf
    bool finite = !anynan && m == m && m < INFINITY && m > -INFINITY;
    bad[leaf] = finite ? 0 : 1;
    ratio[leaf] = finite ? dxs[leaf] / m : INFINITY;
  }
}

__global__ void k_cfl_reduce(int L, const double* ratio, const int* bad, double cfl, double* out, int* bad_leaf,
                             double* dt_dev) {
  __shared__ double sw[32];
  __shared__ int sb[32];
  double w = INFINITY;
  int b = 0x7fffffff;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    w = ratio[i] < w ? ratio[i] : w;
    if (bad[i] && i < b) b = i;
  }
  for (int o = 16; o > 0; o >>= 1) {
    double t = __shfl_xor_sync(0xffffffffu, w, o);
    w = t < w ? t : w;
    int tb = __shfl_xor_sync(0xffffffffu, b, o);
    b = tb < b ? tb : b;
  }
  if ((threadIdx.x & 31) == 0) {
    sw[threadIdx.x >> 5] = w;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
      w = sw[i] < w ? sw[i] : w;
      b = sb[i] < b ? sb[i] : b;
    }
    w = sw[0] < w ? sw[0] : w;
    b = sb[0] < b ? sb[0] : b;
    out[0] = w;
    out[1] = cfl * w;
    *bad_leaf = b == 0x7fffffff ? -1 : b;
    if (dt_dev) *dt_dev = cfl * w;
  }
}

// padded (6,14,14,14) arrays of leaves first .. first+gridDim.y-1: interior + the
// ghost shell exactly as mesh/ghosts.py fills it (AMR regions from the virtual
// leaves k_amr_ghosts filled)
__global__ void k_gather(const double* U, long long fstride, const LeafInfo* info, int first, int bc, double* out) {
  const int leaf = first + blockIdx.y;
  double* o = out + (long long)blockIdx.y * NF * M * M * M;
  for (int c = threadIdx.x + blockIdx.x * blockDim.x; c < M * M * M; c += blockDim.x * gridDim.x) {
    double u[NF];
    gather_cell(U, fstride, info[leaf], bc, c / (M * M), (c / M) % M, c % M, u);
    for (int v = 0; v < NF; v++) o[v * M * M * M + c] = u[v];
  }
}

// AMR ghost regions: one thread per (task, block cell), 6 fields
__global__ void k_amr_ghosts(double* U, long long fstride, const int* __restrict__ tasks, int ntasks) {
  int task = blockIdx.x;
  if (task >= ntasks) return;
  const int* t = tasks + task * 16;
  int tl[16];
#pragma unroll
  for (int i = 0; i < 16; i++) tl[i] = t[i];
  int ncell = amr_block_cells(tl);
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
    int b[3], vcell;
    amr_decode(tl, i, b, vcell);
    double out[NF];
#pragma unroll
    for (int v = 0; v < NF; v++) out[v] = amr_cell(U, fstride, tl, v, b);
#pragma unroll
    for (int v = 0; v < NF; v++) U[v * fstride + (long long)tl[4] * 512 + vcell] = out[v];
  }
}

// reflux (step.py:206-241) + update (step.py:243-288) of one deferred coarse leaf per CTA
__global__ void k_reflux_update(StageArgs A, const int* __restrict__ rleaf, const int* __restrict__ roff,
                                const int* __restrict__ rtasks) {
  extern __shared__ double F[];  // FLUX_SLOT doubles: this leaf's FX | FY | FZ
  int leaf = rleaf[blockIdx.x];
  const double* src = A.flux + (long long)A.info[leaf].slot * FLUX_SLOT;
  for (int i = threadIdx.x; i < FLUX_SLOT; i += blockDim.x) F[i] = src[i];
  __syncthreads();
  // substitutions touch disjoint face blocks: no ordering among them
  for (int q = roff[blockIdx.x]; q < roff[blockIdx.x + 1]; q++) reflux_apply(F, A.flux, rtasks + q * 6, threadIdx.x, blockDim.x);
  __syncthreads();
  update_leaf(A, leaf, F, threadIdx.x, blockDim.x);
}

// per-leaf field sums in a fixed order (x-major rows of 8, pairwise inside a
// row, rows accumulated in order) -- device side of conservation_totals
__global__ void k_leaf_sums(const double* __restrict__ U, long long fstride, int L, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L * NF) return;
  int leaf = i / NF, v = i % NF;
  const double* p = U + v * fstride + (long long)leaf * 512;
  double acc = 0.0;
  for (int r = 0; r < 64; r++) {
    const double* a = p + r * 8;
    acc += ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
  out[leaf * NF + v] = acc;
}

// checkpoint payload order (mesh/checkpoint.py:53-54): per leaf, fields, cells x-fastest
__global__ void k_disk_order(const double* __restrict__ U, long long fstride, int L, double* __restrict__ out) {
  long long total = (long long)L * NF * 512;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i & 511);
    long long lv = i >> 9;
    int v = (int)(lv % NF);
    long long leaf = lv / NF;
    int z = c >> 6, y = (c >> 3) & 7, x = c & 7;  // on disk x varies fastest
    out[i] = U[v * fstride + leaf * 512 + x * 64 + y * 8 + z];
  }
}

// halo exchange packing: whole 8^3 leaves, field-major state <-> leaf-major message
__global__ void k_pack(const double* __restrict__ U, long long fstride, const int* __restrict__ idx, int n,
                       double* __restrict__ out) {
  long long total = (long long)n * NF * 512;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i & 511);
    long long kv = i >> 9;
    int v = (int)(kv % NF);
    long long k = kv / NF;
    out[i] = U[v * fstride + (long long)idx[k] * 512 + c];
  }
}

__global__ void k_unpack(const double* __restrict__ in, int n, double* __restrict__ U, long long fstride, int first) {
  long long total = (long long)n * NF * 512;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i & 511);
    long long kv = i >> 9;
    int v = (int)(kv % NF);
    long long k = kv / NF;
    U[v * fstride + (first + k) * 512 + c] = in[i];
  }
}

// self-test of div_by (Markstein quotient) against the IEEE division on
// random operands spanning 2^[-60,60] with random signs, 1 in 8 numerators 0
// ---------------------------------------------------------------------------
// scalar flux surface (hydro/flux.py:12-94): kt_flux / physical_flux on point
// states, face_flux on 9 point fluxes -- batched, one thread per point
// ---------------------------------------------------------------------------
// state s = (rho, vx, vy, vz, p, eint, tau): PrimitiveState.conserved (flux.py:32-37)
OMB_HD void pt_conserved(const double* s, double* u) {
  // Python float ** 2 is C pow(x, 2.0), i.e. glibc's pow
  double kin = 0.5 * s[0] * ((pow_glibc(s[1], 2.0) + pow_glibc(s[2], 2.0)) + pow_glibc(s[3], 2.0));
  u[0] = s[0];
  u[1] = s[0] * s[1];
  u[2] = s[0] * s[2];
  u[3] = s[0] * s[3];
  u[4] = s[0] * s[5] + kin;
  u[5] = s[6];
}
// physical_flux (flux.py:40-47)
OMB_HD void pt_physical(const double* s, int axis, double* f) {
  double u[NF];
  pt_conserved(s, u);
  double vn = s[1 + axis];
  for (int v = 0; v < NF; v++) f[v] = u[v] * vn;
  f[1 + axis] += s[4];
  f[4] += s[4] * vn;
}
__global__ void k_kt_points(const double* __restrict__ L, const double* __restrict__ R, int n, int axis, double gamma,
                            double* __restrict__ out, int* __restrict__ bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* l = L + 7 * i;
  const double* r = R + 7 * i;
  double* o = out + NF * i;
  for (int k = 0; k < 5; k++)  // flux.py:56-58: rho, v, p must be finite
    if (!isfinite(l[k]) || !isfinite(r[k])) {
      atomicMin(bad, i);
      for (int v = 0; v < NF; v++) o[v] = NAN;
      return;
    }
  double cl = sqrt(gamma * l[4] / l[0]), cr = sqrt(gamma * r[4] / r[0]);
  double vl = l[1 + axis], vr = r[1 + axis];
  // Python max(0.0, a, b) / min(...): the first extreme argument wins
  double ap = 0.0, am = 0.0;
  if (vl + cl > ap) ap = vl + cl;
  if (vr + cr > ap) ap = vr + cr;
  if (vl - cl < am) am = vl - cl;
  if (vr - cr < am) am = vr - cr;
  double fl[NF], fr[NF], ul[NF], ur[NF];
  pt_physical(l, axis, fl);
  if (ap - am <= 0.0) {
    for (int v = 0; v < NF; v++) o[v] = fl[v];
    return;
  }
  pt_physical(r, axis, fr);
  pt_conserved(l, ul);
  pt_conserved(r, ur);
  for (int v = 0; v < NF; v++) o[v] = ((ap * fl[v] - am * fr[v]) + (ap * am) * (ur[v] - ul[v])) / (ap - am);
}
__global__ void k_physical_points(const double* __restrict__ S, int n, int axis, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pt_physical(S + 7 * i, axis, out + NF * i);
}
// face_flux (flux.py:70-91): pts [n][9][6] (centre, 4 edges, 4 vertices) -> out [n][6]
__global__ void k_face_points(const double* __restrict__ pts, int n, int new_mode, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * NF) return;
  int f = i / NF, v = i % NF;
  const double* p = pts + (long long)f * 9 * NF;
  double c = p[v];
  if (!new_mode) {
    out[i] = c;
    return;
  }
  double edev = ((p[1 * NF + v] - c) + (p[2 * NF + v] - c)) + ((p[3 * NF + v] - c) + (p[4 * NF + v] - c));
  double vdev = ((p[5 * NF + v] - c) + (p[6 * NF + v] - c)) + ((p[7 * NF + v] - c) + (p[8 * NF + v] - c));
  out[i] = c + (4.0 * edev + vdev) / 36.0;
}

// passive-scalar pass input: (rho, sx, sy, sz, p, X) per cell
__global__ void k_scalar_input(const double* __restrict__ U, long long fstride, int n_all, const double* __restrict__ x,
                               int n_x, double gamma, double gm1, double eta, double* __restrict__ dst) {
  long long n = (long long)n_all * 512;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    double u[NF], w[NF];
#pragma unroll
    for (int v = 0; v < NF; v++) u[v] = U[v * fstride + c];
    prim_cell(u, gamma, gm1, eta, w);
#pragma unroll
    for (int v = 0; v < 4; v++) dst[v * fstride + c] = u[v];
    dst[4 * fstride + c] = w[4];
    if (x != nullptr && c < (long long)n_x * 512) dst[5 * fstride + c] = x[c];
  }
}

// pow_glibc element-wise (the self-check of omb_pow.cuh against the host's libm)
__global__ void k_pow_batch(const double* __restrict__ x, const double* __restrict__ y, long long n,
                            double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = pow_glibc(x[i], y[i]);
}

__global__ void k_selftest_div(unsigned long long seed, long long n, unsigned long long* bad) {
  unsigned long long s = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x[2];
    for (int j = 0; j < 2; j++) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      unsigned long long m = s & 0xFFFFFFFFFFFFFull;
      // 1 in 4: any biased exponent (subnormals, huge, inf/NaN); else |e| <= 60
      int eb = ((s >> 40) & 3) == 0 ? (int)((s >> 52) % 2048) : (int)((s >> 52) % 121) - 60 + 1023;
      unsigned long long bits = ((unsigned long long)eb << 52) | m | ((s >> 63) << 63);
      x[j] = __longlong_as_double((long long)bits);
    }
    if ((s & 7) == 0) x[0] = (s & 8) ? -0.0 : 0.0;
    double q = __ddiv_rn(x[0], x[1]);
    double y = __ddiv_rn(1.0, x[1]);
    double ab = fabs(x[1]);
    // div_by: divisors in [2^-100, 2^100] only (its precondition)
    double m1 = (ab > 0x1p-100 && ab < 0x1p+100) ? div_by(x[0], x[1], y) : q;
    // kt_axis form (positive divisor): range test of the divisor, straight-line quotient, IEEE redo
    unsigned rare = !div_range_ok(ab);
    double m2 = div_fast(x[0], ab, __ddiv_rn(1.0, ab), rare);
    if (rare) m2 = x[0] / ab;
    double q2 = __ddiv_rn(x[0], ab);
    bool qn = q != q;  // NaN results: any NaN payload is acceptable
    bool b1 = qn ? (m1 == m1) : (__double_as_longlong(q) != __double_as_longlong(m1));
    bool b2 = (q2 != q2) ? (m2 == m2) : (__double_as_longlong(q2) != __double_as_longlong(m2));
    double m3 = div_nz(x[0], x[1]);
    bool b3 = qn ? (m3 == m3) : (__double_as_longlong(q) != __double_as_longlong(m3));
    if (b1 || b2 || b3) {
      nb++;
      if (atomicCAS(bad + 7, 0ull, 1ull) == 0ull) {  // first mismatch: a, b, a/b, div_by, kt form
        bad[1] = (unsigned long long)__double_as_longlong(x[0]);
        bad[2] = (unsigned long long)__double_as_longlong(x[1]);
        bad[3] = (unsigned long long)__double_as_longlong(q);
        bad[4] = (unsigned long long)__double_as_longlong(m1);
        bad[5] = (unsigned long long)__double_as_longlong(m2);
      }
    }
  }
  if (nb) atomicAdd(bad, nb);
}

// row gather / scatter (multi-GPU AMR: exchange of exported flux slots)
__global__ void k_rows(const double* __restrict__ src, long long row, const int* __restrict__ idx, int n,
                       double* __restrict__ dst, int scatter) {
  long long total = (long long)n * row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    long long k = i / row, c = i % row;
    if (scatter) dst[(long long)idx[k] * row + c] = src[i];
    else dst[i] = src[(long long)idx[k] * row + c];
  }
}

// FP64 pipe peak probe (roofline denominator; MEASURED_PEAKS.json has no FP64 entry):
// 8 independent DFMA chains per thread, 2 flops per DFMA.
__global__ void k_dfma_peak(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; k++) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = __fma_rn(a[k], m, c);
  }
  double s = 0.0;
  for (int k = 0; k < 8; k++) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
static std::mutex g_init_mu;
static std::atomic<unsigned long long> g_init_devs{0};
static int lib_init() {
  int dev = 0;
  CK(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= 64) return set_err("device index outside [0, 64)");
  const unsigned long long bit = 1ull << dev;
  if (g_init_devs.load(std::memory_order_acquire) & bit) return 0;
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (g_init_devs.load(std::memory_order_relaxed) & bit) return 0;
  FaceTable ft[3];
  build_face_tables(ft);
  CK(cudaMemcpyToSymbol(c_ft, ft, sizeof(ft)), "face table upload");
  // 512 threads x 128 registers fills the register file; 256/384/576/640 were measured slower
  CK(cudaFuncSetAttribute(k_stage<STAGE_THREADS, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::BYTES),
     "stage smem attribute");
  CK(cudaFuncSetAttribute(k_stage<STAGE_THREADS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::BYTES),
     "scalar stage smem attribute");
  CK(cudaFuncSetAttribute(k_reflux_update, cudaFuncAttributeMaxDynamicSharedMemorySize, FLUX_SLOT * 8),
     "reflux smem attribute");
  g_init_devs.fetch_or(bit, std::memory_order_release);
  return 0;
}

extern "C" {

int omb_abi_version(void) { return OMB_ABI_VERSION; }
const char* omb_last_error(void) { return g_err.c_str(); }
int omb_stage_smem_bytes(void) { return Smem::BYTES; }

// CUDA IPC for the multi-GPU halo reads: a rank allocates its state buffers
// itself (so the IPC handle covers exactly them), peers open them in their
// own device's context with lazy peer access
int omb_ipc_alloc(long long bytes, void** ptr, void* handle64) {
  if (int rc = lib_init()) return rc;
  CK(cudaMalloc(ptr, (size_t)bytes), "omb_ipc_alloc cudaMalloc");
  CK(cudaMemset(*ptr, 0, (size_t)bytes), "omb_ipc_alloc cudaMemset");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, *ptr), "cudaIpcGetMemHandle");
  memcpy(handle64, &h, sizeof(h));
  return 0;
}
int omb_ipc_open(const void* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return 0;
}

// let kernels of the current device read another device's memory (NVLink peer access)
int omb_enable_peer_access(int peer_device) {
  int cur = -1, ok = 0;
  CK(cudaGetDevice(&cur), "cudaGetDevice");
  if (peer_device == cur) return 0;
  CK(cudaDeviceCanAccessPeer(&ok, cur, peer_device), "cudaDeviceCanAccessPeer");
  if (!ok) return set_err("omb_enable_peer_access: no peer access between these devices");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  CK(e, "cudaDeviceEnablePeerAccess");
  return 0;
}
#ifdef OMB_PHASE_PROF
int omb_phase_prof(unsigned long long* out, int reset) {  // profiling build only
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

int omb_primitives(const double* u, int m, double gamma, double eta, double* prim, void* stream) {
  if (int rc = lib_init()) return rc;
  long long nc = (long long)m * m * m;
  int blocks = (int)((nc + 255) / 256);
  k_primitives<<<blocks, 256, 0, (cudaStream_t)stream>>>(u, m, gamma, gamma - 1.0, eta, prim);
  CK(cudaGetLastError(), "omb_primitives launch");
  return 0;
}

int omb_reconstruct(const double* prim, int m, int new_mode, int contact_on, double gamma, double* lo, double* hi,
                    unsigned long long* fallback, void* stream) {
  if (int rc = lib_init()) return rc;
  int nlines = new_mode ? 13 : 3;
  long long total = (long long)(m - 4) * (m - 4) * (m - 4) * nlines;
  int blocks = (int)((total + 255) / 256);
  k_reconstruct<<<blocks, 256, 0, (cudaStream_t)stream>>>(prim, m, nlines, contact_on, gamma, lo, hi, fallback);
  CK(cudaGetLastError(), "omb_reconstruct launch");
  return 0;
}

int omb_fluxes(const double* lo, const double* hi, int n, double gamma, int new_mode, int override_center, double* fx,
               double* fy, double* fz, unsigned long long* amax_bits, void* stream) {
  if (int rc = lib_init()) return rc;
  if (!div_range_ok(gamma - 1.0)) return set_err("omb_fluxes: gamma - 1 outside [2^-100, 2^100]");
  int total = 3 * (n + 1) * n * n;
  k_fluxes<<<(total + 127) / 128, 128, 0, (cudaStream_t)stream>>>(lo, hi, n, gamma, gamma - 1.0, new_mode,
                                                                    override_center, fx, fy, fz, amax_bits);
  CK(cudaGetLastError(), "omb_fluxes launch");
  return 0;
}

static StageArgs stage_args(const OmbStageDesc* d) {
  StageArgs A;
  A.ucur = d->ucur;
  A.u0 = d->u0;
  A.unext = d->unext;
  A.grav = d->grav;
  A.fstride = d->fstride;
  A.info = (const LeafInfo*)d->info;
  A.run_off = d->run_off;
  A.run_leaf = d->run_leaf;
  A.dt = d->dt;
  A.a = d->a;
  A.b = d->b;
  A.gamma = d->gamma;
  A.gm1 = d->gm1;
  A.inv_gm1 = 1.0 / d->gm1;
  A.eta = d->eta;
  A.inv_gamma = d->inv_gamma;
  A.omega = d->omega;
  A.floor_rho = d->floor_rho;
  A.floor_tau = d->floor_tau;
  A.floor_vmax = d->floor_vmax;
  A.bc = d->bc;
  A.new_mode = d->new_mode;
  A.quad = d->new_mode && !d->override_center;
  A.contact = d->contact;
  A.amax_bits = d->amax_bits;
  A.fallback = d->fallback;
  A.flux = d->flux;
  A.halo = d->halo;
  A.nown = d->nown;
  A.scalar = d->scalar;
  A.s_u0 = d->s_u0;
  A.s_next = d->s_next;
  return A;
}

int omb_amr_ghosts(const OmbAmrDesc* d, void* stream) {
  if (int rc = lib_init()) return rc;
  if (d->ntasks <= 0) return 0;
  k_amr_ghosts<<<d->ntasks, 192, 0, (cudaStream_t)stream>>>(d->u, d->fstride, d->tasks, d->ntasks);
  CK(cudaGetLastError(), "omb_amr_ghosts launch");
  return 0;
}

int omb_reflux_update(const OmbRefluxDesc* d, void* stream) {
  if (int rc = lib_init()) return rc;
  if (d->nleaves <= 0) return 0;
  StageArgs A = stage_args(&d->stage);
  k_reflux_update<<<d->nleaves, 256, FLUX_SLOT * 8, (cudaStream_t)stream>>>(A, d->leaf, d->off, d->tasks);
  CK(cudaGetLastError(), "omb_reflux_update launch");
  return 0;
}

int omb_stage(const OmbStageDesc* d, void* stream) {
  if (int rc = lib_init()) return rc;
  if (d->ucur == d->unext) return set_err("omb_stage: unext must not alias ucur");
  if (!div_range_ok(d->gm1)) return set_err("omb_stage: gamma - 1 outside [2^-100, 2^100]");
  StageArgs A = stage_args(d);
  if (d->nruns <= 0) return 0;
  if (d->scalar)
    k_stage<STAGE_THREADS, 1><<<d->nruns, STAGE_THREADS, Smem::BYTES, (cudaStream_t)stream>>>(A);
  else
    k_stage<STAGE_THREADS, 0><<<d->nruns, STAGE_THREADS, Smem::BYTES, (cudaStream_t)stream>>>(A);
  CK(cudaGetLastError(), "omb_stage launch");
  return 0;
}

int omb_cfl(const OmbCflDesc* d, void* stream) {
  if (int rc = lib_init()) return rc;
  if (d->nleaves <= 0) return set_err("omb_cfl: empty batch");
  k_cfl_leaf<<<d->nleaves, 128, 0, (cudaStream_t)stream>>>(d->u, d->fstride, d->dx, d->gamma, d->gm1, d->eta,
                                                           d->ratio, d->bad);
  CK(cudaGetLastError(), "omb_cfl leaf launch");
  k_cfl_reduce<<<1, 1024, 0, (cudaStream_t)stream>>>(d->nleaves, d->ratio, d->bad, d->cfl, d->out, d->bad_leaf,
                                                     d->dt_dev);
  CK(cudaGetLastError(), "omb_cfl reduce launch");
  return 0;
}

int omb_leaf_sums(const double* U, long long fstride, int L, double* out, void* stream) {
  if (L <= 0) return 0;
  k_leaf_sums<<<(L * NF + 127) / 128, 128, 0, (cudaStream_t)stream>>>(U, fstride, L, out);
  CK(cudaGetLastError(), "omb_leaf_sums launch");
  return 0;
}

int omb_disk_order(const double* U, long long fstride, int L, double* out, void* stream) {
  if (L <= 0) return 0;
  long long total = (long long)L * NF * 512;
  int blocks = (int)((total + 255) / 256);
  k_disk_order<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(U, fstride, L, out);
  CK(cudaGetLastError(), "omb_disk_order launch");
  return 0;
}

int omb_gather_rows(const double* src, long long row, const int* idx, int n, double* out, void* stream) {
  if (n <= 0) return 0;
  long long total = (long long)n * row;
  int blocks = (int)((total + 255) / 256);
  k_rows<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(src, row, idx, n, out, 0);
  CK(cudaGetLastError(), "omb_gather_rows launch");
  return 0;
}

int omb_scatter_rows(const double* in, long long row, const int* idx, int n, double* dst, void* stream) {
  if (n <= 0) return 0;
  long long total = (long long)n * row;
  int blocks = (int)((total + 255) / 256);
  k_rows<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(in, row, idx, n, dst, 1);
  CK(cudaGetLastError(), "omb_scatter_rows launch");
  return 0;
}

int omb_pack_leaves(const double* U, long long fstride, const int* idx, int n, double* out, void* stream) {
  if (n <= 0) return 0;
  long long total = (long long)n * NF * 512;
  int blocks = (int)((total + 255) / 256);
  k_pack<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(U, fstride, idx, n, out);
  CK(cudaGetLastError(), "omb_pack_leaves launch");
  return 0;
}

int omb_unpack_leaves(const double* in, int n, double* U, long long fstride, int first, void* stream) {
  if (n <= 0) return 0;
  long long total = (long long)n * NF * 512;
  int blocks = (int)((total + 255) / 256);
  k_unpack<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(in, n, U, fstride, first);
  CK(cudaGetLastError(), "omb_unpack_leaves launch");
  return 0;
}

int omb_selftest_div(unsigned long long seed, long long n, unsigned long long* bad, void* stream) {
  k_selftest_div<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(seed, n, bad);
  CK(cudaGetLastError(), "omb_selftest_div launch");
  return 0;
}

int omb_kt_flux(const double* left, const double* right, int n, int axis, double gamma, double* out, int* bad,
                void* stream) {
  if (n <= 0) return 0;
  if (axis < 0 || axis > 2) return set_err("omb_kt_flux: axis must be 0, 1 or 2");
  k_kt_points<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(left, right, n, axis, gamma, out, bad);
  CK(cudaGetLastError(), "omb_kt_flux launch");
  return 0;
}

int omb_physical_flux(const double* states, int n, int axis, double* out, void* stream) {
  if (n <= 0) return 0;
  if (axis < 0 || axis > 2) return set_err("omb_physical_flux: axis must be 0, 1 or 2");
  k_physical_points<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(states, n, axis, out);
  CK(cudaGetLastError(), "omb_physical_flux launch");
  return 0;
}

int omb_face_flux(const double* pts, int n, int new_mode, double* out, void* stream) {
  if (n <= 0) return 0;
  k_face_points<<<(n * NF + 127) / 128, 128, 0, (cudaStream_t)stream>>>(pts, n, new_mode, out);
  CK(cudaGetLastError(), "omb_face_flux launch");
  return 0;
}

int omb_scalar_input(const double* u, long long fstride, int n_all, const double* x, int n_x, double gamma,
                     double gm1, double eta, double* dst, void* stream) {
  if (n_all <= 0) return 0;
  long long n = (long long)n_all * 512;
  int blocks = (int)((n + 255) / 256);
  k_scalar_input<<<blocks < 148 * 16 ? blocks : 148 * 16, 256, 0, (cudaStream_t)stream>>>(u, fstride, n_all, x, n_x,
                                                                                           gamma, gm1, eta, dst);
  CK(cudaGetLastError(), "omb_scalar_input launch");
  return 0;
}

int omb_selftest_pow(const double* x, const double* y, long long n, double* out, void* stream) {
  if (n <= 0) return 0;
  k_pow_batch<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(x, y, n, out);
  CK(cudaGetLastError(), "omb_selftest_pow launch");
  return 0;
}

// host-side packing of the per-leaf padded arrays (the reference's SubGrid.u,
// (6, m, m, m) C-contiguous) into / out of the [6][L][n^3] device layout;
// multithreaded memcpy of n-element rows
// A small persistent pool for the host-side copies: run(f, nt) calls f(t) for
// t = 0..nt-1, t = 0 on the caller's thread, and returns when all are done.
// (Spawning 16 threads per transfer cost ~1 ms of the ~5 ms upload.)
class HostPool {
 public:
  void run(const std::function<void(int)>& f, int nt) {
    std::lock_guard<std::mutex> serial(run_mu_);  // one job at a time
    ensure(nt - 1);
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      njob_ = nt;
      pending_ = nt - 1;
      gen_++;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void ensure(int n) {
    while ((int)th_.size() < n) {
      int id = (int)th_.size() + 1;
      th_.emplace_back([this, id] { loop(id); });
      th_.back().detach();
    }
  }
  void loop(int id) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= njob_) continue;
        f = job_;
      }
      (*f)(id);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* job_ = nullptr;
  int njob_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
};
static HostPool& host_pool() {
  static HostPool* p = new HostPool();  // never destroyed: its detached threads outlive main
  return *p;
}

static std::atomic<int> g_host_threads(0);  // 0: hardware_concurrency (capped at 16)
static int host_workers(int L) {
  unsigned nt = g_host_threads.load() > 0 ? (unsigned)g_host_threads.load() : std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 16) nt = 16;
  if ((long long)nt > L) nt = L > 0 ? (unsigned)L : 1u;
  return (int)nt;
}
}  // extern "C"
// one unit = an n^3 interior inside a padded host array of edge m: a whole leaf
// (m = n + 6, u = the leaf's array) or an 8^3 block of a 16^3 / 32^3 leaf (u = the
// leaf's array advanced to the block's corner, m = the leaf's padded edge)
template <int NN, int MM>
static void copy_leaf_n(const double* u, double* packed, int i, long long fstride, bool to_packed) {
  constexpr long long n3 = (long long)NN * NN * NN;
  // packing: whole 64-byte rows of the (pinned) staging buffer are written
  // with streaming stores -- no read-for-ownership of the destination lines
  const bool stream = to_packed && NN % 2 == 0 && ((uintptr_t)packed & 15) == 0 && (fstride % 2) == 0;
  for (int v = 0; v < 6; v++) {
    double* P = packed + (long long)v * fstride + (long long)i * n3;
    double* Q = const_cast<double*>(u) + (long long)v * MM * MM * MM + (3 * MM + 3) * MM + 3;
    for (int x = 0; x < NN; x++)
      for (int y = 0; y < NN; y++) {
        double* p = P + (x * NN + y) * NN;
        double* q = Q + (x * MM + y) * MM;
        if (stream) {
#pragma unroll
          for (int k = 0; k < NN; k += 2) _mm_stream_pd(p + k, _mm_loadu_pd(q + k));
        } else if (to_packed) {
          memcpy(p, q, sizeof(double) * NN);  // constant size: inlined vector moves
        } else {
          memcpy(q, p, sizeof(double) * NN);
        }
      }
  }
  if (stream) _mm_sfence();
}
extern "C" {
static void copy_leaf(const double* u, double* packed, int i, int n, int m, long long fstride, bool to_packed) {
  if (n == 8 && m == 14) return copy_leaf_n<8, 14>(u, packed, i, fstride, to_packed);
  if (n == 8 && m == 22) return copy_leaf_n<8, 22>(u, packed, i, fstride, to_packed);
  if (n == 8 && m == 38) return copy_leaf_n<8, 38>(u, packed, i, fstride, to_packed);
  long long n3 = (long long)n * n * n;
  for (int v = 0; v < 6; v++)
    for (int x = 0; x < n; x++)
      for (int y = 0; y < n; y++) {
        double* p = packed + (long long)v * fstride + (long long)i * n3 + ((long long)x * n + y) * n;
        double* q = const_cast<double*>(u) + (((long long)v * m + x + 3) * m + y + 3) * m + 3;
        if (to_packed) memcpy(p, q, sizeof(double) * n);
        else memcpy(q, p, sizeof(double) * n);
      }
}

static void host_copy(const double* const* leaf_u, int L, int n, int m, long long fstride, double* packed,
                      bool to_packed) {
  const int nt = host_workers(L);
  host_pool().run([&](int t) {
    for (int i = (int)((long long)L * t / nt); i < (int)((long long)L * (t + 1) / nt); i++)
      copy_leaf(leaf_u[i], packed, i, n, m, fstride, to_packed);
  }, nt);
}

// host threads of the pack / unpack / transfer pool (0 = all cores); ranks sharing a host split them
int omb_set_host_threads(int n) {
  g_host_threads.store(n < 0 ? 0 : n);
  return 0;
}

static bool bad_pitch(int n, int m) { return n <= 0 || m < n + 6; }

int omb_host_pack(const double* const* leaf_u, int L, int n, int m, long long fstride, double* out) {
  if (bad_pitch(n, m)) return set_err("omb_host_pack: padded edge m < n + 6");
  host_copy(leaf_u, L, n, m, fstride, out, true);
  return 0;
}

int omb_host_unpack(const double* in, int L, int n, int m, long long fstride, double* const* leaf_u) {
  if (bad_pitch(n, m)) return set_err("omb_host_unpack: padded edge m < n + 6");
  host_copy((const double* const*)leaf_u, L, n, m, fstride, const_cast<double*>(in), false);
  return 0;
}

// Pipelined host <-> device transfer of the state of record (the leaves'
// padded host arrays): the leaves are cut into chunks; worker threads pack
// chunk c into the pinned staging buffer while the copy engine moves chunk
// c-1 (upload), or unpack chunk c while chunk c+1 is still in flight
// (download).  One 2D copy per chunk covers the 6 field planes.
int omb_host_upload(const double* const* leaf_u, int L, int n, int m, long long fstride, double* pinned,
                    double* dev, int nchunks, void* stream) {
  if (int rc = lib_init()) return rc;
  if (bad_pitch(n, m)) return set_err("omb_host_upload: padded edge m < n + 6");
  if (L <= 0) return 0;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > L) nchunks = L;
  const int nt = host_workers(L);
  const long long n3 = (long long)n * n * n;
  std::vector<std::atomic<int>> done(nchunks);
  for (auto& d : done) d.store(0);
  auto lo_of = [&](int c) { return (int)((long long)L * c / nchunks); };
  std::atomic<int> err(0);
  std::function<void(int)> work = [&](int t) {
    for (int c = 0; c < nchunks; c++) {
      int lo = lo_of(c), hi = lo_of(c + 1);
      int a = lo + (int)((long long)(hi - lo) * t / nt), b = lo + (int)((long long)(hi - lo) * (t + 1) / nt);
      for (int i = a; i < b; i++) copy_leaf(leaf_u[i], pinned, i, n, m, fstride, true);
      // the thread finishing chunk c last hands it to the copy engine
      if (done[c].fetch_add(1, std::memory_order_acq_rel) == nt - 1) {
        cudaError_t e = cudaMemcpy2DAsync(dev + lo * n3, fstride * 8, pinned + lo * n3, fstride * 8,
                                          (size_t)(hi - lo) * n3 * 8, 6, cudaMemcpyHostToDevice, (cudaStream_t)stream);
        if (e != cudaSuccess) err.store((int)e);
      }
    }
  };
  host_pool().run(work, nt);
  CK((cudaError_t)err.load(), "omb_host_upload copy");
  return 0;
}

int omb_host_download(const double* dev, double* pinned, int L, int n, int m, long long fstride,
                      double* const* leaf_u, int nchunks, void* stream) {
  if (int rc = lib_init()) return rc;
  if (bad_pitch(n, m)) return set_err("omb_host_download: padded edge m < n + 6");
  if (L <= 0) return 0;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > L) nchunks = L;
  const int nt = host_workers(L);
  const long long n3 = (long long)n * n * n;
  auto lo_of = [&](int c) { return (int)((long long)L * c / nchunks); };
  std::vector<cudaEvent_t> ev(nchunks);
  for (int c = 0; c < nchunks; c++) {
    CK(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming), "omb_host_download event");
    int lo = lo_of(c), hi = lo_of(c + 1);
    CK(cudaMemcpy2DAsync(pinned + lo * n3, fstride * 8, dev + lo * n3, fstride * 8, (size_t)(hi - lo) * n3 * 8, 6,
                         cudaMemcpyDeviceToHost, (cudaStream_t)stream), "omb_host_download copy");
    CK(cudaEventRecord(ev[c], (cudaStream_t)stream), "omb_host_download record");
  }
  std::atomic<int> bad(0);
  std::function<void(int)> work = [&](int t) {
    for (int c = 0; c < nchunks; c++) {
      if (cudaEventSynchronize(ev[c]) != cudaSuccess) { bad.store(1); return; }
      int lo = lo_of(c), hi = lo_of(c + 1);
      int a = lo + (int)((long long)(hi - lo) * t / nt), b = lo + (int)((long long)(hi - lo) * (t + 1) / nt);
      for (int i = a; i < b; i++) copy_leaf(leaf_u[i], pinned, i, n, m, fstride, false);
    }
  };
  host_pool().run(work, nt);
  for (auto& e : ev) cudaEventDestroy(e);
  if (bad.load()) return set_err("omb_host_download: copy failed");
  return 0;
}

/* Zero-copy host transfers: the leaves' padded arrays live in mapped pinned host
   memory (the stepper re-homes SubGrid.u into one pinned slab), and these kernels
   read / write them over PCIe directly -- no host thread touches the data.  The unit
   is a (leaf, field, x) span: rows y = 3..10 of the padded array with all 14 z
   (112 doubles), widened to the whole 64 B host lines it touches -- it starts 2 or 6
   doubles into a line, so its hull is exactly 15 lines (120 doubles).  The span's
   interior z = 3..10 go to / come from the device state; its ghost z and the hull's
   edge doubles (neighbouring rows of the padded array) to / from `stash`, so the
   download writes whole lines only (no partial-line read-modify-write on the host)
   and leaves every host ghost cell exactly as it was.  Replaces the per-leaf
   interior copies of octomini's host state of record (mesh/tree.py:58-61). */
constexpr int HULL = 120;              // doubles per span hull (15 lines of 64 B)
constexpr int SPANS_PER_LEAF = 6 * 8;  // (field, x)
constexpr int STASH_PER_SPAN = 56;     // 8 rows x 6 ghost z + 8 edge doubles

__device__ __forceinline__ int span_src(int f, int x) { return ((f * 14 + x + 3) * 14 + 3) * 14; }

// hull position j of span (f, x): its offset in the leaf's padded array, and
// either the interior cell (x, y, z - 3) (returns true) or the stash slot
__device__ __forceinline__ bool hull_pos(int f, int x, int j, int& src, int& cell, int& slot) {
  int s0 = span_src(f, x), r = s0 & 7;  // 2 or 6 (leaf arrays are 64 B aligned)
  src = s0 - r + j;
  int p = j - r;  // position inside the span
  if (p < 0) { slot = j; return false; }
  if (p >= 8 * 14) { slot = r + 48 + (p - 8 * 14); return false; }
  int y = p / 14, z = p - y * 14;
  if (z >= 3 && z <= 10) { cell = x * 64 + y * 8 + (z - 3); return true; }
  slot = r + y * 6 + (z < 3 ? z : z - 8);
  return false;
}

__global__ void __launch_bounds__(256) k_host_gather(const double* const* __restrict__ leaf_u, unsigned total,
                                                     long long fstride, double* __restrict__ dev,
                                                     double* __restrict__ stash) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    unsigned sp = i / HULL, j = i - sp * HULL;
    unsigned leaf = sp / SPANS_PER_LEAF, fx = sp - leaf * SPANS_PER_LEAF;
    int f = fx >> 3, x = fx & 7, src, cell, slot;
    bool in = hull_pos(f, x, (int)j, src, cell, slot);
    double v = __ldcs(leaf_u[leaf] + src);
    if (in)
      dev[f * fstride + leaf * 512LL + cell] = v;
    else
      stash[sp * STASH_PER_SPAN + slot] = v;
  }
}

__global__ void __launch_bounds__(256) k_host_scatter(const double* __restrict__ dev, const double* __restrict__ stash,
                                                      unsigned total, long long fstride,
                                                      double* const* __restrict__ leaf_u) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    unsigned sp = i / HULL, j = i - sp * HULL;
    unsigned leaf = sp / SPANS_PER_LEAF, fx = sp - leaf * SPANS_PER_LEAF;
    int f = fx >> 3, x = fx & 7, src, cell, slot;
    bool in = hull_pos(f, x, (int)j, src, cell, slot);
    double v = in ? dev[f * fstride + leaf * 512LL + cell] : stash[sp * STASH_PER_SPAN + slot];
    __stcs(leaf_u[leaf] + src, v);
  }
}

static int host_xfer_grid(long long total) {
  long long b = (total + 255) / 256;
  return (int)(b < 148 * 8 ? b : 148 * 8);
}

int omb_host_gather(const double* const* leaf_u, int L, long long fstride, double* dev, double* stash,
                    void* stream) {
  if (int rc = lib_init()) return rc;
  if (L <= 0) return 0;
  if ((long long)L * SPANS_PER_LEAF * HULL >= (1LL << 32)) return set_err("omb_host_gather: too many leaves");
  unsigned total = (unsigned)L * SPANS_PER_LEAF * HULL;
  k_host_gather<<<host_xfer_grid(total), 256, 0, (cudaStream_t)stream>>>(leaf_u, total, fstride, dev, stash);
  CK(cudaGetLastError(), "omb_host_gather launch");
  return 0;
}

int omb_host_scatter(const double* dev, const double* stash, int L, long long fstride, double* const* leaf_u,
                     void* stream) {
  if (int rc = lib_init()) return rc;
  if (L <= 0) return 0;
  if ((long long)L * SPANS_PER_LEAF * HULL >= (1LL << 32)) return set_err("omb_host_scatter: too many leaves");
  unsigned total = (unsigned)L * SPANS_PER_LEAF * HULL;
  k_host_scatter<<<host_xfer_grid(total), 256, 0, (cudaStream_t)stream>>>(dev, stash, total, fstride, leaf_u);
  CK(cudaGetLastError(), "omb_host_scatter launch");
  return 0;
}

/* The download overlapped with the stage that produces it: chunk c (leaves
   [bounds[c], bounds[c+1])) is copied on copy_stream once `ready[c]` (an event
   the caller recorded after the launch part that finishes those leaves) has
   fired, and unpacked by the host threads as soon as its copy is done. */
int omb_host_download_after(const double* dev, double* pinned, int n, int m, long long fstride,
                            double* const* leaf_u, int nchunks, const int* bounds, void* const* ready,
                            void* copy_stream) {
  if (int rc = lib_init()) return rc;
  if (bad_pitch(n, m)) return set_err("omb_host_download_after: padded edge m < n + 6");
  if (nchunks <= 0) return 0;
  const int L = bounds[nchunks];
  if (L <= 0) return 0;
  const int nt = host_workers(L);
  const long long n3 = (long long)n * n * n;
  std::vector<cudaEvent_t> ev(nchunks);
  for (int c = 0; c < nchunks; c++) {
    CK(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming), "omb_host_download_after event");
    int lo = bounds[c], hi = bounds[c + 1];
    CK(cudaStreamWaitEvent((cudaStream_t)copy_stream, (cudaEvent_t)ready[c], 0), "omb_host_download_after wait");
    if (hi > lo)
      CK(cudaMemcpy2DAsync(pinned + lo * n3, fstride * 8, dev + lo * n3, fstride * 8, (size_t)(hi - lo) * n3 * 8, 6,
                           cudaMemcpyDeviceToHost, (cudaStream_t)copy_stream), "omb_host_download_after copy");
    CK(cudaEventRecord(ev[c], (cudaStream_t)copy_stream), "omb_host_download_after record");
  }
  std::atomic<int> bad(0);
  std::function<void(int)> work = [&](int t) {
    for (int c = 0; c < nchunks; c++) {
      if (cudaEventSynchronize(ev[c]) != cudaSuccess) { bad.store(1); return; }
      int lo = bounds[c], hi = bounds[c + 1];
      int a = lo + (int)((long long)(hi - lo) * t / nt), b = lo + (int)((long long)(hi - lo) * (t + 1) / nt);
      for (int i = a; i < b; i++) copy_leaf(leaf_u[i], pinned, i, n, m, fstride, false);
    }
  };
  host_pool().run(work, nt);
  for (auto& e : ev) cudaEventDestroy(e);
  if (bad.load()) return set_err("omb_host_download_after: copy failed");
  return 0;
}

/* FP64 peak probe: launches blocks x 256 threads x 8 chains x iters DFMAs */
int omb_fp64_peak(double* scratch, int blocks, int iters, void* stream) {
  k_dfma_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>(scratch, iters);
  CK(cudaGetLastError(), "omb_fp64_peak launch");
  return 0;
}

int omb_gather(const double* u, long long fstride, const OmbLeafInfo* info, int leaf, int bc, double* out,
               void* stream) {
  if (int rc = lib_init()) return rc;
  k_gather<<<11, 256, 0, (cudaStream_t)stream>>>(u, fstride, (const LeafInfo*)info, leaf, bc, out);
  CK(cudaGetLastError(), "omb_gather launch");
  return 0;
}

int omb_gather_leaves(const double* u, long long fstride, const OmbLeafInfo* info, int first, int n, int bc,
                      double* out, void* stream) {
  if (int rc = lib_init()) return rc;
  if (n <= 0) return 0;
  if (n > 65535) return set_err("omb_gather_leaves: more than 65535 leaves per call");
  k_gather<<<dim3(11, n), 256, 0, (cudaStream_t)stream>>>(u, fstride, (const LeafInfo*)info, first, bc, out);
  CK(cudaGetLastError(), "omb_gather_leaves launch");
  return 0;
}

}  // extern "C"
