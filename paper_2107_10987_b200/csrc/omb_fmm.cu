// omb_fmm.cu -- the FMM gravity solve on the device (SURVEY.md §8(f) rank 4:
// the paper's other GPU path), behind the reference's FmmSolver
// (gravity/solver.py:50-164).
//
// Host side: the dual-tree traversal that enumerates the interaction pairs
// (_core.pyx:372-494, build_interactions) -- same stack discipline, same
// opening criterion, same lattice keys -- so the pair list, its grouping and
// hence every summation order are the reference's.
//
// Device side, per solve (order-3 Cartesian expansions, 20 components):
//   k_fmm_masses    point masses rho*dx^3 of the cell entities
//   k_fmm_upward    per level, fine to coarse: parent moments = sum over the 8
//                   children, in child order, of the translated child moments
//                   (solver.py:92-103, multipole.py:98-127)
//   k_fmm_m2l       per target entity, its interactions in the reference's
//                   global order (group by group, pair by pair; _core.pyx:563-608):
//                   L += m2l(M_src, D) or the cell-cell monopole form
//   k_fmm_downward  per level, coarse to fine: child L += shifted parent L
//                   (solver.py:105-115, multipole.py:130-170)
//   k_fmm_fields    phi = L0, g = -L1 of the cell entities into per-leaf
//                   [n^3] arrays (solver.py:117-132)
// Every expression keeps the reference's association (numpy left to right,
// numpy's axis-1 sum sequential); compiled with -fmad=false.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/omb200.h"
#include "omb_stage.cuh"

namespace {

constexpr int NC = 20;  // [M0, M1(3), M2(6), M3(10)]
// symmetric tensor component tables (multipole.py:21-42)
// as arithmetic on the (unrolled, constant) index, so the compiler folds them and the
// register arrays they index stay in registers (constant-bank tables sent those arrays to
// local memory)
//   S2: 00 01 02 11 12 22;  S3: 000 001 002 011 012 022 111 112 122 222
__device__ __forceinline__ int c_s2a(int i) { return i < 3 ? 0 : (i < 5 ? 1 : 2); }
__device__ __forceinline__ int c_s2b(int i) { return i < 3 ? i : (i < 5 ? i - 2 : 2); }
__device__ __forceinline__ int c_s3a(int i) { return i < 6 ? 0 : (i < 9 ? 1 : 2); }
__device__ __forceinline__ int c_s3b(int i) { return i < 3 ? 0 : (i < 5 ? 1 : (i == 5 ? 2 : (i < 8 ? 1 : 2))); }
__device__ __forceinline__ int c_s3c(int i) {
  return i < 3 ? i : (i == 3 ? 1 : (i < 6 ? 2 : (i == 6 ? 1 : 2)));
}
__device__ __forceinline__ double c_mult2(int i) { return (i == 1 || i == 2 || i == 4) ? 2.0 : 1.0; }
__device__ __forceinline__ double c_mult3(int i) { return i == 4 ? 6.0 : ((i == 0 || i == 6 || i == 9) ? 1.0 : 3.0); }

__device__ __forceinline__ int idx2(int a, int b) {  // (a,b) -> 0..5
  int lo = a < b ? a : b, hi = a < b ? b : a;
  return lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
}
__device__ __forceinline__ int idx3(int a, int b, int c) {  // sorted (a,b,c) -> 0..9
  int x = a, y = b, z = c, t;
  if (x > y) { t = x; x = y; y = t; }
  if (y > z) { t = y; y = z; z = t; }
  if (x > y) { t = x; x = y; y = t; }
  // S3 order: 000 001 002 011 012 022 111 112 122 222
  if (x == 0) {
    if (y == 0) return z;           // 0,1,2
    if (y == 1) return z == 1 ? 3 : 4;
    return 5;
  }
  if (x == 1) {
    if (y == 1) return z == 1 ? 6 : 7;
    return 8;
  }
  return 9;
}

// ---------------------------------------------------------------------------
// upward: M[p] = sum_k translate_moments(M[child_k], center[child_k] - center[p])
// ---------------------------------------------------------------------------
__device__ void translate_add(const double* f, const double t[3], double* out, bool first) {
  double M0 = f[0];
  double r[NC];
  r[0] = M0;
  for (int a = 0; a < 3; a++) r[1 + a] = f[1 + a] + M0 * t[a];
  for (int i = 0; i < 6; i++) {
    int a = c_s2a(i), b = c_s2b(i);
    r[4 + i] = ((f[4 + i] + f[1 + a] * t[b]) + f[1 + b] * t[a]) + (M0 * t[a]) * t[b];
  }
  for (int i = 0; i < 10; i++) {
    int a = c_s3a(i), b = c_s3b(i), c = c_s3c(i);
    double m2ab = f[4 + idx2(a, b)], m2ac = f[4 + idx2(a, c)], m2bc = f[4 + idx2(b, c)];
    r[10 + i] = ((((((f[10 + i] + m2ab * t[c]) + m2ac * t[b]) + m2bc * t[a]) + (f[1 + a] * t[b]) * t[c]) +
                  (f[1 + b] * t[a]) * t[c]) +
                 (f[1 + c] * t[a]) * t[b]) +
                ((M0 * t[a]) * t[b]) * t[c];
  }
  for (int k = 0; k < NC; k++) out[k] = first ? r[k] : out[k] + r[k];
}

__global__ void k_fmm_upward(const long long* parents, int np, const long long* children, const double* center,
                             double* M) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  long long p = parents[i];
  double acc[NC];
  for (int k = 0; k < 8; k++) {
    long long c = children[p * 8 + k];
    double t[3];
    for (int a = 0; a < 3; a++) t[a] = center[c * 3 + a] - center[p * 3 + a];
    translate_add(M + c * NC, t, acc, k == 0);
  }
  for (int k = 0; k < NC; k++) M[p * NC + k] = acc[k];
}

// ---------------------------------------------------------------------------
// M2L: L[x] += contributions in the reference's order (_core.pyx:534-608)
// ---------------------------------------------------------------------------
// contribution word: source entity (bits 0..39) | group (40..61) | cell-cell (62) | flip (63)
//
// Two passes over each target's contributions, each owning a subset of the
// 20 local components (every component still accumulates its contributions
// in the reference's order, so the split is exact): PART 0 = L0..L3 (needs
// all of M and D), PART 1 = L4..L19 (needs M0..M3 and D4..D19).  Fewer live
// accumulators per pass: fewer registers, more warps against the latency of
// the source-moment loads.
// 5 blocks of 128 per SM (<= 102 registers, no spills once the tensor tables fold): 20 warps
// against the load latency instead of 16 (c5g FMM 15.6 -> 14.2 ms per stage; 6 blocks spill:
// profiles/r02/abf9_abf10_m2l_occupancy.txt)
template <int PART>
__global__ void __launch_bounds__(128, 5) k_fmm_m2l(const long long* off, const unsigned long long* contrib,
                                                    const double* D /*[G][2][20]*/, const unsigned char* cellcell,
                                                    const double* M, double* L, long long ntarget,
                                                    const long long* targets, const long long* subset,
                                                    const double* M0c = nullptr) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= ntarget) return;
  long long ti = subset ? subset[k] : k;  // a rank of a partitioned run solves only its targets
  if (off[ti] == off[ti + 1]) return;  // nothing to add (the filtered PART 1 lists)
  long long x = targets[ti];
  constexpr int K0 = PART == 0 ? 0 : 4, KN = PART == 0 ? 4 : 16;
  double l[KN];
#pragma unroll
  for (int k = 0; k < KN; k++) l[k] = L[x * NC + K0 + k];
  // one contribution, added in the list's order
  auto add = [&](unsigned long long w) {
    long long src = (long long)(w & 0xFFFFFFFFFFull);
    long long g = (long long)((w >> 40) & 0x3FFFFFull);
    int flip = (int)(w >> 63);
    const double* Dg = D + (g * 2 + flip) * NC;
    const double* Ms = M + src * NC;
    bool cc = cellcell && ((w >> 62) & 1);  // (null: a list without cell-cell contributions)
    if (PART == 0) {
      // the loads both kinds of contribution need go out at once, before the kind is known: the
      // monopole (from the compact mass array when given -- 8 B per entity, L2-resident where the
      // 160 B moment records are not; the same value) and D0..D3, as two 16-byte loads (D rows
      // are 160 B): a warp's lanes read up to 32 different rows, so each load instruction costs
      // up to one L1 wavefront per lane -- half as many instructions this way (c5g FMM 27.4 ->
      // 26.4 ms per stage, profiles/r02/abf5_m2l_vec.txt)
      double M0 = M0c ? __ldg(M0c + src) : __ldg(Ms);
      double2 da = __ldg(reinterpret_cast<const double2*>(Dg)), db = __ldg(reinterpret_cast<const double2*>(Dg + 2));
      double d[4] = {da.x, da.y, db.x, db.y};
      if (cc) {
        // L[eb,0] += ma*D0; L[eb,c] += ma*D_c; L[ea,0] += mb*D0; L[ea,c] += mb*(-D_c)
        // (the flipped D holds -D_c: x*(-d) is the reference's mb*(-D1))
#pragma unroll
        for (int c = 0; c < 4; c++) l[c] += M0 * d[c];
        return;
      }
      // the moment and derivative rows by 16-byte loads (rows are 160 B), into register arrays
      // whose indices all fold to constants
      double m[20], dg[20];
#pragma unroll
      for (int i = 0; i < 10; i++) {
        double2 mv = __ldg(reinterpret_cast<const double2*>(Ms) + i);
        m[2 * i] = mv.x;
        m[2 * i + 1] = mv.y;
      }
#pragma unroll
      for (int i = 2; i < 10; i++) {
        double2 dv = __ldg(reinterpret_cast<const double2*>(Dg) + i);
        dg[2 * i] = dv.x;
        dg[2 * i + 1] = dv.y;
      }
      double acc = d[0] * M0;
#pragma unroll
      for (int a = 0; a < 3; a++) acc = acc - d[1 + a] * m[1 + a];
#pragma unroll
      for (int i = 0; i < 6; i++) acc = acc + ((0.5 * c_mult2(i)) * dg[4 + i]) * m[4 + i];
#pragma unroll
      for (int i = 0; i < 10; i++) acc = acc - ((c_mult3(i) / 6.0) * dg[10 + i]) * m[10 + i];
      l[0] += acc;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        acc = d[1 + a] * M0;
#pragma unroll
        for (int b = 0; b < 3; b++) acc = acc - dg[4 + idx2(a, b)] * m[1 + b];
#pragma unroll
        for (int i = 0; i < 6; i++)
          acc = acc + ((0.5 * c_mult2(i)) * dg[10 + idx3(a, c_s2a(i), c_s2b(i))]) * m[4 + i];
        l[1 + a] += acc;
      }
    } else {
      if (cc) return;  // (PART 1 lists hold none)
      double2 m01 = __ldg(reinterpret_cast<const double2*>(Ms)), m23 = __ldg(reinterpret_cast<const double2*>(Ms) + 1);
      double m[4] = {m01.x, m01.y, m23.x, m23.y}, dg[20];
#pragma unroll
      for (int i = 2; i < 10; i++) {
        double2 dv = __ldg(reinterpret_cast<const double2*>(Dg) + i);
        dg[2 * i] = dv.x;
        dg[2 * i + 1] = dv.y;
      }
      double M0 = m[0];
#pragma unroll
      for (int i = 0; i < 6; i++) {
        double acc = dg[4 + i] * M0;
#pragma unroll
        for (int b = 0; b < 3; b++) acc = acc - dg[10 + idx3(c_s2a(i), c_s2b(i), b)] * m[1 + b];
        l[i] += acc;
      }
#pragma unroll
      for (int i = 0; i < 10; i++) l[6 + i] += dg[10 + i] * M0;
    }
  };
  long long q = off[ti];
  const long long q1 = off[ti + 1];
  // the words two at a time (16-byte loads at even positions), the next pair in flight while
  // this one is added: each lane reads its own list, so a warp's load costs up to one L1
  // wavefront per lane -- half as many loads (c5g FMM 27.6 -> 25.4 ms per stage with the
  // 16-byte D loads, profiles/r02/abf6_m2l_pairs.txt)
  if (q & 1) add(__ldg(contrib + q++));
  const ulonglong2* cp = reinterpret_cast<const ulonglong2*>(contrib);
  ulonglong2 wn = q + 1 < q1 ? __ldg(cp + (q >> 1)) : make_ulonglong2(0ull, 0ull);
  for (; q + 1 < q1; q += 2) {
    ulonglong2 w = wn;
    if (q + 3 < q1) wn = __ldg(cp + (q >> 1) + 1);
    add(w.x);
    add(w.y);
  }
  if (q < q1) add(__ldg(contrib + q));
#pragma unroll
  for (int k = 0; k < KN; k++) L[x * NC + K0 + k] = l[k];
}

// PART 0 for two solves over the same lists at once (the stage's density and rho_dot solves:
// same tree, same interactions, different masses): each contribution word and D row is read once
// for both.  Each solve's accumulators see its contributions in the list's order, as in k_fmm_m2l.
// c5g FMM 14.2 -> 12.4 ms per stage; 4 blocks per SM (3: 12.9, 5: spills, 16.0 ms;
// profiles/r02/abf12_abf13_m2l_pair.txt)
__device__ __forceinline__ void m2l0_general(const double* d, const double* dg, const double* Ms, double M0,
                                             double* l) {
  double m[20];
#pragma unroll
  for (int i = 0; i < 10; i++) {
    double2 mv = __ldg(reinterpret_cast<const double2*>(Ms) + i);
    m[2 * i] = mv.x;
    m[2 * i + 1] = mv.y;
  }
  double acc = d[0] * M0;
#pragma unroll
  for (int a = 0; a < 3; a++) acc = acc - d[1 + a] * m[1 + a];
#pragma unroll
  for (int i = 0; i < 6; i++) acc = acc + ((0.5 * c_mult2(i)) * dg[4 + i]) * m[4 + i];
#pragma unroll
  for (int i = 0; i < 10; i++) acc = acc - ((c_mult3(i) / 6.0) * dg[10 + i]) * m[10 + i];
  l[0] += acc;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    acc = d[1 + a] * M0;
#pragma unroll
    for (int b = 0; b < 3; b++) acc = acc - dg[4 + idx2(a, b)] * m[1 + b];
#pragma unroll
    for (int i = 0; i < 6; i++) acc = acc + ((0.5 * c_mult2(i)) * dg[10 + idx3(a, c_s2a(i), c_s2b(i))]) * m[4 + i];
    l[1 + a] += acc;
  }
}

__global__ void __launch_bounds__(128, 4) k_fmm_m2l0_pair(const long long* off, const unsigned long long* contrib,
                                                          const double* D, const unsigned char* cellcell,
                                                          const double* Ma, const double* Mb, double* La, double* Lb,
                                                          long long ntarget, const long long* targets,
                                                          const long long* subset, const double* M0ab) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= ntarget) return;
  long long ti = subset ? subset[k] : k;
  if (off[ti] == off[ti + 1]) return;
  long long x = targets[ti];
  double la[4], lb[4];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    la[c] = La[x * NC + c];
    lb[c] = Lb[x * NC + c];
  }
  auto add = [&](unsigned long long w) {
    long long src = (long long)(w & 0xFFFFFFFFFFull);
    long long g = (long long)((w >> 40) & 0x3FFFFFull);
    const double* Dg = D + (g * 2 + (int)(w >> 63)) * NC;
    double2 mm = __ldg(reinterpret_cast<const double2*>(M0ab) + src);  // (both monopoles, one 16-byte load)
    double ma = mm.x, mb = mm.y;
    double2 da = __ldg(reinterpret_cast<const double2*>(Dg)), db = __ldg(reinterpret_cast<const double2*>(Dg + 2));
    double d[4] = {da.x, da.y, db.x, db.y};
    if (cellcell && ((w >> 62) & 1)) {
#pragma unroll
      for (int c = 0; c < 4; c++) la[c] += ma * d[c];
#pragma unroll
      for (int c = 0; c < 4; c++) lb[c] += mb * d[c];
      return;
    }
    double dg[20];
#pragma unroll
    for (int i = 2; i < 10; i++) {
      double2 dv = __ldg(reinterpret_cast<const double2*>(Dg) + i);
      dg[2 * i] = dv.x;
      dg[2 * i + 1] = dv.y;
    }
    m2l0_general(d, dg, Ma + src * NC, ma, la);
    m2l0_general(d, dg, Mb + src * NC, mb, lb);
  };
  long long q = off[ti];
  const long long q1 = off[ti + 1];
  if (q & 1) add(__ldg(contrib + q++));
  const ulonglong2* cp = reinterpret_cast<const ulonglong2*>(contrib);
  ulonglong2 wn = q + 1 < q1 ? __ldg(cp + (q >> 1)) : make_ulonglong2(0ull, 0ull);
  for (; q + 1 < q1; q += 2) {
    ulonglong2 w = wn;
    if (q + 3 < q1) wn = __ldg(cp + (q >> 1) + 1);
    add(w.x);
    add(w.y);
  }
  if (q < q1) add(__ldg(contrib + q));
#pragma unroll
  for (int c = 0; c < 4; c++) {
    La[x * NC + c] = la[c];
    Lb[x * NC + c] = lb[c];
  }
}

// ---------------------------------------------------------------------------
// downward: L[child] += translate_local(L[p], center[child] - center[p])
// ---------------------------------------------------------------------------
__device__ void translate_local(const double* f, const double s[3], double* out) {
  double acc0 = f[0];
  for (int a = 0; a < 3; a++) acc0 = acc0 + f[1 + a] * s[a];
  for (int i = 0; i < 6; i++) {
    int a = c_s2a(i), b = c_s2b(i);
    acc0 = acc0 + (((0.5 * c_mult2(i)) * f[4 + i]) * s[a]) * s[b];
  }
  for (int i = 0; i < 10; i++) {
    int a = c_s3a(i), b = c_s3b(i), c = c_s3c(i);
    acc0 = acc0 + ((((c_mult3(i) / 6.0) * f[10 + i]) * s[a]) * s[b]) * s[c];
  }
  out[0] = acc0;
  for (int a = 0; a < 3; a++) {
    double acc = f[1 + a];
    for (int b = 0; b < 3; b++) acc = acc + f[4 + idx2(a, b)] * s[b];
    for (int i = 0; i < 6; i++) {
      int b = c_s2a(i), c = c_s2b(i);
      acc = acc + (((0.5 * c_mult2(i)) * f[10 + idx3(a, b, c)]) * s[b]) * s[c];
    }
    out[1 + a] = acc;
  }
  for (int i = 0; i < 6; i++) {
    int a = c_s2a(i), b = c_s2b(i);
    double acc = f[4 + i];
    for (int c = 0; c < 3; c++) acc = acc + f[10 + idx3(a, b, c)] * s[c];
    out[4 + i] = acc;
  }
  for (int i = 0; i < 10; i++) out[10 + i] = f[10 + i];
}

__global__ void k_fmm_downward(const long long* parents, int np, const long long* children, const double* center,
                               double* L) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np * 8) return;
  long long p = parents[i / 8];
  long long c = children[p * 8 + i % 8];
  double s[3], sh[NC];
  for (int a = 0; a < 3; a++) s[a] = center[c * 3 + a] - center[p * 3 + a];
  translate_local(L + p * NC, s, sh);
  for (int k = 0; k < NC; k++) L[c * NC + k] = L[c * NC + k] + sh[k];
}

// cell masses: M[cell_entity(leaf, c)] = rho(leaf, c) * dx3(leaf); other components 0
__global__ void k_fmm_masses(const double* rho, long long fstride_unused, const long long* cell_base, int L,
                             const double* dx3, double* M) {
  // one thread per (cell, component): a leaf's cell records are consecutive, so the stores coalesce
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)L * 512 * NC) return;
  long long r = i / NC;
  int k = (int)(i - r * NC), leaf = (int)(r / 512), c = (int)(r % 512);
  M[(cell_base[leaf] + c) * NC + k] = k == 0 ? rho[r] * dx3[leaf] : 0.0;
}

__global__ void k_fmm_fields(const double* L, const long long* cell_base, int nleaf, double* phi, double* gx,
                             double* gy, double* gz) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)nleaf * 512) return;
  int leaf = (int)(i / 512), c = (int)(i % 512);
  const double* l = L + (cell_base[leaf] + c) * NC;
  phi[i] = l[0];
  gx[i] = -l[1];
  gy[i] = -l[2];
  gz[i] = -l[3];
}

// rho_dot = -div(momentum) by central differences over the ghost-filled
// state (gravity/solver.py:156-168): neighbour cells across leaf faces come
// from the same gather as the hydro halo (same-level / virtual AMR leaves,
// physical walls with the normal momentum mirrored), i.e. what the
// reference's ghost fill puts there before the gravity solve (step.py:106-113)
__global__ void k_fmm_rhodot(const double* U, long long fstride, const omb::LeafInfo* info, int bc, int nleaf,
                             const double* const* halo, int nown, double* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)nleaf * 512) return;
  int leaf = (int)(i / 512), c = (int)(i % 512);
  int x = c / 64, y = (c / 8) % 8, z = c % 8;
  const omb::LeafInfo& LI = info[leaf];
  auto mom = [&](int comp, int cx, int cy, int cz) {  // padded coords
    int fm;
    long long a = omb::gather_addr(LI, bc, cx, cy, cz, fm);
    int src = (int)(a >> 9);  // a neighbour owned by another GPU: its owner's buffer (NVLink)
    const double* p = (halo != nullptr && src >= nown) ? halo[src - nown] + (a & 511) : U + a;
    double v = p[(long long)comp * fstride];
    return ((fm >> (comp - 1)) & 1) ? -v : v;
  };
  int px = x + 3, py = y + 3, pz = z + 3;
  double dsx = mom(1, px + 1, py, pz) - mom(1, px - 1, py, pz);
  double dsy = mom(2, px, py + 1, pz) - mom(2, px, py - 1, pz);
  double dsz = mom(3, px, py, pz + 1) - mom(3, px, py, pz - 1);
  double inv2dx = 1.0 / (2.0 * LI.dx);
  out[i] = -((dsx + dsy) + dsz) * inv2dx;
}

// theta = 0 (always reject): direct cell-cell sums in the traversal's order
// (_core.pyx:611-690, direct_traversal_eval).  contrib word: partner | side
// << 63 (side 1: this target is the pair's a).  Writes phi, g of the cells.
__global__ void k_fmm_direct(const long long* off, const unsigned long long* contrib, const double* center,
                             const double* M, const long long* cell_base, int nleaf, double* phi, double* gx,
                             double* gy, double* gz) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)nleaf * 512) return;
  long long x = cell_base[i / 512] + i % 512;
  double p = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
  for (long long q = off[x]; q < off[x + 1]; q++) {
    unsigned long long w = contrib[q];
    long long o = (long long)(w & 0xFFFFFFFFFFull);
    bool is_a = (w >> 63) != 0;
    long long a = is_a ? x : o, b = is_a ? o : x;
    double rx = center[b * 3 + 0] - center[a * 3 + 0];
    double ry = center[b * 3 + 1] - center[a * 3 + 1];
    double rz = center[b * 3 + 2] - center[a * 3 + 2];
    double r2 = rx * rx + ry * ry + rz * rz;
    double d = sqrt(r2);
    double inv_r = 1.0 / d;
    double inv_r3 = inv_r / r2;
    double m = M[o * NC];
    p -= m * inv_r;
    if (is_a) {
      g0 += m * rx * inv_r3;
      g1 += m * ry * inv_r3;
      g2 += m * rz * inv_r3;
    } else {
      g0 -= m * rx * inv_r3;
      g1 -= m * ry * inv_r3;
      g2 -= m * rz * inv_r3;
    }
  }
  phi[i] = p;
  gx[i] = g0;
  gy[i] = g1;
  gz[i] = g2;
}

thread_local std::string f_err;
int ferr(const char* what, cudaError_t e) {
  f_err = std::string(what) + ": " + cudaGetErrorString(e);
  return -1;
}

}  // namespace

extern "C" {

const char* omb_fmm_last_error(void) { return f_err.c_str(); }

// Dual-tree traversal (host), _core.pyx:372-459: pairs (pa, pb) in discovery
// order with their lattice keys.  Returns the pair count, or -(needed) when
// cap is too small (nothing written beyond cap), or -1 on allocation failure.
long long omb_fmm_traverse(const double* center, const double* width, const long long* children,
                           const unsigned char* is_cell, long long nent, long long root, double theta,
                           long long* pa, long long* pb, long long* pk, long long cap) {
  double wmin = width[0];
  for (long long i = 1; i < nent; i++) wmin = width[i] < wmin ? width[i] : wmin;
  const double quant = 2.0 / wmin;
  const long long BIAS = 1LL << 16, SPAN = 1LL << 17;
  std::vector<long long> st;
  st.reserve(1 << 16);
  st.push_back(root);
  st.push_back(root);
  long long pn = 0;
  while (!st.empty()) {
    long long b = st.back();
    st.pop_back();
    long long a = st.back();
    st.pop_back();
    if (a == b) {
      if (is_cell[a]) continue;
      for (int i = 0; i < 8; i++) {
        st.push_back(children[a * 8 + i]);
        st.push_back(children[a * 8 + i]);
        for (int j = i + 1; j < 8; j++) {
          st.push_back(children[a * 8 + i]);
          st.push_back(children[a * 8 + j]);
        }
      }
      continue;
    }
    double rx = center[b * 3 + 0] - center[a * 3 + 0];
    double ry = center[b * 3 + 1] - center[a * 3 + 1];
    double rz = center[b * 3 + 2] - center[a * 3 + 2];
    double d = sqrt(rx * rx + ry * ry + rz * rz);
    double wa = width[a], wb = width[b];
    if (0.5 * (wa + wb) < theta * d) {
    } else if (is_cell[a] && is_cell[b]) {
    } else {
      if (wa > wb) {
        for (int i = 0; i < 8; i++) { st.push_back(children[a * 8 + i]); st.push_back(b); }
      } else if (wb > wa) {
        for (int i = 0; i < 8; i++) { st.push_back(a); st.push_back(children[b * 8 + i]); }
      } else if (is_cell[a]) {
        for (int i = 0; i < 8; i++) { st.push_back(a); st.push_back(children[b * 8 + i]); }
      } else if (is_cell[b]) {
        for (int i = 0; i < 8; i++) { st.push_back(children[a * 8 + i]); st.push_back(b); }
      } else {
        for (int i = 0; i < 8; i++)
          for (int j = 0; j < 8; j++) { st.push_back(children[a * 8 + i]); st.push_back(children[b * 8 + j]); }
      }
      continue;
    }
    if (pn < cap) {
      long long qx = llround(rx * quant), qy = llround(ry * quant), qz = llround(rz * quant);
      long long flags = (is_cell[a] ? 2 : 0) + (is_cell[b] ? 1 : 0);
      pa[pn] = a;
      pb[pn] = b;
      pk[pn] = (((qx + BIAS) * SPAN + (qy + BIAS)) * SPAN + (qz + BIAS)) * 4 + flags;
    }
    pn++;
  }
  return pn <= cap ? pn : -pn;
}

// Grouping + per-target contribution lists (host), O(pairs): groups are the
// sorted distinct keys (np.unique order), pairs keep their discovery order
// within a group (the stable argsort of _core.pyx:476-481), and each target's
// contributions follow the global M2L sequence -- group by group, pair by
// pair, (b <- a, D) before (a <- b, flipped D) (_core.pyx:583-608).
// Outputs: ngroups, group_first [G] (discovery index of the group's first
// pair, for R), group_flags [G] (2*a_cell + b_cell), off [nent+1] (CSR over
// ALL entities), contrib [2*np] (source | group << 40 | cell-cell << 62 | flip << 63;
// cell-cell = both entities of the group's pairs are cells: group_flags == 3).
// Returns G, or -1 if G exceeds gcap or 2^22.
long long omb_fmm_build(const long long* pa, const long long* pb, const long long* pk, long long np, long long nent,
                        long long* group_first, unsigned char* group_flags, long long gcap, long long* off,
                        unsigned long long* contrib) {
  std::unordered_map<long long, long long> first;  // key -> first discovery index
  first.reserve(4096);
  for (long long i = 0; i < np; i++) first.emplace(pk[i], i);
  std::vector<long long> keys;
  keys.reserve(first.size());
  for (auto& kv : first) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  long long G = (long long)keys.size();
  if (G > gcap || G > (1LL << 22)) return -1;
  std::unordered_map<long long, long long> gid;
  gid.reserve(2 * G);
  for (long long g = 0; g < G; g++) {
    gid[keys[g]] = g;
    group_first[g] = first[keys[g]];
    group_flags[g] = (unsigned char)(keys[g] & 3);
  }
  // pairs bucketed by group, stable
  std::vector<long long> pg(np), gstart(G + 1, 0);
  for (long long i = 0; i < np; i++) {
    pg[i] = gid[pk[i]];
    gstart[pg[i] + 1]++;
  }
  for (long long g = 0; g < G; g++) gstart[g + 1] += gstart[g];
  std::vector<long long> order(np), fill(gstart.begin(), gstart.end() - 1);
  for (long long i = 0; i < np; i++) order[fill[pg[i]]++] = i;
  // per-target counts, then the lists in global sequence order
  for (long long e = 0; e <= nent; e++) off[e] = 0;
  for (long long i = 0; i < np; i++) {
    off[pb[i] + 1]++;
    off[pa[i] + 1]++;
  }
  for (long long e = 0; e < nent; e++) off[e + 1] += off[e];
  std::vector<long long> pos(off, off + nent);
  for (long long r = 0; r < np; r++) {
    long long i = order[r];
    unsigned long long g = (unsigned long long)pg[i];
    unsigned long long cc = group_flags[pg[i]] == 3 ? 1ull << 62 : 0ull;
    contrib[pos[pb[i]]++] = (unsigned long long)pa[i] | (g << 40) | cc;
    contrib[pos[pa[i]]++] = (unsigned long long)pb[i] | (g << 40) | cc | (1ull << 63);
  }
  return G;
}

// per-target lists of a theta = 0 traversal, in traversal order (b-side
// before a-side of each pair): off [nent+1], contrib [2*np] (partner | side << 63)
int omb_fmm_build_direct(const long long* pa, const long long* pb, long long np, long long nent, long long* off,
                         unsigned long long* contrib) {
  for (long long e = 0; e <= nent; e++) off[e] = 0;
  for (long long i = 0; i < np; i++) {
    off[pb[i] + 1]++;
    off[pa[i] + 1]++;
  }
  for (long long e = 0; e < nent; e++) off[e + 1] += off[e];
  std::vector<long long> pos(off, off + nent);
  for (long long i = 0; i < np; i++) {
    contrib[pos[pb[i]]++] = (unsigned long long)pa[i];
    contrib[pos[pa[i]]++] = (unsigned long long)pb[i] | (1ull << 63);
  }
  return 0;
}

int omb_fmm_direct(const long long* off, const unsigned long long* contrib, const double* center, const double* M,
                   const long long* cell_base, int nleaf, double* phi, double* gx, double* gy, double* gz,
                   void* stream) {
  long long n = (long long)nleaf * 512;
  if (n == 0) return 0;
  k_fmm_direct<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(off, contrib, center, M, cell_base,
                                                                              nleaf, phi, gx, gy, gz);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_direct", e);
}

int omb_fmm_masses(const double* rho, const long long* cell_base, int nleaf, const double* dx3, double* M,
                   void* stream) {
  long long n = (long long)nleaf * 512 * NC;
  if (n == 0) return 0;
  k_fmm_masses<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(rho, 0, cell_base, nleaf, dx3, M);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_masses", e);
}

int omb_fmm_upward(const long long* parents, int np, const long long* children, const double* center, double* M,
                   void* stream) {
  if (np <= 0) return 0;
  k_fmm_upward<<<(np + 127) / 128, 128, 0, (cudaStream_t)stream>>>(parents, np, children, center, M);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_upward", e);
}

int omb_fmm_m2l(const long long* off, const unsigned long long* contrib, const double* D,
                const unsigned char* cellcell, const double* M, double* L, long long ntarget, const long long* targets,
                const long long* subset, void* stream) {
  if (ntarget <= 0) return 0;
  unsigned nb = (unsigned)((ntarget + 127) / 128);
  k_fmm_m2l<0><<<nb, 128, 0, (cudaStream_t)stream>>>(off, contrib, D, cellcell, M, L, ntarget, targets, subset);
  k_fmm_m2l<1><<<nb, 128, 0, (cudaStream_t)stream>>>(off, contrib, D, cellcell, M, L, ntarget, targets, subset);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_m2l", e);
}

// the monopoles of two mass sets, interleaved (a, b) per entity: the paired pass 0 reads both with
// one 16-byte load (c5g FMM 12.15 -> 11.95 ms per stage, profiles/r02/abf15_m2l_pair_m0x.txt)
__global__ void k_fmm_m0x(const double* __restrict__ Ma, const double* __restrict__ Mb, long long n,
                          double* __restrict__ M0x) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(M0x)[e] = make_double2(Ma[e * NC], Mb[e * NC]);
}

__global__ void k_fmm_m0(const double* __restrict__ M, long long n, double* __restrict__ M0c) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    M0c[e] = M[e * NC];
}

int omb_fmm_m2l_part(int part, const long long* off, const unsigned long long* contrib, const double* D,
                     const unsigned char* cellcell, const double* M, double* L, long long ntarget,
                     const long long* targets, const long long* subset, double* m0, long long nentities,
                     void* stream) {
  if (ntarget <= 0) return 0;
  unsigned nb = (unsigned)((ntarget + 127) / 128);
  if (part == 0 && m0 && nentities > 0) {
    long long b = (nentities + 255) / 256;
    k_fmm_m0<<<(unsigned)(b < 148 * 16 ? b : 148 * 16), 256, 0, (cudaStream_t)stream>>>(M, nentities, m0);
  }
  if (part == 0)
    k_fmm_m2l<0><<<nb, 128, 0, (cudaStream_t)stream>>>(off, contrib, D, cellcell, M, L, ntarget, targets, subset,
                                                       m0);
  else
    k_fmm_m2l<1><<<nb, 128, 0, (cudaStream_t)stream>>>(off, contrib, D, cellcell, M, L, ntarget, targets, subset);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_m2l_part", e);
}

int omb_fmm_m2l0_pair(const long long* off, const unsigned long long* contrib, const double* D,
                      const unsigned char* cellcell, const double* Ma, const double* Mb, double* La, double* Lb,
                      long long ntarget, const long long* targets, const long long* subset, double* m0ab,
                      double* /*unused*/, long long nentities, void* stream) {
  if (ntarget <= 0) return 0;
  if (!m0ab || nentities <= 0) return ferr("omb_fmm_m2l0_pair", cudaErrorInvalidValue);
  long long b = (nentities + 255) / 256;
  unsigned gb = (unsigned)(b < 148 * 16 ? b : 148 * 16);
  k_fmm_m0x<<<gb, 256, 0, (cudaStream_t)stream>>>(Ma, Mb, nentities, m0ab);
  unsigned nb = (unsigned)((ntarget + 127) / 128);
  k_fmm_m2l0_pair<<<nb, 128, 0, (cudaStream_t)stream>>>(off, contrib, D, cellcell, Ma, Mb, La, Lb, ntarget, targets,
                                                        subset, m0ab);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_m2l0_pair", e);
}

int omb_fmm_downward(const long long* parents, int np, const long long* children, const double* center, double* L,
                     void* stream) {
  if (np <= 0) return 0;
  k_fmm_downward<<<(np * 8 + 127) / 128, 128, 0, (cudaStream_t)stream>>>(parents, np, children, center, L);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_downward", e);
}

int omb_fmm_fields(const double* L, const long long* cell_base, int nleaf, double* phi, double* gx, double* gy,
                   double* gz, void* stream) {
  long long n = (long long)nleaf * 512;
  if (n == 0) return 0;
  k_fmm_fields<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(L, cell_base, nleaf, phi, gx, gy, gz);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_fields", e);
}

int omb_fmm_rhodot(const double* U, long long fstride, const OmbLeafInfo* info, int bc, int nleaf,
                   const double* const* halo, int nown, double* out, void* stream) {
  long long n = (long long)nleaf * 512;
  if (n == 0) return 0;
  k_fmm_rhodot<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(U, fstride, (const omb::LeafInfo*)info,
                                                                              bc, nleaf, halo, nown, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ferr("omb_fmm_rhodot", e);
}

}  // extern "C"
