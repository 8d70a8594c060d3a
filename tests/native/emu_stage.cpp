// Host emulation of the fused stage kernel (k_stage in omb_kernels.cu).
// TEST HARNESS: runs the exact phase functions of omb_stage.cuh under g++,
// one simulated thread after another between the same barriers the CUDA
// kernel uses, so the kernel's index bookkeeping can be checked against the
// oracle without a GPU.  Never used by the product.
#include <stdlib.h>
#include <string.h>

#include <vector>

#define OMB_EMU_ASYNC  // cp.async copies land at the issuing thread's wait (see omb_stage.cuh)
#include "../../include/omb200.h"
#include "../../paper_2107_10987_b200/csrc/omb_stage.cuh"

using namespace omb;

// ---- simulated cp.async: per simulated thread, committed groups of pending copies
struct Pending {
  double* dst;
  double val;  // global sources are read-only during a stage: the value at issue is the value copied
};
static int g_tid = 0;
static std::vector<std::vector<Pending>> g_open;                 // [thread] uncommitted copies
static std::vector<std::vector<std::vector<Pending>>> g_groups;  // [thread][group]
void omb::omb_emu_async_copy(double* dst, const double* src) { g_open[g_tid].push_back({dst, *src}); }
void omb::omb_emu_async_commit() {
  g_groups[g_tid].push_back(std::move(g_open[g_tid]));
  g_open[g_tid].clear();
}
// keep = 0: cp.async.wait_all (= commit + wait_group 0); keep = 1: wait_group 1
void omb::omb_emu_async_wait(int keep) {
  if (keep == 0) omb_emu_async_commit();
  auto& G = g_groups[g_tid];
  size_t done = G.size() > (size_t)keep ? G.size() - keep : 0;
  for (size_t k = 0; k < done; k++)
    for (const Pending& p : G[k]) *p.dst = p.val;
  G.erase(G.begin(), G.begin() + done);
}

// order in which the simulated threads run inside one barrier interval:
// 0 ascending, 1 descending, 2 a stride-97 permutation.  A result that depends
// on the order is a shared-memory race between threads of one interval.
static int g_order = 0;
extern "C" void emu_set_order(int mode) { g_order = mode; }

extern "C" int emu_stage(const OmbStageDesc* d, int nthr) {
  if (nthr < 256) return -1;  // the phase layout: >= 128 threads; two rounds of <= 500 items: >= 250
  StageArgs A;
  A.ucur = d->ucur; A.u0 = d->u0; A.unext = d->unext; A.grav = d->grav; A.fstride = d->fstride;
  A.info = (const LeafInfo*)d->info; A.run_off = d->run_off; A.run_leaf = d->run_leaf; A.dt = d->dt;
  A.a = d->a; A.b = d->b; A.gamma = d->gamma; A.gm1 = d->gm1; A.inv_gm1 = 1.0 / d->gm1; A.eta = d->eta; A.inv_gamma = d->inv_gamma;
  A.omega = d->omega; A.floor_rho = d->floor_rho; A.floor_tau = d->floor_tau; A.floor_vmax = d->floor_vmax;
  A.bc = d->bc; A.new_mode = d->new_mode; A.quad = d->new_mode && !d->override_center; A.contact = d->contact;
  A.amax_bits = d->amax_bits; A.fallback = d->fallback; A.flux = d->flux; A.halo = d->halo; A.nown = d->nown;
  A.scalar = d->scalar; A.s_u0 = d->s_u0; A.s_next = d->s_next;
  std::vector<double> S(Smem::TOTAL);
  std::vector<int> order(nthr);
  for (int k = 0; k < nthr; k++) order[k] = g_order == 0 ? k : (g_order == 1 ? nthr - 1 - k : (int)((97LL * k) % nthr));
  g_open.assign(nthr, {});
  g_groups.assign(nthr, {});
  for (int run = 0; run < d->nruns; run++) {
    std::fill(S.begin(), S.end(), NAN);  // catch reads of never-written shared memory
    std::vector<Stage> st(nthr);
    std::vector<Hold> h(nthr);
    int off = d->run_off[run];
    for (int t = 0; t < nthr; t++) {
      st[t].S = S.data(); st[t].A = A; st[t].run = run;
      st[t].R = d->run_off[run + 1] - off; st[t].leaves = d->run_leaf + off;
      st[t].amax = 0.0; st[t].fb = 0;
    }
    int R = st[0].R;
#define ALL(stmt) for (int k_ = 0; k_ < nthr; k_++) { int t = order[k_]; g_tid = t; Stage& s = st[t]; (void)s; stmt; }
    ALL(s.bind_run_info(); s.stage_run_info(t, nthr); s.load_items(t));
    // the phase sequence of k_stage (omb_kernels.cu), one ALL() per barrier interval,
    // with its cp.async commits and waits at the same points
    ALL(for (int X = 0; X < 4; X++) s.prefetch_plane(X, t, nthr, Smem::RAW + X * NF * PL);
        s.prefetch_plane(4, t, nthr); async_commit(); async_wait_all());
    for (int X = 0; X < 4; X++) ALL(s.convert_plane(X, t, nthr, Smem::RAW + X * NF * PL));
    const int ngroups = A.new_mode ? 2 : 1;
    const int T6 = NF * NYF - (512 - PL);
    for (int X = 2; X < 8 * R + 4; X++) {
      ALL(s.set_plane(X));
      ALL(if (X + 2 < 8 * R + 6) s.convert_plane(X + 2, t, nthr);
          if (X - 1 >= 3) { s.set_plane(X - 1); s.faces_yz(t, nthr, PL); s.set_plane(X); }
          if (s.interior(X - 2) && t >= T6 && t < T6 + NFACEX) s.prefetch_update(X - 2, t - T6, NFACEX);
          async_commit());
      const bool p6 = X >= 3 && st[0].interior(X - 2);
      for (int g = 0; g < ngroups; g++) {
        ALL(if (g == 0) { if (X + 3 < 8 * R + 6) s.prefetch_plane(X + 3, t, nthr); async_commit(); }
            s.boundary_lines(g, t, nthr, h[t]);
            if (g == 0) async_wait_prev());
        ALL(s.store_hi(h[t]);
            if (X >= 3) { if (g == 0) s.combine_A(t, nthr); else if (A.quad) s.combine_B(t, nthr); }
            if (g == 0 && p6 && t >= nthr - NFACEX) { s.set_plane(X - 1); s.update_plane_a(t - (nthr - NFACEX), NFACEX); s.set_plane(X); });
      }
      ALL(s.inplane_lines(t, nthr);
          if (p6 && t >= nthr - NFACEX) { s.set_plane(X - 1); s.update_plane_b(t - (nthr - NFACEX), NFACEX); s.set_plane(X); });
      ALL(if (s.interior(X)) s.inplane_fluxes(t, nthr); async_wait_all());
    }
    ALL(s.set_plane(8 * R + 3); s.faces_yz(t, nthr); if (t < NFACEX) s.prefetch_update(8 * R + 2, t, NFACEX);
        async_commit(); async_wait_all());
    ALL(s.set_plane(8 * R + 3); s.update_plane(t, nthr));
    for (int t = 0; t < nthr; t++)
      if (!g_open[t].empty() || !g_groups[t].empty()) return -3;  // a copy never waited for
    double m = 0.0;
    long long f = 0;
    for (int t = 0; t < nthr; t++) {
      m = st[t].amax > m ? st[t].amax : m;
      f += st[t].fb;
    }
    unsigned long long bits;
    memcpy(&bits, &m, 8);
    if (bits > *A.amax_bits) *A.amax_bits = bits;
    *A.fallback += f;
  }
  return 0;
}

extern "C" int emu_gather(const double* U, long long fstride, const OmbLeafInfo* info, int leaf, int bc, double* out) {
  for (int c = 0; c < M * M * M; c++) {
    double u[NF];
    gather_cell(U, fstride, ((const LeafInfo*)info)[leaf], bc, c / (M * M), (c / M) % M, c % M, u);
    for (int v = 0; v < NF; v++) out[v * M * M * M + c] = u[v];
  }
  return 0;
}

extern "C" double emu_speed(const double* u6, double gamma, double gm1, double eta) {
  return speed_cell(u6, gamma, gm1, eta);
}

extern "C" int emu_amr_ghosts(const OmbAmrDesc* d) {
  for (int task = 0; task < d->ntasks; task++) {
    const int* t = d->tasks + task * 16;
    int nc = amr_block_cells(t);
    for (int i = 0; i < nc; i++) {
      int b[3], vcell;
      amr_decode(t, i, b, vcell);
      double out[NF];
      for (int v = 0; v < NF; v++) out[v] = amr_cell(d->u, d->fstride, t, v, b);
      for (int v = 0; v < NF; v++) d->u[v * d->fstride + (long long)t[4] * 512 + vcell] = out[v];
    }
  }
  return 0;
}

extern "C" int emu_reflux_update(const OmbRefluxDesc* r) {
  const OmbStageDesc* d = &r->stage;
  StageArgs A;
  A.ucur = d->ucur; A.u0 = d->u0; A.unext = d->unext; A.grav = d->grav; A.fstride = d->fstride;
  A.info = (const LeafInfo*)d->info; A.dt = d->dt; A.a = d->a; A.b = d->b; A.gamma = d->gamma; A.gm1 = d->gm1;
  A.inv_gm1 = 1.0 / d->gm1; A.eta = d->eta; A.inv_gamma = d->inv_gamma; A.omega = d->omega;
  A.floor_rho = d->floor_rho; A.floor_tau = d->floor_tau; A.floor_vmax = d->floor_vmax; A.flux = d->flux; A.halo = d->halo; A.nown = d->nown;
  A.scalar = d->scalar; A.s_u0 = d->s_u0; A.s_next = d->s_next;
  std::vector<double> F(FLUX_SLOT);
  for (int i = 0; i < r->nleaves; i++) {
    int leaf = r->leaf[i];
    const double* src = A.flux + (long long)A.info[leaf].slot * FLUX_SLOT;
    for (int j = 0; j < FLUX_SLOT; j++) F[j] = src[j];
    for (int q = r->off[i]; q < r->off[i + 1]; q++) reflux_apply(F.data(), A.flux, r->tasks + q * 6, 0, 1);
    update_leaf(A, leaf, F.data(), 0, 1);
  }
  return 0;
}

// passive-scalar pass input (omb_scalar_input): (rho, sx, sy, sz, p, X)
extern "C" int emu_scalar_input(const double* U, long long fstride, int n_all, const double* x, int n_x, double gamma,
                                double gm1, double eta, double* dst) {
  for (long long c = 0; c < (long long)n_all * 512; c++) {
    double u[NF], w[NF];
    for (int v = 0; v < NF; v++) u[v] = U[v * fstride + c];
    prim_cell(u, gamma, gm1, eta, w);
    for (int v = 0; v < 4; v++) dst[v * fstride + c] = u[v];
    dst[4 * fstride + c] = w[4];
    if (x != nullptr && c < (long long)n_x * 512) dst[5 * fstride + c] = x[c];
  }
  return 0;
}
