// Native collection of a finished device factorization (host C++).
//
// After the factorization program has run, the only data the host needs from
// the device are the per-interface events (rank k_c, fine count, k_stop).
// This file replays the live offsets (the reference keeps dofs[n_fine:],
// factorize.py:187-190) and produces, in the reference's operator order
// (factorize.py:309-366):
//   * an operator table + neighbour-segment table (payload windows inside the
//     device block pool / factor buffer) from which the Python host builds
//     the Elimination / Scaling / Orthogonal / ErrorCorrection objects lazily;
//   * the permutation, per-interface diagnostics and per-level summaries;
//   * the payload windows whose nonzeros the device counts (nnz_factor);
//   * the structured apply plan (phases of GEMV tiles + ordered scatters in
//     the cluster-contiguous numbering, see apply.cu / fastplan.py).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstdint>
#include <thread>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "planner.h"

namespace {

struct Task {
  int64_t M, ld, rows, cols, trans, rot, in_kind, in_ptr;
  int64_t out_start;   // permuted start of the outputs, or -1: index list
  int64_t out_idx;     // offset into the index store when out_start < 0
  int64_t mode;
  int64_t flag_off = -1;   // elimination panels: first word of the nonzero-row bits
  int lower = 0;           // explicit lower-triangular inverses: zero tiles skipped
};

struct PhaseImage {
  std::vector<int64_t> rows, tiles, chunks, contrib;
  // dataflow schedule inputs: per item its input and output cluster, per
  // chunk its output cluster (cluster-contiguous numbering; ncl = the final
  // block's index list)
  std::vector<int32_t> item_src, item_dst, chunk_dst;
  int64_t pos = 0;
  bool overflow = false;
};

struct Collected {
  std::vector<int64_t> ops;    // 16 per op
  std::vector<int64_t> segs;   // 8 per segment
  std::vector<int64_t> perm;
  std::vector<int64_t> diag;   // 10 per sparsified interface
  std::vector<int64_t> lsum;   // 4 per level: level, n_interiors, interior dofs, skipped
  std::vector<int64_t> views;  // 4 per payload window: base(0 pool,1 fac) | off, ld, rows, cols
  std::vector<int64_t> fine;   // 8 per (interface, neighbour): the fine rows Q_f^T W
                               // {diag row, w, pool off, ld, rows, cols, trans, 0}
  int64_t final_total = 0;
  int64_t critical_steps = 0;  // sum over waves of the largest k_stop (RRQR critical path)
  // apply
  std::vector<std::vector<Task>> fph, bph;
  std::vector<int64_t> fidx;   // permuted indices of the final block
  std::vector<PhaseImage> imgs;  // compiled phases (concatenated by spand_collect_apply_get)
  std::vector<int64_t> img_at;   // image offset of each compiled phase (-1: empty)
  int64_t img_len = 0;
  std::vector<int64_t> phases; // 10 per phase (see spand_collect_apply_get)
  int64_t scratch_len = 0;
  // elimination panels scanned for nonzero rows before the image compiles:
  // {pool offset, ld, rows, cols, first bit word}
  std::vector<int64_t> flag_panels;
  int64_t flag_words = 0;
  // dataflow schedule (spand_collect_dataflow)
  std::vector<int64_t> cstart;             // ncl + 1
  std::vector<int32_t> fin;                // clusters of the final block
  std::vector<int64_t> df_units, df_deps, df_phase;
  int64_t df_nctr = 0, df_scratch = 0;
};

}  // namespace

extern "C" {

void* spand_collect_create(void* plan, const int64_t* events, int scheme) {
  const spand::Plan& pv = *static_cast<spand::Plan*>(plan);
  Collected* C = new Collected();
  const int ncl = pv.ncl;
  std::vector<int64_t> off(ncl, 0), cstart(ncl + 1, 0);
  for (int c = 0; c < ncl; ++c) cstart[c + 1] = cstart[c] + pv.m0[c];
  C->cstart = cstart;
  C->fin.assign(pv.fin.begin(), pv.fin.end());
  auto live = [&](int c) { return pv.m0[c] - off[c]; };
  auto pst = [&](int c) { return cstart[c] + off[c]; };
  // apply phase numbering (forward per level: [G-T][G-A]([D]([Q-T][E-A])*waves))
  const int nlev = (int)pv.lv.size();
  std::vector<int64_t> cnt(nlev), fbase(nlev + 1, 0), bbase(nlev);
  for (int li = 0; li < nlev; ++li) {
    const spand::Level& L = pv.lv[li];
    cnt[li] = 2 + (L.skipped ? 0 : 1 + 2 * L.nwaves);
    fbase[li + 1] = fbase[li] + cnt[li];
  }
  const int64_t nph = fbase[nlev] + 1;
  for (int li = 0; li < nlev; ++li) {
    int64_t s = 1;
    for (int lj = li + 1; lj < nlev; ++lj) s += cnt[lj];
    bbase[li] = s;
  }
  C->fph.assign(nph, {});
  C->bph.assign(nph, {});
  {
    size_t nin = 0, nint = 0, nact = 0;
    for (const spand::Level& L : pv.lv) {
      nin += L.inb_blk.size();
      nint += L.interiors.size();
      nact += L.active.size();
    }
    C->segs.reserve(8 * nin + 8 * 16 * nact);
    C->views.reserve(4 * (nin + nint + 2 * nact) + 64 * nact);
    C->ops.reserve(16 * (nint + 3 * nact + 1));
    C->perm.reserve(pv.dofs.size());
  }
  auto add = [&](std::vector<Task>& ph, int64_t M, int64_t ld, int64_t rows, int64_t cols,
                 int vtrans, int optrans, int64_t rot, int64_t in_start, int64_t out_start,
                 int64_t mode) {
    Task t;
    t.M = M;
    t.ld = ld;
    t.rows = rows;
    t.cols = cols;
    t.trans = (vtrans != optrans) ? 1 : 0;
    t.rot = rot;
    t.in_kind = 1;
    t.in_ptr = in_start;        // permuted index; turned into an address at build
    t.out_start = out_start;
    t.out_idx = 0;
    t.mode = mode;
    ph.push_back(t);
  };
  auto T0 = std::chrono::steady_clock::now();
  double tint = 0, tres = 0, tsp = 0;
  for (int li = 0; li < nlev; ++li) {
    auto Ta = std::chrono::steady_clock::now();
    const spand::Level& L = pv.lv[li];
    const int64_t fb = fbase[li], bb = bbase[li];
    const int64_t nw = L.skipped ? 0 : L.nwaves;
    const int64_t gfT = fb, gfA = fb + 1;
    const int64_t gbA = bb + (L.skipped ? 0 : 2 * nw + 1), gbT = bb + (L.skipped ? 1 : 2 * nw + 2);
    int64_t nint = 0, ndofs = 0;
    C->fph[gfA].reserve(L.inb_blk.size());
    C->bph[gbA].reserve(L.inb_blk.size());
    C->fph[gfT].reserve(L.interiors.size());
    C->bph[gbT].reserve(L.interiors.size());
    for (int k = 0; k < (int)L.interiors.size(); ++k) {
      const int s = L.interiors[k];
      const int64_t ns = live(s);
      if (ns == 0) continue;
      ++nint;
      ndofs += ns;
      const int64_t m0s = pv.m0[s];
      const int64_t lower = pv.boff[pv.block(s, s)] + off[s] + off[s] * m0s;
      const int64_t linv = pv.elim_linv[s] + off[s] + off[s] * m0s;
      const int64_t sb = (int64_t)C->segs.size() / 8;
      const int* blk = L.inb_blk.data() + L.inb_ptr[k];   // block(w, s), from the planner
      for (size_t u = 0; u < L.inbrs[k].size(); ++u) {
        const int w = L.inbrs[k][u];
        const int64_t lw = live(w);
        if (lw == 0) continue;
        const int64_t a = pv.boff[blk[u]] + off[w] + off[s] * pv.m0[w];
        C->segs.insert(C->segs.end(), {w, off[w], lw, a, pv.m0[w], lw, ns, 0});
        C->views.insert(C->views.end(), {a, pv.m0[w], lw, ns});
        add(C->fph[gfA], a, pv.m0[w], lw, ns, 0, 0, 0, pst(s), pst(w), 1);
        add(C->bph[gbA], a, pv.m0[w], lw, ns, 0, 1, 0, pst(w), pst(s), 1);
        // the panel's rows of w not coupled to s are zero (the reference
        // stores them densely): their nonzero-row bits select row runs
        C->fph[gfA].back().flag_off = C->bph[gbA].back().flag_off = C->flag_words;
        C->flag_panels.insert(C->flag_panels.end(), {a, pv.m0[w], lw, ns, C->flag_words});
        C->flag_words += (lw + 31) / 32;
      }
      const int64_t se = (int64_t)C->segs.size() / 8;
      C->ops.insert(C->ops.end(), {0, s, li, 0, off[s], ns, 0, lower, m0s, linv, -1, 0, sb, se, 0, 0});
      C->views.insert(C->views.end(), {lower, m0s, ns, ns});
      add(C->fph[gfT], linv | (int64_t(1) << 62), m0s, ns, ns, 0, 0, 0, pst(s), pst(s), 0);
      add(C->bph[gbT], linv | (int64_t(1) << 62), m0s, ns, ns, 0, 1, 0, pst(s), pst(s), 0);
      C->fph[gfT].back().lower = C->bph[gbT].back().lower = 1;
      for (int64_t i = 0; i < ns; ++i) C->perm.push_back(pv.dofs[pv.dptr[s] + off[s] + i]);
    }
    C->lsum.insert(C->lsum.end(), {L.level, nint, ndofs, L.skipped});
    auto Tb = std::chrono::steady_clock::now();
    tint += std::chrono::duration<double>(Tb - Ta).count();
    if (L.skipped) continue;
    // rescales
    for (int k = 0; k < (int)L.active.size(); ++k) {
      const int p = L.active[k];
      const int64_t mp = live(p);
      if (mp == 0) continue;
      const int64_t m0p = pv.m0[p];
      const int64_t lo = L.l_off[k] + off[p] + off[p] * m0p;
      const int64_t li2 = L.linv_off[k] + off[p] + off[p] * m0p;
      C->ops.insert(C->ops.end(), {1, p, li, 0, off[p], mp, 0, lo, m0p, li2, -1, 0, 0, 0, 1, 0});
      C->views.insert(C->views.end(), {lo | (int64_t(1) << 62), m0p, mp, mp});
      add(C->fph[fb + 2], li2 | (int64_t(1) << 62), m0p, mp, mp, 0, 0, 0, pst(p), pst(p), 0);
      add(C->bph[bb + 2 * nw], li2 | (int64_t(1) << 62), m0p, mp, mp, 0, 1, 0, pst(p), pst(p), 0);
      C->fph[fb + 2].back().lower = C->bph[bb + 2 * nw].back().lower = 1;
    }
    // RRQR critical path: waves run one after the other, panels of a wave
    // concurrently
    {
      std::vector<int64_t> wmax(L.nwaves, 0);
      for (int k = 0; k < (int)L.active.size(); ++k)
        wmax[L.wave[k]] = std::max(wmax[L.wave[k]], events[12 * L.slot[k] + 3]);
      for (int64_t v : wmax) C->critical_steps += v;
    }
    auto Tc = std::chrono::steady_clock::now();
    tres += std::chrono::duration<double>(Tc - Tb).count();
    // sparsifications in ascending id order
    for (int k = 0; k < (int)L.active.size(); ++k) {
      const int p = L.active[k];
      const int64_t mp = live(p);
      if (mp == 0) continue;
      const int64_t* e = events + 12 * L.slot[k];
      const int64_t k_stop = e[3], k_c = e[4], rf2 = e[5], n_fine = e[6];
      const int wv = L.wave[k];
      const int64_t qfT = fb + 3 + 2 * wv, efA = fb + 4 + 2 * wv;
      const int64_t back = bb + 2 * (nw - 1 - wv), ebA = back, qbT = back + 1;
      const int64_t qo = L.q_off[k];
      C->ops.insert(C->ops.end(), {2, p, li, wv, off[p], mp, 0, 0, mp, 0, qo, k_c, 0, 0, 0, 0});
      C->views.insert(C->views.end(), {qo | (int64_t(1) << 62), mp, mp, mp});
      add(C->fph[qfT], qo | (int64_t(1) << 62), mp, mp, mp, 0, 1, k_c, pst(p), pst(p), 0);
      add(C->bph[qbT], qo | (int64_t(1) << 62), mp, mp, mp, 0, 0, k_c, pst(p), pst(p), 0);
      int64_t ncorr = 0;
      if (scheme == 1) ncorr = n_fine;
      else if (scheme == 2) ncorr = k_stop - k_c;
      int64_t ntot = 0;
      for (int w : L.anbrs[k]) ntot += live(w);
      if (ncorr && ntot) {
        const int64_t sb = (int64_t)C->segs.size() / 8;
        for (int w : L.anbrs[k]) {
          const int64_t lw = live(w);
          if (lw == 0) continue;
          if (w > p) {
            const int64_t a = pv.boff[pv.block(p, w)] + off[p] + off[w] * pv.m0[p];
            C->segs.insert(C->segs.end(), {w, off[w], lw, a, pv.m0[p], ncorr, lw, 0});
            C->views.insert(C->views.end(), {a, pv.m0[p], ncorr, lw});
            add(C->fph[efA], a, pv.m0[p], ncorr, lw, 0, 1, 0, pst(p), pst(w), 1);
            add(C->bph[ebA], a, pv.m0[p], ncorr, lw, 0, 0, 0, pst(w), pst(p), 1);
          } else {
            const int64_t a = pv.boff[pv.block(w, p)] + off[w] + off[p] * pv.m0[w];
            C->segs.insert(C->segs.end(), {w, off[w], lw, a, pv.m0[w], lw, ncorr, 1});
            C->views.insert(C->views.end(), {a, pv.m0[w], lw, ncorr});
            add(C->fph[efA], a, pv.m0[w], lw, ncorr, 1, 1, 0, pst(p), pst(w), 1);
            add(C->bph[ebA], a, pv.m0[w], lw, ncorr, 1, 0, 0, pst(w), pst(p), 1);
          }
        }
        const int64_t se = (int64_t)C->segs.size() / 8;
        C->ops.insert(C->ops.end(), {3, p, li, wv, off[p], ncorr, 0, 0, 0, 0, -1, 0, sb, se, 0, 0});
      }
      for (int64_t i = 0; i < n_fine; ++i) C->perm.push_back(pv.dofs[pv.dptr[p] + off[p] + i]);
      // fine rows of every neighbour block (all schemes; filled by the RRQR
      // only for the correction rows unless local errors are requested)
      if (n_fine) {
        const int64_t drow = (int64_t)C->diag.size() / 10;
        for (int w : L.anbrs[k]) {
          const int64_t lw = live(w);
          if (lw == 0) continue;
          if (w > p) {
            const int64_t a = pv.boff[pv.block(p, w)] + off[p] + off[w] * pv.m0[p];
            C->fine.insert(C->fine.end(), {drow, w, a, pv.m0[p], n_fine, lw, 0, 0});
          } else {
            const int64_t a = pv.boff[pv.block(w, p)] + off[w] + off[p] * pv.m0[w];
            C->fine.insert(C->fine.end(), {drow, w, a, pv.m0[w], lw, n_fine, 1, 0});
          }
        }
      }
      C->diag.insert(C->diag.end(), {li, p, mp, k_c, rf2, e[7], e[8], k_stop, e[2], 0});
      off[p] += n_fine;
    }
    tsp += std::chrono::duration<double>(std::chrono::steady_clock::now() - Tc).count();
  }
  if (getenv("SPAND_COLLECT_TIMES"))
    fprintf(stderr, "collect: interiors %.1f ms rescale %.1f sparsify %.1f total %.1f\n", 1e3 * tint,
            1e3 * tres, 1e3 * tsp,
            1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - T0).count());
  // final dense block
  int64_t total = 0;
  for (int c : pv.fin) total += live(c);
  C->final_total = total;
  if (total) {
    const int64_t foff = pv.fcap - total;
    const int64_t lower = pv.f_off + foff + foff * pv.fcap;
    const int64_t linv = pv.flinv_off + foff + foff * pv.fcap;
    C->ops.insert(C->ops.end(), {4, -1, nlev, 0, 0, total, 0, lower, pv.fcap, linv, -1, 0, 0, 0, 1, 0});
    C->views.insert(C->views.end(), {lower | (int64_t(1) << 62), pv.fcap, total, total});
    for (int c : pv.fin) {
      for (int64_t i = 0; i < live(c); ++i) {
        C->perm.push_back(pv.dofs[pv.dptr[c] + off[c] + i]);
        C->fidx.push_back(pst(c) + i);
      }
    }
    Task tf;
    tf.M = linv | (int64_t(1) << 62);
    tf.ld = pv.fcap;
    tf.rows = tf.cols = total;
    tf.trans = 0;
    tf.rot = 0;
    tf.in_kind = 0;
    tf.in_ptr = 0;
    tf.out_start = -1;
    tf.out_idx = 0;
    tf.mode = 0;
    tf.lower = 1;
    C->fph[nph - 1].push_back(tf);
    tf.trans = 1;
    C->bph[0].push_back(tf);
  }
  return C;
}

void spand_collect_destroy(void* h) { delete static_cast<Collected*>(h); }

// out[8]: nops, nsegs, nperm, ndiag, nlsum, nviews, final_total, nfine
int spand_collect_sizes(void* h, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  out[0] = (int64_t)C->ops.size() / 16;
  out[1] = (int64_t)C->segs.size() / 8;
  out[2] = (int64_t)C->perm.size();
  out[3] = (int64_t)C->diag.size() / 10;
  out[4] = (int64_t)C->lsum.size() / 4;
  out[5] = (int64_t)C->views.size() / 4;
  out[6] = C->final_total;
  out[7] = (int64_t)C->fine.size() / 8;
  return 0;
}

// out[1]: RRQR critical-path steps (sum over waves of the largest k_stop)
int spand_collect_stats(void* h, int64_t* out) {
  out[0] = static_cast<Collected*>(h)->critical_steps;
  return 0;
}

// fine-row views of the sparsified interfaces (8 int64 each, see Collected)
int spand_collect_fine(void* h, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  if (!C->fine.empty()) std::memcpy(out, C->fine.data(), C->fine.size() * sizeof(int64_t));
  return 0;
}

int spand_collect_get(void* h, int64_t* ops, int64_t* segs, int64_t* perm, int64_t* diag,
                      int64_t* lsum, int64_t* views, int64_t* fidx) {
  Collected* C = static_cast<Collected*>(h);
  auto cp = [](int64_t* dst, const std::vector<int64_t>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int64_t));
  };
  cp(ops, C->ops);
  cp(segs, C->segs);
  cp(perm, C->perm);
  cp(diag, C->diag);
  cp(lsum, C->lsum);
  cp(views, C->views);
  cp(fidx, C->fidx);
  return 0;
}

// ---- structured apply plan ------------------------------------------------
// Device image (int64): per phase {task rows (8 each), tile rows (8 each,
// apply.cu layout), run chunks (8 each, spand_apply_runs), contribution
// bases}.  Every task writes one whole destination run (a live cluster range
// in the cluster-contiguous numbering, or the final block's index list), so
// the ordered accumulation is described per run, not per element: tasks that
// hit the same run contribute their scratch blocks in task order.
// Addresses: payload windows pool_base/fac_base (bit 62 of the window offset
// selects the factor buffer), inputs xbuf + 8 * permuted index.

static void compile_phase(PhaseImage& P, const std::vector<Task>& ph, int64_t pool_base,
                          int64_t fac_base, int64_t xbuf, int64_t idx_addr, const uint32_t* bits,
                          const std::vector<int64_t>& cstart) {
  const int ncl = (int)cstart.size() - 1;
  auto cluster_of = [&](int64_t x) {
    return (int32_t)(std::upper_bound(cstart.begin(), cstart.end(), x) - cstart.begin() - 1);
  };
  constexpr int64_t RUN = 64;
  constexpr int64_t GAP = 8;   // zero-row gaps shorter than this stay inside a row run
  // warp work items of ~32 KB of payload (apply.cu gemv_items_kernel):
  //   trans 0: kc <= 64 columns x oc <= 128 rows (64 rows for wide tasks)
  //   trans 1: oc <= 4 columns x kc <= 1024 rows
  std::vector<int64_t>& rows = P.rows;
  std::vector<int64_t>& tiles = P.tiles;
  std::vector<int64_t>& chunks = P.chunks;
  std::vector<int64_t>& contrib = P.contrib;
  // A piece is the scratch block one k-tile of one (sub)task produces for a
  // destination range [start, start + len): absolute x positions (key 0) or
  // positions in the final block's index list (key 1).  Pieces of one phase
  // may overlap (many operators update one interface); the destination is
  // cut into segments covered by a fixed set of pieces, summed in task order.
  struct Piece { int64_t key, start, len, part, mode, order, grp; };
  std::vector<Piece> pieces;
  int64_t pos = 0, order = 0;
  // first row >= i (< n) whose bit equals `want` (word-level scans)
  auto next_bit = [&](int64_t off, int64_t i, int64_t n, bool want) -> int64_t {
    while (i < n) {
      uint32_t w = bits[off + (i >> 5)];
      if (!want) w = ~w;
      w &= ~0u << (i & 31);
      if (w) {
        const int64_t r = (i & ~int64_t(31)) + __builtin_ctz(w);
        return r < n ? r : n;
      }
      i = (i & ~int64_t(31)) + 32;
    }
    return n;
  };
  // sub-tasks: elimination panels split into runs of nonzero rows
  // Results must not depend on the bits (the first image of a factor has
  // none, the compressed one replaces it later): items and k-tiles keep the
  // uncompressed shapes, transposed tasks only drop all-zero k-tiles, and the
  // accumulation sums each output's parts in order (apply.cu runs_kernel),
  // so a dropped part -- an exact zero -- changes nothing.
  struct Sub { const Task* t; int64_t ra, rb; };
  std::vector<Sub> subs;
  int64_t payload = 0;
  for (const Task& t : ph) {
    if ((t.trans ? t.cols : t.rows) == 0) continue;
    payload += t.rows * t.cols * 8 / (t.lower ? 2 : 1);
    if (t.flag_off >= 0 && bits && !t.trans) {
      const int64_t nr = t.rows;
      int64_t i = next_bit(t.flag_off, 0, nr, true);
      while (i < nr) {
        // extend over runs of nonzero rows and zero gaps of <= GAP rows
        int64_t last = next_bit(t.flag_off, i, nr, false) - 1;
        for (;;) {
          const int64_t nx = next_bit(t.flag_off, last + 1, nr, true);
          if (nx >= nr || nx - last > GAP) break;
          last = next_bit(t.flag_off, nx, nr, false) - 1;
        }
        subs.push_back({&t, i, last + 1});
        i = next_bit(t.flag_off, last + 1, nr, true);
      }
    } else {
      subs.push_back({&t, 0, t.rows});
    }
  }
  // item size: ~32 KB, smaller when the phase is small, so that every phase
  // offers about one item per resident warp (148 SMs x 32 warps)
  const int64_t isz = std::max<int64_t>(4096, std::min<int64_t>(32768, payload / (148 * 32)));
  for (const Sub& sb : subs) {
    const Task& t = *sb.t;
    const int64_t srows = sb.rb - sb.ra;
    const int64_t nout = t.trans ? t.cols : srows;
    const int64_t nk = t.trans ? srows : t.cols;
    if (nout == 0 || nk == 0) continue;
    if (nout >= (int64_t(1) << 20) || nk >= (int64_t(1) << 17)) P.overflow = true;
    const bool in_fac = (t.M >> 62) & 1;
    const int64_t moff = (t.M & ((int64_t(1) << 62) - 1)) + sb.ra;
    const int64_t maddr = (in_fac ? fac_base : pool_base) + 8 * moff;
    const int64_t in_ptr = t.in_ptr + (t.trans ? sb.ra : 0);
    const int64_t inp = t.in_kind == 1 ? xbuf + 8 * in_ptr : idx_addr;
    const int64_t tid = (int64_t)rows.size() / 8;
    rows.insert(rows.end(), {maddr, t.ld, srows, t.cols, t.trans, t.rot, t.in_kind, inp});
    int64_t TO, TK;
    if (t.trans) {
      TO = 4;
      TK = std::max<int64_t>(64, std::min<int64_t>(1024, isz / (8 * TO) / 32 * 32));
    } else {
      TO = nk <= 32 ? 128 : 64;
      TK = std::max<int64_t>(8, std::min<int64_t>(64, isz / (8 * TO)));
    }
    const int64_t out0 = t.out_start >= 0 ? t.out_start + (t.trans ? 0 : sb.ra) : 0;
    const int64_t key = t.out_start >= 0 ? 0 : 1;
    const int32_t src = t.in_kind == 1 ? cluster_of(in_ptr) : ncl;
    const int32_t dst = key ? ncl : cluster_of(out0);
    const int64_t nkt = std::max<int64_t>(1, (nk + TK - 1) / TK);
    for (int64_t kb = 0; kb < nkt; ++kb) {
      const int64_t k0 = kb * TK;
      const int64_t kc = std::max<int64_t>(0, std::min(TK, nk - k0));
      // transposed elimination panel: a k-tile of all-zero rows adds nothing
      if (t.trans && t.flag_off >= 0 && bits && kc > 0 &&
          next_bit(t.flag_off, sb.ra + k0, sb.ra + k0 + kc, true) >= sb.ra + k0 + kc)
        continue;
      // the outputs this k-tile touches: all, or the lower-triangular part
      int64_t lo = 0, hi = nout;
      if (t.lower) {
        if (!t.trans) lo = std::min(nout, k0);          // rows >= the tile's first column
        else hi = std::min(nout, k0 + kc);              // columns <= the tile's last row
      }
      if (lo >= hi) continue;
      const int64_t part = pos;
      for (int64_t ob = lo; ob < hi; ob += TO) {
        const int64_t oc = std::min(TO, hi - ob);
        // packed item (apply.cu): task | ob | oc, out_off | kb | kc
        tiles.insert(tiles.end(), {(tid << 32) | (ob << 12) | oc,
                                   ((part + ob - lo) << 28) | (k0 << 11) | kc});
        P.item_src.push_back(src);
        P.item_dst.push_back(dst);
      }
      // summation group of the part: fixed by (task, k-tile), the same in
      // the compressed and uncompressed images
      pieces.push_back({key, out0 + lo, hi - lo, part, t.mode, order++,
                        ((int64_t)(&t - ph.data()) + kb) & 3});
      pos += hi - lo;
    }
  }
  if (rows.empty()) return;
  // packed-item field limits (apply.cu): ob < 2^20, inner offset < 2^17,
  // scratch offset < 2^35
  if (pos >= (int64_t(1) << 35)) P.overflow = true;
  // segments: the destination (per key) is cut where pieces begin or end;
  // every segment has a fixed set of covering pieces, summed in task order
  // (contribution = part - start: output e of the segment reads
  // scratch[contrib + e]); chunks of <= RUN outputs of one segment
  std::sort(pieces.begin(), pieces.end(), [](const Piece& x, const Piece& y) {
    return x.key != y.key ? x.key < y.key : (x.start != y.start ? x.start < y.start : x.order < y.order);
  });
  size_t i0 = 0;
  std::vector<int64_t> cuts;
  std::vector<size_t> active;
  while (i0 < pieces.size()) {
    size_t i1 = i0;
    while (i1 < pieces.size() && pieces[i1].key == pieces[i0].key) ++i1;
    const int64_t key = pieces[i0].key;
    cuts.clear();
    for (size_t q = i0; q < i1; ++q) {
      cuts.push_back(pieces[q].start);
      cuts.push_back(pieces[q].start + pieces[q].len);
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    active.clear();
    size_t nxt = i0;
    int64_t cb = -1, ce = -1, splits = 0;   // the current covering list (reused while unchanged)
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
      const int64_t a = cuts[c], b = cuts[c + 1];
      size_t w = 0;
      bool changed = false;
      for (size_t q : active) {
        if (pieces[q].start + pieces[q].len > a) active[w++] = q;
        else changed = true;
      }
      active.resize(w);
      while (nxt < i1 && pieces[nxt].start == a) {
        active.push_back(nxt++);
        changed = true;
      }
      if (active.empty()) continue;
      if (changed || cb < 0) {
        // by summation group, task order within a group; split points of
        // groups 1-3 packed (16 bits each, relative to cb) in the chunk row
        std::sort(active.begin(), active.end(), [&](size_t x, size_t y) {
          return pieces[x].grp != pieces[y].grp ? pieces[x].grp < pieces[y].grp
                                                : pieces[x].order < pieces[y].order;
        });
        cb = (int64_t)contrib.size();
        int64_t cnt[4] = {0, 0, 0, 0};
        for (size_t q : active) {
          contrib.push_back(pieces[q].part - pieces[q].start);
          ++cnt[pieces[q].grp];
        }
        ce = (int64_t)contrib.size();
        if (ce - cb >= 65536) P.overflow = true;
        splits = cnt[0] | ((cnt[0] + cnt[1]) << 16) | ((cnt[0] + cnt[1] + cnt[2]) << 32);
      }
      const int64_t md = pieces[active[0]].mode;
      for (int64_t e = a; e < b; e += RUN) {
        chunks.insert(chunks.end(), {0, std::min(RUN, b - e), md, cb, ce, e, key ? idx_addr : 0,
                                     splits});
        P.chunk_dst.push_back(key ? ncl : cluster_of(e));
      }
    }
    i0 = i1;
  }
  P.pos = pos;
}

static void append_phase(Collected* C, const PhaseImage& P) {
  // image layout of the phase: rows, items, chunks, contributions (copied
  // into place by spand_collect_apply_get)
  const int64_t a = C->img_len, b = a + (int64_t)P.rows.size(), c = b + (int64_t)P.tiles.size(),
                d = c + (int64_t)P.chunks.size();
  C->img_len = d + (int64_t)P.contrib.size();
  // persistent warps: 4 CTAs (32 warps) per SM, one warp per item below that
  const int64_t nitem = (int64_t)P.tiles.size() / 2;
  const int64_t grid = std::min<int64_t>((nitem + 7) / 8, 148 * 4);
  C->phases.insert(C->phases.end(), {a, (int64_t)P.rows.size() / 8, b, nitem,
                                     c, (int64_t)P.chunks.size() / 8, d, grid, 0, P.pos});
  C->scratch_len = std::max(C->scratch_len, P.pos);
}

// Dataflow schedule of the whole apply (forward then backward phases): one
// unit per work item and per accumulation chunk, in phase order (items
// before chunks).  Counters (uint64, zeroed per launch; 0 = the dispatch
// counter): per phase and output cluster, the items done; per phase and
// input cluster, the items done (readers); per phase and output cluster,
// the chunks done.  An item waits for the chunks of the last phase that
// wrote its input cluster; a chunk waits for the items of its own phase
// that produce its cluster, for the last writer of its cluster and for
// every reader of the cluster since then (write-after-read).  Every
// dependency points to an earlier unit, so persistent warps taking units in
// order never deadlock.  Unit rows (8 int64): {phase, kind (0 item,
// 1 chunk), index in the phase, first dep, ndeps, counter to bump, second
// counter (-1: none), 0}; deps: {counter, target}; phase rows (8 int64):
// {tasks, items, chunks, contributions (image offsets), scratch base, 0...}.
static void build_dataflow(Collected* C) {
  const int ncl = (int)C->cstart.size() - 1;
  const int32_t FIN = ncl;
  std::vector<int64_t>& U = C->df_units;
  std::vector<int64_t>& D = C->df_deps;
  std::vector<int64_t>& PH = C->df_phase;
  U.clear();
  D.clear();
  PH.clear();
  int64_t nctr = 1;
  std::vector<int64_t> lw_ctr(ncl, -1), lw_tgt(ncl, 0);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> readers(ncl);
  std::vector<std::pair<int64_t, int64_t>> dep;
  auto each = [&](int32_t c, auto&& f) {
    if (c == FIN) {
      for (int32_t q : C->fin) f(q);
    } else {
      f(c);
    }
  };
  auto flush_deps = [&]() -> std::pair<int64_t, int64_t> {
    std::sort(dep.begin(), dep.end());
    dep.erase(std::unique(dep.begin(), dep.end()), dep.end());
    const int64_t at = (int64_t)D.size() / 2;
    for (auto& d : dep) D.insert(D.end(), {d.first, d.second});
    return {at, (int64_t)dep.size()};
  };
  int64_t sb = 0;
  int64_t g = 0;
  for (size_t k = 0; k < C->imgs.size(); ++k) {
    if (C->img_at[k] < 0) continue;
    const PhaseImage& P = C->imgs[k];
    const int64_t* row = C->phases.data() + 10 * g;
    PH.insert(PH.end(), {row[0], row[2], row[4], row[6], sb, 0, 0, 0});
    const int64_t nitem = row[3], nchunk = row[5];
    std::unordered_map<int32_t, std::pair<int64_t, int64_t>> ictr, sctr, cctr;
    for (int64_t i = 0; i < nitem; ++i) {
      auto& a = ictr[P.item_dst[i]];
      if (a.second++ == 0) a.first = nctr++;
      auto& b = sctr[P.item_src[i]];
      if (b.second++ == 0) b.first = nctr++;
    }
    for (int64_t i = 0; i < nchunk; ++i) {
      auto& a = cctr[P.chunk_dst[i]];
      if (a.second++ == 0) a.first = nctr++;
    }
    for (int64_t i = 0; i < nitem; ++i) {
      dep.clear();
      each(P.item_src[i], [&](int32_t c) {
        if (lw_ctr[c] >= 0) dep.push_back({lw_ctr[c], lw_tgt[c]});
      });
      const auto at = flush_deps();
      U.insert(U.end(), {g, 0, i, at.first, at.second, ictr[P.item_dst[i]].first,
                         sctr[P.item_src[i]].first, 0});
    }
    for (auto& kv : sctr)
      each(kv.first, [&](int32_t c) { readers[c].push_back(kv.second); });
    for (int64_t i = 0; i < nchunk; ++i) {
      const int32_t d = P.chunk_dst[i];
      dep.clear();
      auto ic = ictr.find(d);
      if (ic != ictr.end()) dep.push_back(ic->second);
      each(d, [&](int32_t c) {
        if (lw_ctr[c] >= 0) dep.push_back({lw_ctr[c], lw_tgt[c]});
        for (auto& r : readers[c]) dep.push_back(r);
      });
      const auto at = flush_deps();
      U.insert(U.end(), {g, 1, i, at.first, at.second, cctr[d].first, -1, 0});
    }
    for (auto& kv : cctr)
      each(kv.first, [&](int32_t c) {
        lw_ctr[c] = kv.second.first;
        lw_tgt[c] = kv.second.second;
        readers[c].clear();
      });
    sb += row[9];
    ++g;
  }
  C->df_nctr = nctr;
  C->df_scratch = std::max<int64_t>(sb, 1);
}

// Build the apply image.  idx_addr: device address of the final block's
// permuted index list (int32, spand_collect_get's fidx).  out[4]: image
// length, number of forward phases, number of backward phases, scratch.
int spand_collect_apply(void* h, int64_t pool_base, int64_t fac_base, int64_t xbuf,
                        int64_t idx_addr, const uint32_t* bits, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  C->phases.clear();
  C->img_len = 0;
  C->scratch_len = 1;
  // phases compile independently (host threads, largest first), then are
  // laid out in order
  const size_t nf = C->fph.size(), nt = nf + C->bph.size();
  auto phase = [&](size_t k) -> const std::vector<Task>& { return k < nf ? C->fph[k] : C->bph[k - nf]; };
  std::vector<size_t> order(nt);
  for (size_t k = 0; k < nt; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t x, size_t y) { return phase(x).size() > phase(y).size(); });
  C->imgs.assign(nt, PhaseImage());
  std::vector<PhaseImage>& imgs = C->imgs;
  std::atomic<size_t> next{0};
  auto work = [&]() {
    for (size_t q = next++; q < nt; q = next++)
      compile_phase(imgs[order[q]], phase(order[q]), pool_base, fac_base, xbuf, idx_addr, bits,
                    C->cstart);
  };
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned i = 1; i < nth; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  for (const auto& P : imgs)
    if (P.overflow) return -2;   // operator too large for the packed item format
  int64_t nfw = 0, nbw = 0;
  C->img_at.assign(nt, -1);
  for (size_t k = 0; k < nt; ++k) {
    if (imgs[k].rows.empty()) continue;
    C->img_at[k] = C->img_len;
    append_phase(C, imgs[k]);
    if (k < nf) ++nfw;
    else ++nbw;
  }
  out[0] = C->img_len;
  out[1] = nfw;
  out[2] = nbw;
  out[3] = C->scratch_len;
  if (getenv("SPAND_APPLY_DATAFLOW") && getenv("SPAND_APPLY_DATAFLOW")[0] == '1') build_dataflow(C);
  return 0;
}

// the dataflow schedule (after spand_collect_apply): out[4] = units, deps,
// counters, scratch doubles per right-hand side
int spand_collect_dataflow_sizes(void* h, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  out[0] = (int64_t)C->df_units.size() / 8;
  out[1] = (int64_t)C->df_deps.size() / 2;
  out[2] = C->df_nctr;
  out[3] = C->df_scratch;
  return 0;
}

int spand_collect_dataflow(void* h, int64_t* units, int64_t* deps, int64_t* phases) {
  Collected* C = static_cast<Collected*>(h);
  auto cp = [](int64_t* dst, const std::vector<int64_t>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int64_t));
  };
  cp(units, C->df_units);
  cp(deps, C->df_deps);
  cp(phases, C->df_phase);
  return 0;
}

// elimination panels to scan for nonzero rows: out[0] = panel count,
// out[1] = bit words (spand_collect_flag_panels fills 5 int64 per panel:
// {address, ld, rows, cols, first word})
int spand_collect_flag_sizes(void* h, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  out[0] = (int64_t)C->flag_panels.size() / 5;
  out[1] = C->flag_words;
  return 0;
}

int spand_collect_flag_panels(void* h, int64_t pool_base, int64_t* out) {
  Collected* C = static_cast<Collected*>(h);
  const size_t np = C->flag_panels.size() / 5;
  for (size_t k = 0; k < np; ++k) {
    const int64_t* r = C->flag_panels.data() + 5 * k;
    out[5 * k] = pool_base + 8 * r[0];
    for (int q = 1; q < 5; ++q) out[5 * k + q] = r[q];
  }
  return 0;
}

// phase rows (10 int64): tasks_off, ntask, items_off, nitem, chunks_off,
// nchunk, contrib_off, grid (gemv_items CTAs), 0, scratch_used
int spand_collect_apply_get(void* h, int64_t* image, int64_t* phases) {
  Collected* C = static_cast<Collected*>(h);
  if (C->imgs.size() != C->img_at.size()) return -1;   // once per spand_collect_apply
  // each phase's four arrays straight into the caller's (pinned) image, in
  // parallel over phases
  const size_t nt = C->imgs.size();
  std::atomic<size_t> next{0};
  auto work = [&]() {
    for (size_t k = next++; k < nt; k = next++) {
      if (C->img_at[k] < 0) continue;
      int64_t* dst = image + C->img_at[k];
      const PhaseImage& P = C->imgs[k];
      for (const std::vector<int64_t>* v : {&P.rows, &P.tiles, &P.chunks, &P.contrib}) {
        if (!v->empty()) std::memcpy(dst, v->data(), v->size() * sizeof(int64_t));
        dst += v->size();
      }
    }
  };
  const unsigned nth = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned i = 1; i < nth; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  std::memcpy(phases, C->phases.data(), C->phases.size() * sizeof(int64_t));
  // the compiled phases are no longer needed
  std::vector<PhaseImage>().swap(C->imgs);
  return 0;
}

}  // extern "C"
