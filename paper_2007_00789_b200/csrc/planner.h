// Shared definitions of the native level scheduler (planner.cpp) and the
// native collector (collect.cpp).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>

extern "C" int spand_rrqr_capacity(int vmax);
extern "C" int spand_rrqr_cluster_capacity(int vmax, int cs);
extern "C" int spand_rrqr_max_rows_clustered(int cs);

namespace spand {

constexpr int kTile = 64;
// grouped-GEMM tile shapes (gemm.cu, launch tri >> 4): 64x64, 64x16, 32x32,
// 16x16, 16x64, 64x32, 32x64.  Each target gets the smallest shape that covers a narrow
// side; the targets of one logical GEMM are launched once per shape used.
constexpr int kNShape = 7;
constexpr int kShapeM[kNShape] = {64, 64, 32, 16, 16, 64, 32};
constexpr int kShapeN[kNShape] = {64, 16, 32, 16, 64, 32, 64};
inline int tile_shape(int64_t mm, int64_t nn) {
  if (mm <= 16 && nn <= 16) return 3;
  if (nn <= 16) return 1;
  if (mm <= 16) return 4;
  if (mm <= 32 && nn <= 32) return 2;
  if (nn <= 32) return 5;
  if (mm <= 32) return 6;
  return 0;
}
inline void push_tiles(std::vector<int64_t>& v, int64_t t, int64_t mm, int64_t nn, int s,
                       bool lower) {
  const int tm = kShapeM[s], tn = kShapeN[s];
  for (int64_t i = 0; i < mm; i += tm)
    for (int64_t j = 0; j < nn; j += tn) {
      if (lower && j >= i + tm) continue;
      v.push_back((t << 32) | ((i / tm) << 16) | (j / tn));
    }
}
constexpr int kBigPotrf = 256;   // larger diagonal blocks use the blocked (multi-CTA) Cholesky
constexpr int kMaxGroupTotal = 148 * 16;   // >= any cooperative RRQR grid

// Open-addressing hash map int64 -> int32 (linear probing, splitmix64),
// for the block-id lookups of the symbolic analysis and the emission (an
// std::unordered_map spent most of the analysis in node allocation and
// pointer chasing, and its teardown took ~20 ms on C4-L15).
struct BlockMap {
  std::vector<int64_t> keys;
  std::vector<int32_t> vals;
  size_t mask = 0, used = 0;
  static uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap <= keys.size()) return;
    std::vector<int64_t> ok;
    std::vector<int32_t> ov;
    ok.swap(keys);
    ov.swap(vals);
    keys.assign(cap, -1);
    vals.assign(cap, -1);
    mask = cap - 1;
    used = 0;
    for (size_t s = 0; s < ok.size(); ++s)
      if (ok[s] >= 0) put(ok[s], ov[s]);
  }
  void put(int64_t k, int32_t v) {
    if (2 * (used + 1) > keys.size()) reserve(keys.empty() ? 16 : keys.size());
    size_t s = mix((uint64_t)k) & mask;
    while (keys[s] >= 0 && keys[s] != k) s = (s + 1) & mask;
    if (keys[s] < 0) {
      keys[s] = k;
      ++used;
    }
    vals[s] = v;
  }
  int32_t find(int64_t k) const {
    if (keys.empty()) return -1;
    size_t s = mix((uint64_t)k) & mask;
    while (keys[s] >= 0) {
      if (keys[s] == k) return vals[s];
      s = (s + 1) & mask;
    }
    return -1;
  }
};

struct Level {
  int level = 0;
  bool skipped = true;
  std::vector<int> interiors;
  std::vector<std::vector<int>> inbrs;      // neighbours of each interior
  std::vector<int> targets;                 // Schur target block ids (creation order)
  // contributing interiors per target, CSR: tseg_idx[tseg_ptr[t] .. tseg_ptr[t + 1]);
  // tseg_blk holds the segment's two panel blocks {block(wa, s) << 32 | block(wb, s)}
  std::vector<int> tseg_ptr, tseg_idx;
  std::vector<int64_t> tseg_blk;
  // panel blocks block(w, s) of each interior, aligned with inbrs (CSR)
  std::vector<int> inb_ptr, inb_blk;
  std::vector<int> active;
  std::vector<int> resc_blocks;             // off-diagonal blocks among active
  std::vector<int> wave;                    // per active cluster
  std::vector<std::vector<int>> anbrs;      // neighbours of each active cluster
  int nwaves = 0;
  // layout
  std::vector<int64_t> l_off, linv_off, q_off, slot;   // per active
};

struct Plan {
  int ncl = 0, levels = 0, skip = 0;
  std::vector<int64_t> m0;
  std::vector<int32_t> depth;
  std::vector<int64_t> dofs, dptr;   // cluster dofs (original numbering), concatenated
  std::vector<int32_t> bi, bj;
  std::vector<int32_t> bcreated;   // level at which each block came to exist (levels + 1: A's)
  int cur_level = 0;
  BlockMap bid;
  std::vector<Level> lv;
  std::vector<int> fin, fin_blocks;
  // layout
  std::vector<int64_t> boff, elim_linv;
  int64_t pool_size = 0, fac_size = 0, fcap = 0, f_off = 0, flinv_off = 0;
  int64_t n_events = 0, n_info = 0, temp_size = 0, temp_bound = 0;
  // program
  std::vector<int64_t> prog, launches;
  int cap_override = 0;
  int nk = 0;   // near-kernel vectors (extension; 0: reference path)
  // RRQR group sizes within a wave: 0 ~ m n, 1 ~ m^2, 2 ~ m sqrt(m n),
  // 3 ~ m^a n^b.  The default m^1.25 n^0.5 (C4-L15 sweep: 1.14 s at m n,
  // 1.105 s here) gives tall panels -- more sequential steps -- more CTAs
  int group_weight = 3;
  double gexp_m = 1.25, gexp_n = 0.5;
  // clustered RRQR waves (rrqr.cu): cluster size (0 = off) and the smallest
  // panel height for which a wave is launched clustered
  int cluster_cs = 0, cluster_min_rows = 256;
  static constexpr int64_t kNkHead = 19;   // nearkernel.cu kWsHead
  int64_t nk_ws(int64_t mc) const { return nk ? kNkHead + 2 * mc * nk + mc * mc : 0; }

  // Trailing-matrix fingerprints (reference EliminationState.digest,
  // factorize.py:222-229, recorded per level at :347).  When on, every
  // level ends with a launch (type 11) that hashes the live window of each
  // block alive at that point into a record {i, j, rows, cols, h}; the host
  // folds the records of a level, in key order, into a sha256.  A block
  // (i, j) is alive at the end of level l iff it exists by then (created at
  // level >= l) and neither cluster has been eliminated (depth < l).
  bool digest = false;
  int64_t dig_base = 0;                       // device address of the records
  std::vector<std::vector<int>> dig_blocks;   // per level (lv order), key order
  std::vector<int64_t> dig_first;             // first record index per level
  int64_t dig_records = 0;
  void prepare_digest() {
    dig_blocks.assign(lv.size(), {});
    for (size_t b = 0; b < bi.size(); ++b) {
      const int death = std::max(depth[bi[b]], depth[bj[b]]);
      for (int l = std::min(bcreated[b], levels); l > death && l >= 1; --l)
        dig_blocks[(size_t)(levels - l)].push_back((int)b);
    }
    dig_first.assign(lv.size() + 1, 0);
    for (size_t k = 0; k < lv.size(); ++k) {
      auto& v = dig_blocks[k];
      std::sort(v.begin(), v.end(), [&](int x, int y) {
        return key(bi[x], bj[x]) < key(bi[y], bj[y]);
      });
      dig_first[k + 1] = dig_first[k] + (int64_t)v.size();
    }
    dig_records = dig_first[lv.size()];
  }

  int64_t key(int i, int j) const { return (int64_t)i * ncl + j; }
  int block(int i, int j) const { return bid.find(key(i, j)); }
  int new_block(int i, int j, std::vector<std::vector<int>>& cb) {
    const int b = (int)bi.size();
    bi.push_back(i);
    bj.push_back(j);
    bcreated.push_back(cur_level);
    bid.put(key(i, j), b);
    cb[i].push_back(b);
    if (j != i) cb[j].push_back(b);
    return b;
  }

  // Symbolic elimination over the levels (factorize.py:309-362): which
  // blocks exist, which interiors update which targets, the active sets and
  // sparsification waves.  Adjacency and block lists use lazy deletion
  // (eliminated clusters are filtered when read); the result is identical
  // to the ordered-set formulation (neighbour lists are sorted on read).
  void symbolic(int64_t npairs, const int64_t* pairs) {
    std::vector<std::vector<int>> adj(ncl), cb(ncl);
    {
      std::vector<int> cnt(ncl, 1);
      for (int64_t t = 0; t < npairs; ++t) {
        ++cnt[pairs[t] / ncl];
        ++cnt[pairs[t] % ncl];
      }
      for (int c = 0; c < ncl; ++c) {
        cb[c].reserve(2 * cnt[c]);
        adj[c].reserve(2 * cnt[c]);
      }
    }
    bid.reserve((size_t)npairs * 4);
    bi.reserve((size_t)npairs * 2);
    bj.reserve((size_t)npairs * 2);
    bcreated.reserve((size_t)npairs * 2);
    cur_level = levels + 1;
    for (int64_t t = 0; t < npairs; ++t) {
      const int i = (int)(pairs[t] / ncl), j = (int)(pairs[t] % ncl);
      new_block(i, j, cb);
      if (i != j) {
        adj[i].push_back(j);
        adj[j].push_back(i);
      }
    }
    for (int c = 0; c < ncl; ++c)
      if (bid.find(key(c, c)) < 0) new_block(c, c, cb);
    std::vector<char> alive(ncl, 1);
    auto live_nbrs = [&](int c) {
      std::vector<int> nb;
      nb.reserve(adj[c].size());
      for (int w : adj[c])
        if (alive[w]) nb.push_back(w);
      std::sort(nb.begin(), nb.end());
      adj[c] = nb;   // compact
      return nb;
    };
    std::vector<int> seg_t, seg_s;   // (target index, interior) pairs of a level
    std::vector<int64_t> seg_b;      // their panel blocks
    std::vector<int> tpos;      // block id -> target index at this level, stamped
    std::vector<int> tstamp;
    std::vector<int> wave_of(ncl, 0);
#ifdef SPAND_PLAN_TIMING
    double t_int = 0, t_act = 0;
#endif
    for (int level = levels; level >= 1; --level) {
#ifdef SPAND_PLAN_TIMING
      auto c0 = std::chrono::steady_clock::now();
#endif
      Level L;
      L.level = level;
      cur_level = level;
      for (int c = 0; c < ncl; ++c)
        if (alive[c] && depth[c] == level) L.interiors.push_back(c);
      L.inb_ptr.assign(1, 0);
      for (int s : L.interiors) {
        std::vector<int> nb = live_nbrs(s);
        L.inbrs.push_back(nb);
        const size_t ib0 = L.inb_blk.size();
        for (int w : nb) L.inb_blk.push_back(bid.find(key(w, s)));
        L.inb_ptr.push_back((int)L.inb_blk.size());
        for (size_t a2 = 0; a2 < nb.size(); ++a2)
          for (size_t b2 = a2; b2 < nb.size(); ++b2) {
            const int wa = nb[a2], wb = nb[b2];
            int blk = bid.find(key(wa, wb));
            if (blk < 0) {
              blk = new_block(wa, wb, cb);
              if (wa != wb) {
                adj[wa].push_back(wb);
                adj[wb].push_back(wa);
              }
            }
            if ((int)tpos.size() <= blk) {
              tpos.resize(bi.size() + 1024, -1);
              tstamp.resize(bi.size() + 1024, -1);
            }
            if (tstamp[blk] != level) {
              tstamp[blk] = level;
              tpos[blk] = (int)L.targets.size();
              L.targets.push_back(blk);
            }
            seg_t.push_back(tpos[blk]);
            seg_s.push_back(s);
            seg_b.push_back(((int64_t)L.inb_blk[ib0 + a2] << 32) |
                            (int64_t)L.inb_blk[ib0 + b2]);
          }
        alive[s] = 0;
        adj[s].clear();
        cb[s].clear();
      }
      // group the (target, interior) pairs by target, interior order kept
      L.tseg_ptr.assign(L.targets.size() + 1, 0);
      for (int t2 : seg_t) ++L.tseg_ptr[t2 + 1];
      for (size_t t2 = 0; t2 < L.targets.size(); ++t2) L.tseg_ptr[t2 + 1] += L.tseg_ptr[t2];
      L.tseg_idx.resize(seg_s.size());
      L.tseg_blk.resize(seg_s.size());
      {
        std::vector<int> fillp(L.tseg_ptr.begin(), L.tseg_ptr.end() - 1);
        for (size_t q = 0; q < seg_s.size(); ++q) {
          const int at = fillp[seg_t[q]]++;
          L.tseg_idx[at] = seg_s[q];
          L.tseg_blk[at] = seg_b[q];
        }
      }
      seg_t.clear();
      seg_s.clear();
      seg_b.clear();
      L.skipped = (levels - level) < skip;
#ifdef SPAND_PLAN_TIMING
      auto c1 = std::chrono::steady_clock::now();
      t_int += std::chrono::duration<double>(c1 - c0).count();
#endif
      if (!L.skipped) {
        for (int c = 0; c < ncl; ++c)
          if (alive[c]) L.active.push_back(c);
        std::vector<std::pair<int, int>> rb;
        for (int c : L.active)
          for (int b2 : cb[c])
            if (bi[b2] == c && bj[b2] != c && alive[bj[b2]]) rb.push_back({bi[b2], bj[b2]});
        std::sort(rb.begin(), rb.end());
        for (auto& pr : rb) L.resc_blocks.push_back(block(pr.first, pr.second));
        for (int p : L.active) {
          std::vector<int> nb = live_nbrs(p);
          int wv = 0;
          for (int q : nb)
            if (q < p) wv = std::max(wv, wave_of[q] + 1);
          wave_of[p] = wv;
          L.wave.push_back(wv);
          L.anbrs.push_back(nb);
          L.nwaves = std::max(L.nwaves, wv + 1);
        }
      }
#ifdef SPAND_PLAN_TIMING
      t_act += std::chrono::duration<double>(std::chrono::steady_clock::now() - c1).count();
#endif
      lv.push_back(std::move(L));
    }
#ifdef SPAND_PLAN_TIMING
    printf("interiors %.4f actives %.4f\n", t_int, t_act);
#endif
    for (int c = 0; c < ncl; ++c)
      if (alive[c]) fin.push_back(c);
    std::vector<std::pair<int, int>> fb;
    for (int c : fin)
      for (int b2 : cb[c])
        if (bi[b2] == c && alive[bj[b2]]) fb.push_back({bi[b2], bj[b2]});
    std::sort(fb.begin(), fb.end());
    for (auto& pr : fb) fin_blocks.push_back(block(pr.first, pr.second));
  }

  void layout() {
    boff.resize(bi.size());
    pool_size = 0;
    for (size_t b = 0; b < bi.size(); ++b) {
      boff[b] = pool_size;
      pool_size += m0[bi[b]] * m0[bj[b]];
    }
    elim_linv.assign(ncl, -1);
    fac_size = 0;
    n_events = n_info = 0;
    for (auto& L : lv) {
      for (int s : L.interiors) {
        elim_linv[s] = fac_size;
        fac_size += m0[s] * m0[s];
      }
      n_info += (int64_t)L.interiors.size();
      if (!L.skipped) {
        for (int p : L.active) {
          L.l_off.push_back(fac_size);
          fac_size += m0[p] * m0[p];
          L.linv_off.push_back(fac_size);
          fac_size += m0[p] * m0[p];
          L.q_off.push_back(fac_size);
          fac_size += m0[p] * m0[p];
          L.slot.push_back(n_events++);
        }
        n_info += (int64_t)L.active.size();
      }
    }
    fcap = 0;
    for (int c : fin) fcap += m0[c];
    f_off = fac_size;
    fac_size += fcap * fcap;
    flinv_off = fac_size;
    fac_size += fcap * fcap;
    n_info += 1;
    // temporary workspace bound (max over sequential phases), so the
    // program can be emitted in one pass after a single allocation
    int64_t need = fcap * fcap;
    for (auto& L : lv) {
      int64_t trsm = 0, tri = 0, pflag_bytes = 0;
      for (size_t k = 0; k < L.interiors.size(); ++k) {
        const int s = L.interiors[k];
        tri += m0[s] * m0[s];
        for (int w : L.inbrs[k]) {
          trsm += m0[w] * m0[s];
          pflag_bytes += (m0[w] + 15) / 16;   // row-chunk flags behind the products
        }
      }
      trsm += (pflag_bytes + 7) / 8 + 1;
      need = std::max({need, trsm, tri});
      if (L.skipped) continue;
      int64_t resc = 0, tri2 = 0, kmask_bytes = 0;
      for (int b : L.resc_blocks) {
        resc += m0[bi[b]] * m0[bj[b]];
        kmask_bytes += (m0[bi[b]] + 15) / 16;   // K-chunk masks behind the products
      }
      resc += (kmask_bytes + 7) / 8 + 1;
      for (int p : L.active) tri2 += m0[p] * m0[p];
      need = std::max({need, resc, tri2});
      for (int wv = 0; wv < L.nwaves; ++wv) {
        int64_t rq = 68 * (int64_t)kMaxGroupTotal, lists = 4 * (int64_t)kMaxGroupTotal;
        int64_t mn = INT64_MAX, np = 0;
        for (size_t k = 0; k < L.active.size(); ++k) {
          if (L.wave[k] != wv) continue;
          int64_t ncap = 0;
          for (int w : L.anbrs[k]) ncap += m0[w];
          const int64_t mc = m0[L.active[k]];
          rq += mc * std::max<int64_t>(ncap, 1) + mc * mc + 32 * (ncap + mc) + 32 * mc + 1024 +
                2 * ncap +
                3 * mc + 8 + 1024 + (3 * ncap + 1) / 2 + 1 + 1 + 68 + nk_ws(mc);
          lists += 2 * 8 * std::max<int64_t>(ncap, 1) + 1;
          mn = std::min(mn, mc);
          ++np;
        }
        // a clustered wave's list copies (superset of the emission test)
        if (cluster_cs > 1 && np > 0 && mn >= cluster_min_rows &&
            np <= kMaxGroupTotal / cluster_cs)
          rq += lists;
        need = std::max(need, rq);
      }
    }
    temp_bound = std::max<int64_t>(need, 1);
  }

  // ---------------------------------------------------------------- emit
  int64_t pool_base = 0, fac_base = 0, temp_base = 0, ctr_base = 0;
  int64_t info_next = 0, ctr_next = 0;

  int64_t blk_ptr(int i, int j) const { return pool_base + 8 * boff[block(i, j)]; }
  // Small vector with inline storage: GEMM targets are built by the hundred
  // thousand per level, and two heap vectors per target dominated the emission
  struct SmallVec {
    static constexpr int kIn = 16;
    int64_t buf[kIn];
    std::vector<int64_t> heap;
    int n = 0;
    void push_back(int64_t x) {
      if (n < kIn) {
        buf[n] = x;
      } else {
        if (n == kIn) heap.assign(buf, buf + kIn);
        heap.push_back(x);
      }
      ++n;
    }
    const int64_t* data() const { return n <= kIn ? buf : heap.data(); }
    size_t size() const { return (size_t)n; }
    bool empty() const { return n == 0; }
  };
  template <class V>
  static void opnd(V& v, int64_t p, int rc, int cc, int64_t rs = 0, int64_t cs = 0,
                   int64_t rn = -1, int64_t cn = -1) {
    const int64_t e[7] = {p, rc, cc, rs, cs, rn, cn};
    for (int64_t x : e) v.push_back(x);
  }
  // sub-operand at (rs, cs) of o, clamped to rn x cn (< 0: to o's extent)
  template <class V>
  static void sub(V& v, const int64_t* o, int64_t rs, int64_t cs, int64_t rn, int64_t cn) {
    const int64_t rl = o[5] < 0 ? -1 : std::max(o[5] - rs, (int64_t)0);
    const int64_t cl = o[6] < 0 ? -1 : std::max(o[6] - cs, (int64_t)0);
    const int64_t r = rn < 0 ? rl : (rl < 0 ? rn : std::min(rn, rl));
    const int64_t c = cn < 0 ? cl : (cl < 0 ? cn : std::min(cn, cl));
    const int64_t e[7] = {o[0], o[1], o[2], o[3] + rs, o[4] + cs, r, c};
    for (int64_t x : e) v.push_back(x);
  }
  bool dry = false;   // sizing pass: compute temp_size only, emit nothing
  std::vector<int64_t> blkflag;   // block -> row-chunk flag offset (panels of the level being emitted)
  int64_t push(const std::vector<int64_t>& rows) {
    if (dry) return 0;
    const int64_t at = (int64_t)prog.size();
    prog.insert(prog.end(), rows.begin(), rows.end());
    return at;
  }
  void launch(int64_t type, int64_t count, int64_t a, int64_t b = 0, int64_t c = 0,
              int64_t x0 = 0, int64_t x1 = 0, int64_t x2 = 0, double alpha = 0.0,
              double beta = 0.0) {
    int64_t ab, bb;
    std::memcpy(&ab, &alpha, 8);
    std::memcpy(&bb, &beta, 8);
    if (dry) return;
    launches.insert(launches.end(), {type, count, a, b, c, x0, x1, x2, ab, bb, 0, 0, 0, 0, 0, 0});
  }

  struct Target {
    SmallVec c;          // 7
    SmallVec segs;       // 14 per segment (or 1 per segment, compact)
    int64_t mm, nn;
  };
  // tri: triangular-operand K bounds (gemm.cu): 1 A lower, 2 B lower with
  // C = A B^T, 4 B lower with C = A B
  // mask_addr != 0: K-chunk masks (gemm.cu kmask_kernel) of the targets' B
  // operands at that device address, one byte per 16 rows of B, target t at
  // the running sum of ceil(mm / 16) (mm = the static row count of C and B)
  void gemm(const std::vector<Target>& ts, double alpha, double beta, int bT, int lower,
            int tri = 0, int compact = 0, int64_t mask_addr = 0) {
    if (ts.empty()) return;
    const int64_t sw = compact ? 1 : 14;
    std::vector<int64_t> trow, srow, tiles[kNShape], kmoff;
    int64_t nseg = 0, moff = 0;
    trow.reserve(8 * ts.size() + 8);
    for (size_t t = 0; t < ts.size(); ++t) {
      if (mask_addr) {
        kmoff.push_back(moff);
        moff += (ts[t].mm + 15) / 16;
      }
      trow.insert(trow.end(), ts[t].c.data(), ts[t].c.data() + ts[t].c.size());
      trow.push_back(nseg);
      srow.insert(srow.end(), ts[t].segs.data(), ts[t].segs.data() + ts[t].segs.size());
      nseg += (int64_t)ts[t].segs.size() / sw;
      if (dry) continue;
      push_tiles(tiles[tile_shape(ts[t].mm, ts[t].nn)], (int64_t)t, ts[t].mm, ts[t].nn,
                 tile_shape(ts[t].mm, ts[t].nn), lower != 0);
    }
    trow.insert(trow.end(), {0, 0, 0, 0, 0, 0, 0, nseg});
    if (dry) return;
    emit_gemm(tiles, trow, srow, alpha, beta, bT, lower, tri, compact, mask_addr,
              mask_addr ? &kmoff : nullptr);
  }
  void emit_gemm(std::vector<int64_t> (&tiles)[kNShape], std::vector<int64_t>& trow,
                 std::vector<int64_t>& srow, double alpha, double beta, int bT, int lower,
                 int tri, int compact, int64_t mask_addr = 0,
                 const std::vector<int64_t>* kmoff = nullptr, bool mask_pass = true) {
    int64_t b = -1, c = -1, ko = 0;
    for (int s = 0; s < kNShape; ++s) {
      if (tiles[s].empty()) continue;
      if (b < 0) {
        if (srow.empty()) srow.assign(14, 0);
        b = push(trow);
        c = push(srow);
        if (mask_addr) {
          ko = push(*kmoff);
          // which operand the bytes describe: B's K chunks (C = A B) or A's rows
          // (mask_pass = false: the flags were written by an earlier launch)
          if (mask_pass) launch(12, (int64_t)kmoff->size(), b, c, ko, mask_addr, bT ? 0 : 1);
        }
      }
      const int64_t a = push(tiles[s]);
      launch(3, (int64_t)tiles[s].size(), a, b, c, bT, lower, tri | (s << 4), alpha, beta);
      launches[launches.size() - 6] = compact;   // field 10
      if (mask_addr) {
        launches[launches.size() - 5] = mask_addr;   // field 11
        // field 12: the offsets row relative to the targets row (only the
        // fields a, b, c are rebased when a program chunk is exported)
        launches[launches.size() - 4] = ko - b;
      }
    }
  }

  // Flat GEMM target list, written in place (the per-level hot paths: the
  // panel TRSMs and the grouped Schur updates emit ~10^5 targets each on the
  // leaf levels; no intermediate Target objects)
  struct FlatGemm {
    std::vector<int64_t> trow, srow, tiles[kNShape];
    int64_t nseg = 0, sw = 14, ntarget = 0;
    bool lower = false;
    void reserve(size_t nt, size_t nsegs) {
      trow.reserve(8 * nt + 8);
      srow.reserve(sw * nsegs + 14);
      tiles[0].reserve(nt / 4 + 16);
    }
    // begin a target: C operand (7 values), extents for the tile grid
    template <class... A>
    void target(int64_t mm, int64_t nn, bool dry, A... c) {
      const int64_t e[7] = {c...};
      trow.insert(trow.end(), e, e + 7);
      trow.push_back(nseg);
      if (!dry) {
        const int s = tile_shape(mm, nn);
        push_tiles(tiles[s], ntarget, mm, nn, s, lower);
      }
      ++ntarget;
    }
    void seg(int64_t s) {
      srow.push_back(s);
      if (sw == 1) ++nseg;
    }
    void seg_opnds(const int64_t* a, const int64_t* b) {
      srow.insert(srow.end(), a, a + 7);
      srow.insert(srow.end(), b, b + 7);
      ++nseg;
    }
  };
  void gemm_flat(FlatGemm& g, double alpha, double beta, int bT, int tri = 0,
                 int64_t mask_addr = 0, const std::vector<int64_t>* kmoff = nullptr,
                 bool mask_pass = true) {
    if (g.ntarget == 0) return;
    g.trow.insert(g.trow.end(), {0, 0, 0, 0, 0, 0, 0, g.nseg});
    if (dry) return;
    emit_gemm(g.tiles, g.trow, g.srow, alpha, beta, bT, g.lower ? 1 : 0, tri, g.sw == 1 ? 1 : 0,
              mask_addr, kmoff, mask_pass);
  }

  // batched triangular inverses: 64-tiles + recursive doubling GEMMs
  void trtri(const std::vector<std::vector<int64_t>>& Ls, const std::vector<std::vector<int64_t>>& Xs,
             const std::vector<int64_t>& sizes, int64_t temp_at) {
    if (Ls.empty()) return;
    std::vector<int64_t> rows;
    int64_t nmax = 0;
    for (size_t t = 0; t < Ls.size(); ++t) {
      nmax = std::max(nmax, sizes[t]);
      for (int64_t o = 0; o < sizes[t]; o += kTile) {
        sub(rows, Ls[t].data(), o, o, kTile, kTile);
        sub(rows, Xs[t].data(), o, o, kTile, kTile);
      }
    }
    if (!rows.empty()) launch(2, (int64_t)rows.size() / 14, push(rows));
    if (nmax <= kTile) return;
    std::vector<int64_t> toff;
    int64_t acc = temp_at;
    for (size_t t = 0; t < Ls.size(); ++t) {
      toff.push_back(acc);
      acc += m0v(Ls[t][1]) * m0v(Ls[t][1]);
    }
    temp_size = std::max(temp_size, acc);
    for (int64_t s = kTile; s < nmax; s *= 2) {
      std::vector<Target> g1, g2;
      for (size_t t = 0; t < Ls.size(); ++t) {
        std::vector<int64_t> tmp(Xs[t]);
        tmp[0] = temp_base + 8 * toff[t];
        for (int64_t o = 0; o < sizes[t] - s; o += 2 * s) {
          Target a;
          sub(a.c, tmp.data(), o + s, o, s, s);
          sub(a.segs, Ls[t].data(), o + s, o, s, s);
          sub(a.segs, Xs[t].data(), o, o, s, s);
          a.mm = s;
          a.nn = s;
          g1.push_back(std::move(a));
          Target b;
          sub(b.c, Xs[t].data(), o + s, o, s, s);
          sub(b.segs, Xs[t].data(), o + s, o + s, s, s);
          sub(b.segs, tmp.data(), o + s, o, s, s);
          b.mm = s;
          b.nn = s;
          g2.push_back(std::move(b));
        }
      }
      gemm(g1, 1.0, 0.0, 0, 0, 4);    // tmp = L21 X11 (X11 lower)
      gemm(g2, -1.0, 0.0, 0, 0, 1);   // X21 = -X22 tmp (X22 lower)
    }
  }
  int64_t m0v(int64_t c) const { return c < ncl ? m0[c] : fcap; }

  // Cholesky of a batch of diagonal operands (full live windows, 7 int64
  // each) with info slots info_next.. in operator order.  Blocks up to
  // kBigPotrf rows: one CTA each.  Larger blocks: right-looking blocked
  // Cholesky over 64-wide panels -- diagonal potrf, 64x64 inverse, panel
  // TRSM and lower trailing update as tensor-core GEMMs -- so a 3000-row
  // block uses the whole GPU instead of one SM.  Scratch: an m0 x m0 image
  // in temp per large block (temp_at on).
  void potrf(const std::vector<std::vector<int64_t>>& ops, int64_t temp_at) {
    std::vector<int64_t> small;
    std::vector<size_t> big;
    for (size_t t = 0; t < ops.size(); ++t) {
      const int64_t sz = m0v(ops[t][1]);
      if (sz > kBigPotrf) big.push_back(t);
      else {
        small.insert(small.end(), ops[t].begin(), ops[t].end());
        small.push_back(info_next + (int64_t)t);
      }
    }
    if (!small.empty()) launch(1, (int64_t)small.size() / 8, push(small), 0, 0, 0, 0);
    if (!big.empty()) {
      std::vector<int64_t> scr;
      int64_t acc = temp_at, smax = 0;
      for (size_t t : big) {
        scr.push_back(acc);
        const int64_t sz = m0v(ops[t][1]);
        acc += sz * sz;
        smax = std::max(smax, sz);
      }
      temp_size = std::max(temp_size, acc);
      for (int64_t o = 0; o < smax; o += kTile) {
        std::vector<int64_t> diag, tri, cps;
        std::vector<Target> pan, trail;
        for (size_t u = 0; u < big.size(); ++u) {
          const size_t t = big[u];
          const int64_t sz = m0v(ops[t][1]);
          if (sz <= o) continue;
          const int64_t* op = ops[t].data();
          std::vector<int64_t> tmp(ops[t]);
          tmp[0] = temp_base + 8 * scr[u];
          sub(diag, op, o, o, kTile, kTile);
          diag.push_back(info_next + (int64_t)t);
          sub(tri, op, o, o, kTile, kTile);
          sub(tri, tmp.data(), o, o, kTile, kTile);
          if (sz > o + kTile) {
            sub(cps, op, o + kTile, o, -1, kTile);
            sub(cps, tmp.data(), o + kTile, o, -1, kTile);
            cps.push_back(0);
            Target a;
            sub(a.c, op, o + kTile, o, -1, kTile);
            sub(a.segs, tmp.data(), o + kTile, o, -1, kTile);
            sub(a.segs, tmp.data(), o, o, kTile, kTile);
            a.mm = sz - o - kTile;
            a.nn = kTile;
            pan.push_back(std::move(a));
            Target b;
            sub(b.c, op, o + kTile, o + kTile, -1, -1);
            sub(b.segs, op, o + kTile, o, -1, kTile);
            sub(b.segs, op, o + kTile, o, -1, kTile);
            b.mm = b.nn = sz - o - kTile;
            trail.push_back(std::move(b));
          }
        }
        launch(1, (int64_t)diag.size() / 8, push(diag), 0, 0, o, 1);
        launch(2, (int64_t)tri.size() / 14, push(tri));
        if (!cps.empty()) launch(4, (int64_t)cps.size() / 15, push(cps));
        gemm(pan, 1.0, 0.0, 1, 0, 2);   // L21 = A21 L11^-T
        gemm(trail, -1.0, 1.0, 1, 1);   // A22 -= L21 L21^T (lower tiles)
      }
      // zero the strict upper triangles (dpotrf clean, dense.py:53)
      std::vector<int64_t> z;
      for (size_t t : big) {
        z.insert(z.end(), ops[t].begin(), ops[t].end());
        z.insert(z.end(), ops[t].begin(), ops[t].end());
        z.push_back(1);
      }
      launch(4, (int64_t)z.size() / 15, push(z));
    }
    info_next += (int64_t)ops.size();
  }

  static std::vector<int> groups(const std::vector<int64_t>& works, int cap) {
    double total = 0;
    for (auto w : works) total += (double)w;
    std::vector<int> g;
    for (auto w : works) g.push_back(std::max(1, total > 0 ? (int)(cap * (double)w / total) : 1));
    int64_t sum = 0;
    for (int x : g) sum += x;
    while (sum > cap) {
      auto it = std::max_element(g.begin(), g.end());
      if (*it == 1) break;
      --*it;
      --sum;
    }
    return g;
  }

  void emit() {
    emit_begin();
    while (emit_next()) {
    }
  }
  // Incremental emission, one level per call (then the final block), so
  // the host can launch level l while it emits level l + 1.  The chunk of a
  // call is prog[chunk_prog0:] / launches[chunk_launch0:].
  size_t next_level = 0, chunk_prog0 = 0, chunk_launch0 = 0;
  bool final_done = false;
  void emit_begin() {
    prog.clear();
    launches.clear();
    info_next = ctr_next = 0;
    temp_size = 1;
    next_level = 0;
    final_done = false;
    chunk_prog0 = chunk_launch0 = 0;
  }
  bool emit_next() {
    chunk_prog0 = prog.size();
    chunk_launch0 = launches.size();
    if (next_level < lv.size()) {
      emit_level(lv[next_level++]);
      return true;
    }
    if (!final_done) {
      final_done = true;
      emit_final();
      return true;
    }
    return false;
  }
  void emit_level(Level& L) {
    emit_level_core(L);
    if (digest) emit_digest((size_t)(levels - L.level));
  }
  // pieces {block ptr, i, j, first column, columns, record address}, at
  // most 64K stored entries each (digest_kernel in dense_small.cu)
  void emit_digest(size_t k) {
    std::vector<int64_t> rows;
    int64_t rec = dig_first[k];
    for (int b : dig_blocks[k]) {
      const int i = bi[b], j = bj[b];
      const int64_t cpp = std::max<int64_t>(1, 65536 / std::max<int64_t>(m0[i], 1));
      const int64_t addr = dig_base + 40 * rec++;
      for (int64_t c0 = 0; c0 < std::max<int64_t>(m0[j], 1); c0 += cpp)
        rows.insert(rows.end(), {pool_base + 8 * boff[b], i, j, c0,
                                 std::min<int64_t>(cpp, m0[j] - c0), addr});
    }
    if (!rows.empty()) launch(11, (int64_t)rows.size() / 6, push(rows));
  }
  void emit_level_core(Level& L) {
    {
      if (!L.interiors.empty()) {
        std::vector<std::vector<int64_t>> pops;
        for (int s : L.interiors) {
          pops.emplace_back();
          opnd(pops.back(), blk_ptr(s, s), s, s);
        }
        potrf(pops, 0);
        std::vector<std::vector<int64_t>> Ls, Xs;
        std::vector<int64_t> sz;
        for (int s : L.interiors) {
          std::vector<int64_t> l, x;
          opnd(l, blk_ptr(s, s), s, s);
          opnd(x, fac_base + 8 * elim_linv[s], s, s);
          Ls.push_back(std::move(l));
          Xs.push_back(std::move(x));
          sz.push_back(m0[s]);
        }
        trtri(Ls, Xs, sz, 0);
        // panel TRSM as a product with the explicit inverse, into temp, copied back
        FlatGemm tg;
        std::vector<int64_t> cps, pflag;   // pflag: row-chunk flag offset of every panel
        int64_t acc = 0, flag_bytes = 0;
        tg.reserve(L.inb_blk.size(), L.inb_blk.size());
        cps.reserve(15 * L.inb_blk.size());
        for (size_t k = 0; k < L.interiors.size(); ++k) {
          const int s = L.interiors[k];
          const int64_t linv_s = fac_base + 8 * elim_linv[s];
          for (size_t u = 0; u < L.inbrs[k].size(); ++u) {
            const int w = L.inbrs[k][u];
            const int64_t pws = pool_base + 8 * boff[L.inb_blk[L.inb_ptr[k] + u]];
            // a panel one column tile wide is updated in place: each tile
            // reads its own rows of the block over the whole K range before
            // its epilogue writes them (no other tile touches those rows)
            const bool inplace = m0[s] <= kShapeN[tile_shape(m0[w], m0[s])];
            const int64_t tmp = inplace ? pws : temp_base + 8 * acc;
            tg.target(m0[w], m0[s], dry, tmp, (int64_t)w, (int64_t)s, (int64_t)0, (int64_t)0,
                      (int64_t)-1, (int64_t)-1);
            const int64_t oa[7] = {pws, w, s, 0, 0, -1, -1};
            const int64_t ob[7] = {linv_s, s, s, 0, 0, -1, -1};
            tg.seg_opnds(oa, ob);
            pflag.push_back(flag_bytes);
            {
              const int blk = L.inb_blk[L.inb_ptr[k] + u];
              if ((int)blkflag.size() <= blk) blkflag.resize(bi.size() + 1024, 0);
              blkflag[blk] = flag_bytes;
            }
            flag_bytes += (m0[w] + 15) / 16;
            if (inplace) continue;
            cps.insert(cps.end(), {tmp, w, s, 0, 0, -1, -1, pws, w, s, 0, 0, -1, -1, 0});
            acc += m0[w] * m0[s];
          }
        }
        // row-chunk flags of the panels behind the products' temp: an
        // interior touches a few dofs of each separator, so most 64-row tiles
        // of a panel hold only zeros and are skipped (gemm.cu)
        const int64_t flag_addr = temp_base + 8 * acc;
        temp_size = std::max(temp_size, acc + (flag_bytes + 7) / 8 + 1);
        gemm_flat(tg, 1.0, 0.0, 1, 2, flag_addr, &pflag);    // panel L_s^-T
        if (!cps.empty()) launch(4, (int64_t)cps.size() / 15, push(cps));
        // grouped Schur / fill update: off-diagonal targets, then diagonal
        // ones (lower tiles only: potrf reads the lower triangle)
        for (int diag = 0; diag < 2; ++diag) {
          FlatGemm st;
          std::vector<int64_t> sflag;   // per segment: {A panel flags << 32 | B panel flags}
          st.sw = 1;
          st.lower = diag == 1;
          st.reserve(L.targets.size(), L.tseg_idx.size());
          sflag.reserve(L.tseg_idx.size());
          for (size_t t = 0; t < L.targets.size(); ++t) {
            const int b = L.targets[t];
            const int wa = bi[b], wb = bj[b];
            if ((wa == wb) != (diag == 1)) continue;
            st.target(m0[wa], m0[wb], dry, pool_base + 8 * boff[b], (int64_t)wa, (int64_t)wb,
                      (int64_t)0, (int64_t)0, (int64_t)-1, (int64_t)-1);
            for (int q = L.tseg_ptr[t]; q < L.tseg_ptr[t + 1]; ++q) {
              // (the two table reads are random over ~10^5 blocks: prefetch ahead)
              if ((size_t)q + 16 < L.tseg_blk.size()) {
                __builtin_prefetch(&blkflag[L.tseg_blk[q + 16] >> 32]);
                __builtin_prefetch(&blkflag[L.tseg_blk[q + 16] & 0xffffffffLL]);
              }
              st.seg(L.tseg_blk[q]);
              sflag.push_back((blkflag[L.tseg_blk[q] >> 32] << 32) |
                              blkflag[L.tseg_blk[q] & 0xffffffffLL]);
            }
          }
          // the panels' row-chunk flags (written before the panel TRSM) pick
          // the segments each tile opens
          gemm_flat(st, -1.0, 1.0, 1, 0, flag_addr, &sflag, false);
        }
      }
      if (L.skipped) return;
      // rescale every active interface (factorize.py:165-173)
      const size_t na = L.active.size();
      std::vector<int64_t> c1, c2;
      std::vector<std::vector<int64_t>> pops;
      std::vector<std::vector<int64_t>> Ls, Xs;
      std::vector<int64_t> sz;
      for (size_t k = 0; k < na; ++k) {
        const int p = L.active[k];
        opnd(c1, blk_ptr(p, p), p, p);
        opnd(c1, fac_base + 8 * L.l_off[k], p, p);
        c1.push_back(1);
        pops.emplace_back();
        opnd(pops.back(), fac_base + 8 * L.l_off[k], p, p);
        std::vector<int64_t> l, x;
        opnd(l, fac_base + 8 * L.l_off[k], p, p);
        opnd(x, fac_base + 8 * L.linv_off[k], p, p);
        Ls.push_back(std::move(l));
        Xs.push_back(std::move(x));
        sz.push_back(m0[p]);
        opnd(c2, blk_ptr(p, p), p, p);
        opnd(c2, blk_ptr(p, p), p, p);
        c2.push_back(2);
      }
      if (na) {
        launch(4, (int64_t)na, push(c1));
        potrf(pops, 0);
        if (nk) {
          // near-kernel coordinates: u_p <- Z_p^T u_p (nearkernel.cu)
          std::vector<int64_t> rr;
          int64_t vm = 1;
          for (size_t k = 0; k < na; ++k) {
            const int p = L.active[k];
            rr.insert(rr.end(), {p, fac_base + 8 * L.l_off[k], dptr[p]});
            vm = std::max(vm, m0[p]);
          }
          launch(7, (int64_t)na, push(rr), 0, 0, vm);
        }
        trtri(Ls, Xs, sz, 0);
        launch(4, (int64_t)na, push(c2));
      }
      std::unordered_map<int, int64_t> linv_of;
      for (size_t k = 0; k < na; ++k) linv_of[L.active[k]] = L.linv_off[k];
      if (!L.resc_blocks.empty()) {
        std::vector<Target> g1, g2;
        int64_t acc = 0, mask_bytes = 0;
        for (int b : L.resc_blocks) {
          const int i = bi[b], j = bj[b];
          Target t1;
          opnd(t1.c, temp_base + 8 * acc, i, j);
          opnd(t1.segs, fac_base + 8 * linv_of.at(i), i, i);
          opnd(t1.segs, pool_base + 8 * boff[b], i, j);
          t1.mm = m0[i];
          t1.nn = m0[j];
          g1.push_back(std::move(t1));
          Target t2;
          opnd(t2.c, pool_base + 8 * boff[b], i, j);
          opnd(t2.segs, temp_base + 8 * acc, i, j);
          opnd(t2.segs, fac_base + 8 * linv_of.at(j), j, j);
          t2.mm = m0[i];
          t2.nn = m0[j];
          g2.push_back(std::move(t2));
          acc += m0[i] * m0[j];
          mask_bytes += (m0[i] + 15) / 16;
        }
        // K-chunk masks of the unscaled blocks behind the products' temp
        const int64_t mask_addr = temp_base + 8 * acc;
        temp_size = std::max(temp_size, acc + (mask_bytes + 7) / 8 + 1);
        gemm(g1, 1.0, 0.0, 0, 0, 1, 0, mask_addr);   // T = Z_i^-1 B
        gemm(g2, 1.0, 0.0, 1, 0, 2);   // B = T Z_j^-T
      }
      // sparsify, wave by wave (factorize.py:323-340)
      for (int wv = 0; wv < L.nwaves; ++wv) {
        std::vector<size_t> pan;
        int64_t vm = 1;
        for (size_t k = 0; k < na; ++k)
          if (L.wave[k] == wv) {
            pan.push_back(k);
            vm = std::max(vm, m0[L.active[k]]);
          }
        int cap = std::max(1, spand_rrqr_capacity((int)vm));
        if (cap_override > 0) cap = std::min(cap, cap_override);
        // a wave of few large panels runs clustered: every panel gets whole
        // clusters of cs CTAs (one at least), so cap counts clusters
        int cs = 1;
        if (cluster_cs > 1 && cap_override <= 0 && vm >= cluster_min_rows &&
            vm <= spand_rrqr_max_rows_clustered(cluster_cs)) {
          int mn = (int)vm;
          for (size_t k : pan) mn = std::min<int>(mn, (int)m0[L.active[k]]);
          const int capc = spand_rrqr_cluster_capacity((int)vm, cluster_cs) / cluster_cs;
          if (mn >= cluster_min_rows && capc >= 1 && (int)pan.size() <= capc) {
            cs = cluster_cs;
            cap = capc;
          }
        }
        for (size_t c0 = 0; c0 < pan.size(); c0 += cap) {
          const size_t c1e = std::min(pan.size(), c0 + (size_t)cap);
          std::vector<int64_t> works;
          for (size_t u = c0; u < c1e; ++u) {
            const size_t k = pan[u];
            int64_t ncap = 0;
            for (int w : L.anbrs[k]) ncap += m0[w];
            const double mw = (double)m0[L.active[k]], nw = (double)std::max<int64_t>(ncap, 1);
            double wgt = mw * nw;                                   // 0: panel size
            if (group_weight == 1) wgt = mw * mw;                   // 1: rows^2 (step count x height)
            else if (group_weight == 2) wgt = mw * std::sqrt(mw * nw);
            else if (group_weight == 3) wgt = std::pow(mw, gexp_m) * std::pow(nw, gexp_n);
            works.push_back(std::max<int64_t>(1, (int64_t)wgt));
          }
          const std::vector<int> gs = groups(works, cap);
          std::vector<int64_t> prow, nrow, krow;
          int64_t need = 0, gbeg = 0, vmax = 1, colbeg = 0, qbeg = 0;
          for (size_t u = c0; u < c1e; ++u) {
            const size_t k = pan[u];
            const int p = L.active[k];
            const int g = gs[u - c0] * cs;
            int64_t ncap = 0;
            for (int w : L.anbrs[k]) ncap += m0[w];
            const int64_t mc = m0[p];
            // W | V | int lists (32 (ncap + mc)) | WY T blocks of Q (32 mc + 1024)
            const int64_t wsz =
                mc * std::max<int64_t>(ncap, 1) + mc * mc + 32 * (ncap + mc) + 32 * mc + 1024;
            const int64_t asz = 2 * ncap + 3 * mc + 68 * (int64_t)g + 8 + 1024;
            const int64_t isz = (3 * ncap + 1) / 2 + 1;
            const int64_t nb0 = (int64_t)nrow.size() / 4;
            for (int w : L.anbrs[k]) {
              if (w > p) nrow.insert(nrow.end(), {w, blk_ptr(p, w), 0, 0});
              else nrow.insert(nrow.end(), {w, blk_ptr(w, p), 1, 0});
            }
            const int64_t nb1 = (int64_t)nrow.size() / 4;
            int64_t qdst = fac_base + 8 * L.q_off[k], nkws = 0;
            if (nk) {
              // near-kernel: the RRQR writes q2 into the workspace, nk_qform
              // builds the Orthogonal op's factor in its fac slot
              nkws = temp_base + 8 * (need + wsz + asz + isz + 1);
              const int64_t q2 = nkws + 8 * (kNkHead + 2 * mc * nk);
              krow.insert(krow.end(), {p, nkws, q2, qdst, nb0, nb1, colbeg, qbeg, L.slot[k],
                                       dptr[p]});
              colbeg += ncap;
              qbeg += mc;
              qdst = q2;
            }
            // clustered: every CTA keeps the cluster's 4 column lists
            const int64_t lsz =
                cs > 1 ? (4 * (int64_t)g * (std::max<int64_t>(ncap, 1) / (g / cs) + 2) + 1) / 2 : 0;
            const int64_t lptr = cs > 1 ? temp_base + 8 * (need + wsz + asz + isz + 1 + nk_ws(mc)) : 0;
            prow.insert(prow.end(),
                        {p, nb0, nb1, temp_base + 8 * need, qdst,
                         temp_base + 8 * (need + wsz), temp_base + 8 * (need + wsz + asz), gbeg,
                         g, ctr_base + 8 * ctr_next, L.slot[k], ncap, mc, nkws, lptr, 0});
            ++ctr_next;
            need += wsz + asz + isz + 1 + nk_ws(mc) + lsz;
            gbeg += g;
            vmax = std::max(vmax, mc);
          }
          if (nrow.empty()) nrow.assign(4, 0);
          temp_size = std::max(temp_size, need);
          const int64_t a = push(prow), b = push(nrow);
          const int64_t np = (int64_t)(c1e - c0);
          int64_t kr = 0;
          if (nk) {
            kr = push(krow);
            launch(8, np, kr, b);                   // basis of u_p, rank r
            launch(9, np, kr, b, 0, colbeg, vmax);  // W <- rotate(H^T W)
          }
          launch(5, np, a, b, 0, gbeg, vmax, cs);
          if (nk) launch(10, np, kr, 0, 0, qbeg, vmax);   // Q = [U_perp q2_c, U, U_perp q2_f]
        }
      }
    }
  }
  void emit_final() {
    // final dense block (factorize.py:198-220); virtual cluster id = ncl
    if (!fin.empty()) {
      std::unordered_map<int, int> index;
      for (size_t k = 0; k < fin.size(); ++k) index[fin[k]] = (int)k;
      std::vector<int64_t> cl(fin.begin(), fin.end()), br;
      for (int b : fin_blocks)
        br.insert(br.end(), {index.at(bi[b]), index.at(bj[b]), pool_base + 8 * boff[b], 0});
      if (br.empty()) br.assign(4, 0);
      const int64_t a = push(cl), b = push(br);
      launch(6, (int64_t)fin.size(), a, b, 0, (int64_t)fin_blocks.size(), ncl, f_off);
      std::vector<std::vector<int64_t>> pops(1);
      opnd(pops[0], fac_base + 8 * f_off, ncl, ncl);
      potrf(pops, 0);
      std::vector<int64_t> l, x;
      opnd(l, fac_base + 8 * f_off, ncl, ncl);
      opnd(x, fac_base + 8 * flinv_off, ncl, ncl);
      trtri({l}, {x}, {fcap}, 0);
    }
  }
};


}  // namespace spand
