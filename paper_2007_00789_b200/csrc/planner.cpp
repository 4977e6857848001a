// Native level scheduler of the device factorization (host C++).
//
// Restates the block-structure evolution of the reference driver
// (/root/reference/pkg/src/spdkit/factorize.py: EliminationState :51-239,
// factorize :285-366) symbolically -- the structure does not depend on the
// ranks the sparsification finds, only the live sizes do, and those are
// read on the device -- and emits the whole numeric factorization as a flat
// PROGRAM: operand / tile / segment / panel rows for every batched launch
// plus a launch list.  The Python host uploads the program once and walks
// the launch list; no per-level host planning remains on the critical path.
//
// Launch record (16 x int64):
//   [0] type  [1] count  [2] a_off  [3] b_off  [4] c_off  [5] x0  [6] x1
//   [7] x2  [8] bits(alpha)  [9] bits(beta)  [10..15] 0
// types: 1 potrf(a=ops, x0=info index)  2 trtri tiles(a=ops)
//        3 gemm(a=tiles, b=targets, c=segs, x0=bT, x1=lower_only, alpha, beta)
//          (tile rows are packed: target << 32 | (i0 / 64) << 16 | (j0 / 64))
//        4 copy(a=ops)  5 rrqr wave(a=panels, b=nbrs, x0=grid, x1=vmax)
//        6 assemble final(a=cluster ids, b=block rows, x0=nblk, x1=final id,
//          x2=fac offset of the dense block)
//        near-kernel extension (nearkernel.cu): 7 rescale(a=rows, x0=vmax)
//        8 basis(a=nk rows, b=nbrs)  9 deflate(a, b, x0=grid, x1=vmax)
//        10 qform(a=nk rows, x0=grid, x1=vmax)
//        11 trailing-matrix digest pieces (a=rows of 6, count=pieces)
// Offsets are in int64 units into the program array.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

extern "C" int spand_rrqr_capacity(int vmax);

#include "planner.h"

using spand::Plan;

extern "C" {

void* spand_plan_create(int ncl, const int64_t* m0, const int32_t* depth, int levels, int skip,
                        int64_t npairs, const int64_t* pairs, int cap_override) {
  Plan* p = new Plan();
  p->ncl = ncl;
  p->levels = levels;
  p->skip = skip;
  p->cap_override = cap_override;
  p->m0.assign(m0, m0 + ncl);
  p->depth.assign(depth, depth + ncl);
  p->symbolic(npairs, pairs);
  p->layout();
  return p;
}

void spand_plan_destroy(void* h) { delete static_cast<Plan*>(h); }

// Cluster-pair keys (ci * ncl + cj, ci <= cj, ascending, unique) of the
// nonzeros of A: the initial blocks of the symbolic elimination
// (factorize.py:61-96).  cdofs/cptr: cluster dofs concatenated in id order.
// out must hold nnz entries; returns the number of keys.
int64_t spand_plan_pairs(int ncl, const int64_t* row_ptr, const int64_t* col_idx,
                         const int64_t* cluster_of, const int64_t* cdofs, const int64_t* cptr,
                         int64_t* out) {
  std::vector<int> stamp(ncl, -1), list;
  int64_t cnt = 0;
  for (int ci = 0; ci < ncl; ++ci) {
    list.clear();
    for (int64_t u = cptr[ci]; u < cptr[ci + 1]; ++u) {
      const int64_t r = cdofs[u];
      for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
        const int cj = (int)cluster_of[col_idx[e]];
        if (cj >= ci && stamp[cj] != ci) {
          stamp[cj] = ci;
          list.push_back(cj);
        }
      }
    }
    std::sort(list.begin(), list.end());
    for (int cj : list) out[cnt++] = (int64_t)ci * ncl + cj;
  }
  return cnt;
}

// Pool positions of A's entries (factorize.py:61-96, the initial blocks):
// where[e] for CSR entry e = (r, c) with cluster(r) <= cluster(c) is the
// column-major offset of (slot(r), slot(c)) inside block (cluster(r),
// cluster(c)); -1 for the other triangle.  Needs spand_plan_set_dofs.
int spand_plan_scatter(void* h, const int64_t* row_ptr, const int64_t* col_idx,
                       const int64_t* cluster_of, int64_t* where) {
  Plan* p = static_cast<Plan*>(h);
  const int ncl = p->ncl;
  const int64_t n = p->dptr[ncl];
  std::vector<int64_t> slot(n);
  for (int c = 0; c < ncl; ++c)
    for (int64_t u = p->dptr[c]; u < p->dptr[c + 1]; ++u) slot[p->dofs[u]] = u - p->dptr[c];
  std::vector<int> stamp(ncl, -1);
  std::vector<int64_t> base(ncl, 0);
  for (int ci = 0; ci < ncl; ++ci) {
    for (int64_t u = p->dptr[ci]; u < p->dptr[ci + 1]; ++u) {
      const int64_t r = p->dofs[u];
      for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
        const int64_t c = col_idx[e];
        const int cj = (int)cluster_of[c];
        if (cj < ci) {
          where[e] = -1;
          continue;
        }
        if (stamp[cj] != ci) {
          stamp[cj] = ci;
          const int b = p->block(ci, cj);
          if (b < 0) return -1;
          base[cj] = p->boff[b];
        }
        where[e] = base[cj] + slot[r] + slot[c] * p->m0[ci];
      }
    }
  }
  return 0;
}

// RRQR group-size weighting (tuning): 0 ~ m n, 1 ~ m^2, 2 ~ m sqrt(m n)
int spand_plan_set_group_weight(void* h, int w, double em, double en) {
  Plan* p = static_cast<Plan*>(h);
  p->group_weight = w;
  p->gexp_m = em;
  p->gexp_n = en;
  return 0;
}

// clustered RRQR waves: cluster size (0 or 1 = off; 2, 4, 8) and the
// smallest panel height of a clustered wave
int spand_plan_set_cluster(void* h, int cs, int min_rows) {
  Plan* p = static_cast<Plan*>(h);
  if (cs < 0 || cs > 8 || (cs > 1 && (cs & (cs - 1)))) return -1;
  p->cluster_cs = cs;
  p->cluster_min_rows = min_rows;
  p->layout();   // the workspace bound depends on it
  return 0;
}

// near-kernel extension: number of vectors (0 = reference path); resizes
// the workspace bound, so call before spand_plan_sizes / emission
int spand_plan_set_nk(void* h, int k) {
  Plan* p = static_cast<Plan*>(h);
  if (k < 0 || k > 16) return -1;
  p->nk = k;
  p->layout();
  return 0;
}

// Trailing-matrix digests on (1) / off (0); out_base is the device address
// of dig_records x {i, j, rows, cols, h} int64 records (zeroed by the
// caller).  Returns the record count; counts[nlevels + 1] (may be null)
// receives the first record index of each level.
int64_t spand_plan_set_digest(void* h, int on, int64_t out_base, int64_t* counts) {
  Plan* p = static_cast<Plan*>(h);
  p->digest = on != 0;
  p->dig_base = out_base;
  if (!p->digest) return 0;
  if (p->dig_first.empty()) p->prepare_digest();
  if (counts) std::memcpy(counts, p->dig_first.data(), p->dig_first.size() * sizeof(int64_t));
  return p->dig_records;
}

// cluster dofs (original numbering) concatenated in id order, dptr[ncl+1]
int spand_plan_set_dofs(void* h, const int64_t* dofs, const int64_t* dptr) {
  Plan* p = static_cast<Plan*>(h);
  p->dptr.assign(dptr, dptr + p->ncl + 1);
  p->dofs.assign(dofs, dofs + p->dptr[p->ncl]);
  return 0;
}

// out[16]: pool_size, fac_size, temp_size, n_events, n_info, n_ctr, nblocks,
// nlevels, fcap, f_off, flinv_off, nfinal, prog_len, n_launch, meta_len,
// temp_bound (workspace upper bound known before emission)
int spand_plan_sizes(void* h, int64_t* out) {
  Plan* p = static_cast<Plan*>(h);
  int64_t meta = 9 + 3 * (int64_t)p->bi.size() + p->ncl + (int64_t)p->fin.size() +
                 (int64_t)p->fin_blocks.size();
  for (auto& L : p->lv) {
    meta += 5;
    for (size_t k = 0; k < L.interiors.size(); ++k) meta += 2 + (int64_t)L.inbrs[k].size();
    for (size_t k = 0; k < L.active.size(); ++k) meta += 7 + (int64_t)L.anbrs[k].size();
  }
  const int64_t v[16] = {p->pool_size, p->fac_size, p->temp_size, p->n_events, p->n_info,
                         p->n_events, (int64_t)p->bi.size(), (int64_t)p->lv.size(), p->fcap,
                         p->f_off, p->flinv_off, (int64_t)p->fin.size(), (int64_t)p->prog.size(),
                         (int64_t)p->launches.size() / 16, meta, p->temp_bound};
  std::memcpy(out, v, sizeof(v));
  return 0;
}

// Build the program for the given device base addresses.  A dry call only
// sizes the temporary workspace (spand_plan_sizes); then emit for real.
int spand_plan_emit(void* h, int64_t pool_base, int64_t fac_base, int64_t temp_base,
                    int64_t ctr_base, int dry) {
  Plan* p = static_cast<Plan*>(h);
  p->dry = dry != 0;
  p->pool_base = pool_base;
  p->fac_base = fac_base;
  p->temp_base = temp_base;
  p->ctr_base = ctr_base;
  p->emit();
  return 0;
}

// Incremental emission: begin, then next() until it returns 0; after each
// next(), chunk_sizes gives {chunk program length, chunk launch count} and
// chunk() copies them with program offsets RELATIVE to the chunk start.
int spand_plan_emit_begin(void* h, int64_t pool_base, int64_t fac_base, int64_t temp_base,
                          int64_t ctr_base) {
  Plan* p = static_cast<Plan*>(h);
  p->dry = false;
  p->pool_base = pool_base;
  p->fac_base = fac_base;
  p->temp_base = temp_base;
  p->ctr_base = ctr_base;
  p->emit_begin();
  return 0;
}

int spand_plan_emit_next(void* h, int64_t* chunk_sizes) {
  Plan* p = static_cast<Plan*>(h);
  const bool more = p->emit_next();
  chunk_sizes[0] = (int64_t)(p->prog.size() - p->chunk_prog0);
  chunk_sizes[1] = (int64_t)(p->launches.size() - p->chunk_launch0) / 16;
  chunk_sizes[2] = p->temp_size;
  return more ? 1 : 0;
}

int spand_plan_chunk(void* h, int64_t* prog, int64_t* launches) {
  Plan* p = static_cast<Plan*>(h);
  const int64_t base = (int64_t)p->chunk_prog0;
  std::memcpy(prog, p->prog.data() + base, (p->prog.size() - base) * sizeof(int64_t));
  const size_t l0 = p->chunk_launch0;
  for (size_t r = l0; r < p->launches.size(); r += 16) {
    int64_t* o = launches + (r - l0);
    std::memcpy(o, p->launches.data() + r, 16 * sizeof(int64_t));
    // program offsets a, b, c (fields 2..4) become chunk-relative
    for (int f = 2; f <= 4; ++f) o[f] -= base;
  }
  return 0;
}

int spand_plan_program(void* h, int64_t* prog, int64_t* launches) {
  Plan* p = static_cast<Plan*>(h);
  std::memcpy(prog, p->prog.data(), p->prog.size() * sizeof(int64_t));
  std::memcpy(launches, p->launches.data(), p->launches.size() * sizeof(int64_t));
  return 0;
}

// Structure for the host-side operator assembly (see engine.py for the
// decoder): header {ncl, nblocks, nlevels, nfinal, nfinblocks, fcap, f_off,
// flinv_off, n_events}, bi[], bj[], boff[], elim_linv[ncl], then per level
// {level, skipped, n_int, n_act, nwaves} + per interior {s, nnb, nbrs...}
// + per active {p, wave, l_off, linv_off, q_off, slot, nnb, nbrs...},
// then fin[], fin_blocks[].
int spand_plan_meta(void* h, int64_t* out) {
  Plan* p = static_cast<Plan*>(h);
  int64_t* o = out;
  const int64_t hdr[9] = {p->ncl, (int64_t)p->bi.size(), (int64_t)p->lv.size(),
                          (int64_t)p->fin.size(), (int64_t)p->fin_blocks.size(), p->fcap,
                          p->f_off, p->flinv_off, p->n_events};
  for (int k = 0; k < 9; ++k) *o++ = hdr[k];
  for (auto x : p->bi) *o++ = x;
  for (auto x : p->bj) *o++ = x;
  for (auto x : p->boff) *o++ = x;
  for (auto x : p->elim_linv) *o++ = x;
  for (auto& L : p->lv) {
    *o++ = L.level;
    *o++ = L.skipped;
    *o++ = (int64_t)L.interiors.size();
    *o++ = (int64_t)L.active.size();
    *o++ = L.nwaves;
    for (size_t k = 0; k < L.interiors.size(); ++k) {
      *o++ = L.interiors[k];
      *o++ = (int64_t)L.inbrs[k].size();
      for (int w : L.inbrs[k]) *o++ = w;
    }
    for (size_t k = 0; k < L.active.size(); ++k) {
      *o++ = L.active[k];
      *o++ = L.wave[k];
      *o++ = L.l_off[k];
      *o++ = L.linv_off[k];
      *o++ = L.q_off[k];
      *o++ = L.slot[k];
      *o++ = (int64_t)L.anbrs[k].size();
      for (int w : L.anbrs[k]) *o++ = w;
    }
  }
  for (int c : p->fin) *o++ = c;
  for (int b : p->fin_blocks) *o++ = b;
  return 0;
}

}  // extern "C"
