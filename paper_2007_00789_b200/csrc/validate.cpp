// Input validation of a symmetric CSR matrix (host C++), the checks of the
// reference SparseSymMatrix constructor (/root/reference/pkg/src/spdkit/
// sparse.py:40-58) after the O(n) shape checks done in Python: one pass per
// property so the FIRST failing property is reported, as in the reference.
#include <algorithm>
#include <cstdint>

extern "C" {

// returns 0 ok, 1 column out of range, 2 columns not strictly increasing,
// 3 pattern or values not symmetric, 4 missing / nonpositive diagonal
int spand_csr_check(int64_t n, const int64_t* rp, const int64_t* ci, const double* va) {
  const int64_t nnz = rp[n];
  for (int64_t e = 0; e < nnz; ++e)
    if (ci[e] < 0 || ci[e] >= n) return 1;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t e = rp[r] + 1; e < rp[r + 1]; ++e)
      if (ci[e] <= ci[e - 1]) return 2;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int64_t c = ci[e];
      const int64_t* b = ci + rp[c];
      const int64_t* f = ci + rp[c + 1];
      const int64_t* it = std::lower_bound(b, f, r);
      // the reference compares values, (csr != csr.T).nnz: a stored zero
      // whose mirror is not stored equals the implicit zero there
      if (it == f || *it != r) {
        if (va[e] == 0.0) continue;
        return 3;
      }
      if (!(va[it - ci] == va[e])) return 3;
    }
  for (int64_t r = 0; r < n; ++r) {
    const int64_t* b = ci + rp[r];
    const int64_t* f = ci + rp[r + 1];
    const int64_t* it = std::lower_bound(b, f, r);
    if (it == f || *it != r || !(va[it - ci] > 0.0)) return 4;
  }
  return 0;
}

}  // extern "C"
