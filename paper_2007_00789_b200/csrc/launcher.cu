// Native launcher of the factorization program (engine.py used to issue the
// ~10k launch records of a C4-L15 factorization one ctypes call at a time,
// ~5 us of host time each, which left the device idle on the leaf levels).
// Record layout (16 int64, csrc/planner.h launch()): {type, count, a, b, c,
// x0, x1, x2, alpha bits, beta bits, compact, ...}; a / b / c are offsets of
// the record's rows in the uploaded program (int64 units from `base`).
#include <cstring>
#include <vector>

#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {
// CUDA-event timing of selected launch types (profile of the timed region)
struct Timer {
  std::vector<cudaEvent_t> ev;
  std::vector<int> type;
  size_t used = 0;
};
Timer g_timer;

cudaEvent_t timer_event() {
  const size_t k = g_timer.used++;
  if (k >= g_timer.ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_timer.ev.push_back(e);
  }
  return g_timer.ev[k];
}
}  // namespace

extern "C" {

int spand_run_launches(int nl, const int64_t* recs, int64_t base, int32_t* m0, int32_t* off,
                       int32_t* info, int64_t* events, int64_t fac_base, const int64_t* btab,
                       double eps, int rrqr_flags, double* U, int64_t ldu, int nkv,
                       double nk_rtol, int time_mask, int64_t* counts, void* stream) {
  auto P = [&](int64_t o) { return reinterpret_cast<const int64_t*>(base + 8 * o); };
  auto PM = [&](int64_t o) { return reinterpret_cast<int64_t*>(base + 8 * o); };
  for (int i = 0; i < nl; ++i) {
    const int64_t* r = recs + 16 * (int64_t)i;
    const int typ = (int)r[0];
    const int cnt = (int)r[1];
    const int64_t ao = r[2], bo = r[3], co = r[4], x0 = r[5], x1 = r[6], x2 = r[7];
    const bool timed = typ >= 0 && typ < 32 && ((time_mask >> typ) & 1);
    if (timed) {
      g_timer.type.push_back(typ);
      cudaEventRecord(timer_event(), (cudaStream_t)stream);
    }
    int st = 0;
    switch (typ) {
      case 1:
        st = spand_potrf_batched(cnt, P(ao), m0, off, info, (int)x0, (int)x1, stream);
        break;
      case 2:
        st = spand_trtri_tiles(cnt, P(ao), m0, off, stream);
        break;
      case 3: {
        double alpha, beta;
        std::memcpy(&alpha, r + 8, 8);
        std::memcpy(&beta, r + 9, 8);
        // fields 11 / 12: K-chunk masks (device address; offsets row relative
        // to the targets row), written by the type-12 record just before
        st = spand_gemm_grouped_masked(cnt, P(ao), P(bo), P(co), m0, off, alpha, beta, (int)x0,
                                       (int)x1, (int)x2, btab, (int)r[10],
                                       reinterpret_cast<const unsigned char*>(r[11]),
                                       r[11] ? P(bo + r[12]) : nullptr, stream);
        break;
      }
      case 12:
        st = spand_gemm_kmask(cnt, P(ao), P(bo), m0, off, reinterpret_cast<unsigned char*>(x0),
                              P(co), (int)x1, stream);
        break;
      case 4:
        st = spand_copy_batched(cnt, P(ao), m0, off, stream);
        break;
      case 5:
        if (x2 > 1)
          st = spand_rrqr_wave_clustered(cnt, (int)x0, (int)x1, (int)x2, P(ao), P(bo), m0, off, eps,
                                         rrqr_flags, events, stream);
        else
          st = spand_rrqr_wave(cnt, (int)x0, (int)x1, P(ao), P(bo), m0, off, eps, rrqr_flags, events,
                               stream);
        break;
      case 6:
        st = spand_assemble_final(cnt, P(ao), x0, P(bo), m0, off, (int32_t)x1,
                                  reinterpret_cast<double*>(fac_base + 8 * x2), stream);
        break;
      case 7:
        st = spand_nk_rescale(cnt, P(ao), m0, off, U, ldu, nkv, (int)x0, stream);
        break;
      case 8:
        st = spand_nk_basis(cnt, P(ao), P(bo), m0, off, U, ldu, nkv, nk_rtol, stream);
        break;
      case 9:
        st = spand_nk_deflate(cnt, x0, P(ao), P(bo), m0, off, (int)x1, stream);
        break;
      case 10:
        st = spand_nk_qform(cnt, x0, P(ao), events, (int)x1, stream);
        break;
      case 11:
        st = spand_digest_pieces(cnt, P(ao), m0, off, stream);
        break;
      default:
        st = -100;
    }
    (void)PM;
    if (timed) cudaEventRecord(timer_event(), (cudaStream_t)stream);
    if (st != 0) return st > 0 ? st : -(1000 * (i + 1)) + st;
    if (counts && typ >= 0 && typ < 16) ++counts[typ];
  }
  return 0;
}

// launch timing: reset before a run; read after the stream is synchronized
// (ms summed per type into ms[32] and the launch count into n[32])
int spand_launch_timer_reset(void) {
  g_timer.used = 0;
  g_timer.type.clear();
  return 0;
}

int spand_launch_timer_read(double* ms, int64_t* n) {
  for (int t = 0; t < 32; ++t) {
    ms[t] = 0.0;
    n[t] = 0;
  }
  for (size_t k = 0; k < g_timer.type.size(); ++k) {
    float v = 0.f;
    cudaEventSynchronize(g_timer.ev[2 * k + 1]);
    cudaEventElapsedTime(&v, g_timer.ev[2 * k], g_timer.ev[2 * k + 1]);
    ms[g_timer.type[k]] += v;
    ++n[g_timer.type[k]];
  }
  g_timer.used = 0;
  g_timer.type.clear();
  return 0;
}

}  // extern "C"
