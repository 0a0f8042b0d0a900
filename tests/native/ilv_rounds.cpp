// Test harness (CPU): the round structure of K_ilv (kernels.cu, DESIGN.md V.2)
// without the arithmetic -- every stage runs its next op in a round once the
// op's input was produced in an earlier round -- to bound how far a producer
// runs ahead of the table position its consumer reads.  The kernel's rings
// hold Q >= P/2 + 2 entries per stage; ilv_max_lead(P, v, m) returns the
// largest (ops produced - position read) seen, or -1 on a deadlock.
#include <algorithm>
#include <cstdint>
#include <vector>

extern "C" int ilv_max_lead(int P, int v, int m) {
  const int64_t n = (int64_t)m * v, pv = (int64_t)P * v;
  std::vector<int64_t> p(P, 0), nf(P, 0), nb(P, 0);
  int lead = 0;
  for (;;) {
    bool act = false, ran = false;
    std::vector<int> run(P, 0), isf(P, 0);
    for (int s = 0; s < P; ++s) {
      if (p[s] >= 2 * n) continue;
      act = true;
      const int64_t w = std::min<int64_t>(2 * (P - 1 - s) + (int64_t)(v - 1) * P, n);
      const bool f = p[s] < w || (p[s] < 2 * n - w && !((p[s] - w) & 1));
      const int64_t idx = f ? nf[s] : nb[s];
      const int64_t rem = idx % pv, gi = idx / pv;
      const int k = f ? (int)(rem / P) : v - 1 - (int)(rem / P);
      int ps = -1;
      int64_t x = 0;
      bool fr = f;
      if (f) {
        if (s > 0) { ps = s - 1; x = idx; }
        else if (k > 0) { ps = P - 1; x = idx - P; }
      } else {
        if (s < P - 1) { ps = s + 1; x = idx; }
        else if (k < v - 1) { ps = 0; x = idx - P; }
        else { ps = s; fr = true; x = gi * pv + (int64_t)(v - 1) * P + rem % P; }
      }
      if (ps >= 0) {
        const int64_t have = fr ? nf[ps] : nb[ps];
        if (have <= x) continue;
        lead = std::max<int>(lead, (int)(have - x));
      }
      run[s] = 1;
      isf[s] = f;
      ran = true;
    }
    if (!act) break;
    if (!ran) return -1;
    for (int s = 0; s < P; ++s)
      if (run[s]) {
        if (isf[s]) ++nf[s]; else ++nb[s];
        ++p[s];
      }
  }
  return lead;
}
