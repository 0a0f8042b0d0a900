// Test harness (not product code): the product's register-resident 1F1B
// recurrence Pipe<P> (paper_2508_05370_b200/csrc/hsim_core.cuh), compiled for
// the host so its exact steady-regime acceleration (affine / cyclic jumps) can
// be checked against the CPU oracle's event-driven pipeline on many stress
// inputs without a GPU.  The GPU parity tests check the same code on device.
#include "../../paper_2508_05370_b200/csrc/hsim_core.cuh"

using namespace hsim;

template <int P>
static i64 run_p(i64 m, const i64* f, const i64* g, const i64* c, i64* skipped) {
  Pipe<P> p;
  for (int s = 0; s < P; ++s) {
    p.f[s] = (double)f[s];
    p.g[s] = (double)g[s];
    p.c[s] = s + 1 < P ? (double)(2 * c[s]) : 0.0;
  }
  return p.run(m, *skipped);
}

extern "C" i64 pipe_host_run(int P, i64 m, const i64* f, const i64* g, const i64* c, i64* skipped) {
  switch (P) {
#define C_(k) case k: return run_p<k>(m, f, g, c, skipped);
    C_(1) C_(2) C_(3) C_(4) C_(5) C_(6) C_(7) C_(8) C_(9) C_(10) C_(11) C_(12) C_(13) C_(14) C_(15) C_(16)
#undef C_
    default: return -1;
  }
}
