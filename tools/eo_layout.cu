// Prints the folded kernel's compile-time layout per (p, q, precision): CTA size, elements per
// batch, tile geometry, qdata mode and shared memory (host only; nvcc tools/eo_layout.cu).
#include <cstdio>
#include "elas_apply_eo.cuh"
using namespace elas;
template <int P, int Q, typename T>
void show() {
  using L = LayEO<P, Q, T>;
  printf("p%d q%d %s NT=%d EB=%d RS=%d B=%d EL=%d RW=%d R=%d STAGE=%d smem=%zu (%.1f KB) cps=%d minb=%d\n", P, Q,
         sizeof(T) == 8 ? "f64" : "f32", L::NT, L::EB, L::RS, L::B, L::EL, L::RW, L::R, (int)L::STAGE, L::smem,
         L::smem / 1024.0, CpsEOT<P, T>::value, MinbEOT<P, T>::value);
}
#define BOTH(P) show<P, P + 1, double>(); show<P, P + 2, double>(); show<P, P + 1, float>(); show<P, P + 2, float>();
int main() { BOTH(1) BOTH(2) BOTH(3) BOTH(4) BOTH(5) BOTH(6) BOTH(7) BOTH(8) return 0; }
