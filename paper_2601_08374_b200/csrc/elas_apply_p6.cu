// Kernel instances for degree p = 6 (q = p+1 and p+2); see elas_apply.cuh.
#include "elas_apply.cuh"
ELAS_DEFINE_DEGREE(6)
