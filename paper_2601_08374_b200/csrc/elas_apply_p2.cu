// Kernel instances for degree p = 2 (q = p+1 and p+2); see elas_apply.cuh.
#include "elas_apply.cuh"
ELAS_DEFINE_DEGREE(2)
