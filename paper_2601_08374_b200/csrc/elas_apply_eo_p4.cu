// Folded-SIMT kernel instances for degree p = 4 (q = p+1 and p+2); see elas_apply_eo.cuh.
#include "elas_apply_fg.cuh"
ELAS_DEFINE_DEGREE_EO(4)
