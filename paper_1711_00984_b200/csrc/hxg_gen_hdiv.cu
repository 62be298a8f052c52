// Specialized kernels of space HDIV (isotropic p = 1..10): general path (L = p + 1),
// constant-Jacobian path and extrusion path.  The launcher body is shared by the
// four spaces (hxg_gen_body.cuh); one translation unit per space keeps the builds parallel.
#include "hxg_gen_body.cuh"

HXG_GEN_DEFINE_LAUNCHERS(hxg::HDIV, hdiv)
