// k_plane3.cu — the 3D instantiations of the plane kernels (k_plane.cu), compiled separately
// so that the two instantiation sets build in parallel.
#define SBK_PLANE_3D 1
#include "k_plane.cu"
