// Lorenz-96 tangent-linear / adjoint kernels (filled in with the c2 path).
#include "internal.h"
