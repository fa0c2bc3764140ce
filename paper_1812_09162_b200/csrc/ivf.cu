// ivf.cu -- placeholder translation unit; the IVF path lands here.
#include "common.cuh"
