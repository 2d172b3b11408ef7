// check_common.cuh — the fp64 SIMT building blocks shared by the check-mode kernels
// (check.cu) and the EB-GFN proposal kernel (eb.cu); both TUs are compiled with
// --fmad=false so the fp64 arithmetic follows the reference's operation order.
#pragma once

#include "engine.h"

namespace gfnx {
namespace {

struct DevLayout {
  int n_trunk, H, act_sz, A, O;
  int dims[10];
  int64_t off_w[10], off_b[10];
  int64_t off_fw, off_fb, off_flw, off_flb;
  int act_off[10];
};

DevLayout make_dev_layout(const Ctx& c) {
  DevLayout d{};
  d.n_trunk = c.L.n_trunk;
  d.H = c.L.H();
  d.A = c.shape.num_actions;
  d.O = c.shape.obs_dim;
  int o = 0;
  for (int l = 0; l <= c.L.n_trunk; ++l) d.dims[l] = c.L.dims[l];
  for (int l = 0; l < c.L.n_trunk; ++l) {
    d.off_w[l] = c.L.off_w[l];
    d.off_b[l] = c.L.off_b[l];
    d.act_off[l] = o;
    o += c.L.dims[l + 1];
  }
  d.act_sz = o;
  d.off_fw = c.L.off_fw;
  d.off_fb = c.L.off_fb;
  d.off_flw = c.L.off_flw;
  d.off_flb = c.L.off_flb;
  return d;
}

// z = matmul(h, W) + b (+ReLU), one output per thread, sequential over the input index
// exactly like matmul_acc (tensor.cpp:67-77) followed by the bias/ReLU loop (nn.cpp:64-74).
__device__ void dense_block(const double* h, int in, const double* W, const double* b, int out,
                            double* z, bool relu) {
  for (int j = threadIdx.x; j < out; j += blockDim.x) {
    double acc = 0.0;
    for (int p = 0; p < in; ++p) acc += h[p] * W[(size_t)p * out + j];
    acc += b[j];
    if (relu && acc < 0.0) acc = 0.0;
    z[j] = acc;
  }
}

}  // namespace
}  // namespace gfnx
