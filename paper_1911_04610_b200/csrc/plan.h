// plan.h -- static plan of the network on the GPU: shapes, partition, fused blocks, arena.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/xpipe.h"

namespace xp {

struct Shape {
  int c = 0, h = 0, w = 0;
  int64_t size() const { return (int64_t)c * h * w; }
};

struct LayerInfo {
  xpipe_layer d{};
  int src0 = -1, src1 = -1;
  Shape in0, in1, out;
  int stage = 0;
  int64_t nw_torch = 0, nb = 0;   // PyTorch-layout element counts (weight, bias)
  int64_t nw_gpu = 0;             // GPU-layout weight elements (conv: Cout*R*S*Cin_pad)
  int64_t woff = -1, boff = -1;   // offsets in the stage arena
  int cin_pad = 0;                // conv: input channels padded to a multiple of 8 (bf16)
};

// A fused execution unit of the GPU path:
//   BK_LINEAR : Linear [+ ReLU]                         (fp32 contract or bf16 operands)
//   BK_CONV   : Conv2d [+ BatchNorm2d] [+ ReLU] [+ MaxPool2d]   (bf16, tcgen05)
//   BK_XENT   : softmax cross-entropy on the logits
enum { BK_LINEAR = 1, BK_CONV = 2, BK_XENT = 3 };

struct Block {
  int kind = 0;
  int lmain = -1, lbn = -1, lrelu = -1, lpool = -1;
  Shape in, mid, out;      // mid = conv output before BN/ReLU/pool
  bool logits = false;     // output feeds the softmax-xent (kept fp32)
};

struct StagePlan {
  int l0 = 0, l1 = 0;
  std::vector<Block> blocks;
  int64_t P = 0;           // arena elements (multiple of 64)
  Shape in, out;           // stage input / output shapes
  size_t in_bytes = 0;     // gradient message bytes (n x in) / input slot bytes
  size_t in_slot_bytes = 0;
  size_t out_bytes = 0;    // activation message bytes (n x out)
  int64_t max_act = 0;     // max elements of any activation of the stage (per micro-batch)
};

struct NetPlan {
  std::vector<LayerInfo> layers;
  std::vector<StagePlan> stages;
};

int build_net_plan(const xpipe_layer* layers, int n_layers, int K, const xpipe_config& cfg, int n_micro,
                   NetPlan* out, std::string* err);
void gpu_to_torch_layout(const LayerInfo& L, int tensor, const float* gpu, float* torch);
void torch_to_gpu_layout(const LayerInfo& L, int tensor, const float* torch, float* gpu);

}  // namespace xp
