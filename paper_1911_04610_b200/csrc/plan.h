// plan.h -- static plan of the network on the GPU: shapes, partition, fused ops, tensors, arena.
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
  int cin_pad = 0;                // conv: input channel stride (Cin padded to 8 on stage 0's input)
};

// A fused execution unit of the GPU path (one stage = a DAG of ops in layer order):
//   OP_CONV    : Conv2d + BatchNorm2d [+ ReLU] [+ MaxPool2d]         (bf16, tcgen05)
//                or, with in1 >= 0, Conv2d + BatchNorm2d + residual Add (in1) [+ ReLU]: the
//                Add that follows a bias-free, activation-free conv block is folded into the
//                BN-apply (the ResNet bottleneck's last conv or its downsample branch)
//   OP_LINEAR  : Linear [+ ReLU]                                      (fp32 contract or bf16)
//   OP_ADD     : residual add [+ ReLU]
//   OP_CONCAT  : channel concat of two tensors (removed from the plan when both inputs can be
//                written in place: their producers then store into the concat output at their
//                channel offset, and their backward reads the gradient slice, see TensorInfo)
//   OP_MAXPOOL / OP_AVGPOOL : standalone pooling;  OP_GAP : global average pool
//   OP_XENT    : softmax cross-entropy on the logits
enum { OP_LINEAR = 1, OP_CONV, OP_XENT, OP_ADD, OP_CONCAT, OP_MAXPOOL, OP_AVGPOOL, OP_GAP };

struct Op {
  int kind = 0;
  int lmain = -1, lbn = -1, lrelu = -1, lpool = -1;
  int ladd = -1;            // OP_CONV with a folded residual Add: the Add layer (in1 = residual)
  int in0 = -1, in1 = -1;   // input tensor ids (0 = the stage input)
  int out = -1;             // output tensor id (stashed per micro-batch)
  Shape sin0, sin1, smid, sout;
  bool relu = false;
  bool logits = false;      // output feeds the softmax-xent (kept fp32)
};

struct TensorInfo {
  Shape shape;
  int es = 2;               // bytes per element (bf16 activations, fp32 logits / fp32 path)
  int producer = -1;        // op index (-1 = stage input, -2 = unused)
  int consumers = 0;
  // channel-offset view (a concat input written in place): the tensor is channels
  // [coff, coff + shape.c) of tensor `alias`, rows of pitch() elements; no buffers of its own
  int alias = -1, coff = 0, base_c = 0;
  int pitch() const { return alias >= 0 ? base_c : shape.c; }
};

struct StagePlan {
  int l0 = 0, l1 = 0;
  std::vector<Op> ops;
  std::vector<TensorInfo> tensors;   // [0] = stage input
  int out_tensor = 0;                // the stage output (message to the next stage / logits)
  int64_t P = 0;                     // arena elements (multiple of 64)
  Shape in, out;
  size_t in_bytes = 0;               // gradient message bytes (n x in)
  size_t in_slot_bytes = 0;          // input ring slot bytes (stage 0: channel-padded bf16)
  size_t out_bytes = 0;              // activation message bytes (n x out)
  int64_t max_act = 0;               // max elements of any activation of the stage (per micro-batch)
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
