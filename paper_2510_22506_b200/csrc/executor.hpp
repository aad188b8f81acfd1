// Device-side executor interface used by the planner.  The CUDA
// implementation lives in fctn_ctx.cu; the planner only sees buffer ids.
#pragma once

#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace fctn {

class Executor {
 public:
  virtual ~Executor() {}
  // a buffer for a tensor with these labels (extents: the executor's own,
  // possibly sharded, shape)
  virtual int64_t alloc_labels(const std::vector<int>& labels) = 0;
  virtual void free(int64_t buf) = 0;
  virtual bool is_fixed_buffer(int64_t buf) const = 0;
  virtual void contract(const ContractOp& op) = 0;
  virtual void permute(const LTensor& in, const LTensor& out) = 0;
};

}  // namespace fctn
