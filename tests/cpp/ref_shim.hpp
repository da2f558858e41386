// Force-included (-include) when test programs compile the reference's
// policy.hpp: policy.hpp:145,246 pass std::vector<bool> to
// softmax_masked(span<const double>, span<const bool>) (nn.hpp:207-208), a
// hard error under g++ 13. This overload forwards to the
// reference's own function; oracle/ref_capi.cpp carries the same shim.
#pragma once
#include <memory>
#include <span>
#include <vector>

#include "shardplan/nn.hpp"

namespace shardplan {
inline std::vector<double> softmax_masked(std::span<const double> logits,
                                          const std::vector<bool>& mask) {
  std::unique_ptr<bool[]> m(new bool[mask.size()]);
  for (std::size_t i = 0; i < mask.size(); ++i) m[i] = mask[i];
  return softmax_masked(logits, std::span<const bool>(m.get(), mask.size()));
}
}  // namespace shardplan
