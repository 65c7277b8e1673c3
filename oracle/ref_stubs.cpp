// TEST INFRASTRUCTURE (oracle/_ref build only).
//
// Link stubs for the reverse-mode tape (proj/include/vqnqs/autodiff.hpp:39-100).
// proj/src/model.cpp references ad::Graph from its training-graph builders
// (model.cpp:531-640), which are OUT OF SCOPE for the local-energy path
// (autodiff is training/backward). autodiff.cpp itself needs far
// more of Eigen than the hot path does, so instead of compiling it we satisfy
// the linker with stubs that fail loudly if anything ever reaches them. The
// evaluation paths (log_prob_batch, dedup_log_prob, local_energy_batch) never
// touch ad::Graph; ad::Parameter is header-only.
#include <stdexcept>

#include "vqnqs/autodiff.hpp"

namespace vqnqs::ad {

namespace {
[[noreturn]] void no_tape() {
  throw CapabilityError("oracle/_ref: training tape not built (out of scope)");
}
}  // namespace

Graph::Id Graph::constant(Tensor) { no_tape(); }
Graph::Id Graph::param(Parameter&) { no_tape(); }
Graph::Id Graph::linear(Id, Id, Id) { no_tape(); }
Graph::Id Graph::layer_norm(Id, Id, Id, double) { no_tape(); }
Graph::Id Graph::log_softmax_rows(Id) { no_tape(); }
Graph::Id Graph::gelu(Id) { no_tape(); }
Graph::Id Graph::add(Id, Id) { no_tape(); }
Graph::Id Graph::attention(Id, Id, Id, int64_t, int64_t, int, Mask) { no_tape(); }
Graph::Id Graph::embedding(Parameter&, const std::vector<int>&) { no_tape(); }
Graph::Id Graph::mean_pool_seq(Id, int64_t, int64_t) { no_tape(); }
Graph::Id Graph::pick_sum_per_seq(Id, const std::vector<int>&, int64_t, int64_t) {
  no_tape();
}
Graph::Id Graph::vq_quantize(Id, Parameter&, const VqOptions&, std::vector<int>*) {
  no_tape();
}

}  // namespace vqnqs::ad
