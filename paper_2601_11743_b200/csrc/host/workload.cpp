// The workload engine (include/nixie_workload/workload_sim.hpp) instantiated
// over this library: run_workload_model() is the product-side trace whose
// reference twin is oracle/ref_workload (same engine, reference headers and
// library).
#include "nixie/workload.hpp"

#include <nixie_workload/workload_sim.hpp>

namespace nixie {

std::string run_workload_model(const std::string& text) {
  const workload::Spec spec = workload::parse(text);
  MemState mem;
  spec.hw.apply_to(mem);
  workload::Engine eng(spec, mem);
  return eng.run().trace;
}

}  // namespace nixie
