// nixie-b200 — MLFQ-driven workloads on the virtual clock.
// The engine itself is header-only (include/nixie_workload/workload_sim.hpp)
// so that it also compiles against the reference library for trace parity;
// this header is the product's entry point.
#pragma once

#include <string>

namespace nixie {

// Parses a workload (workload_sim.hpp grammar), runs it to its horizon on the
// virtual clock with reference-identical link timing, and returns the trace.
std::string run_workload_model(const std::string& text);

}  // namespace nixie
