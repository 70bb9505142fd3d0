// TEST INFRASTRUCTURE ONLY (oracle/). The workload engine
// (include/nixie_workload/workload_sim.hpp, written against the `nixie`
// namespace API alone) instantiated over the UNMODIFIED reference: the
// include path puts /root/reference/proj/include first, so <nixie/mlfq.hpp>,
// <nixie/planner.hpp>, <nixie/transfer.hpp> and <nixie/mem_model.hpp> are the
// reference's and the link is oracle/_ref/libnixie_ref.a. Reference calls made
// by the engine: MlfqScheduler register_app / on_api_event / infer_all /
// select_next / is_idle / should_preempt / enqueue_request / clear_request /
// add_execution / on_grant_start / on_grant_end / victim_hint
// (proj/src/mlfq.cpp:51-225), plan_switch + MigrationPlan::dump
// (proj/src/planner.cpp:18-25, 111-216), execute (proj/src/transfer.cpp:250-271),
// MemState allocate / audit (proj/src/mem_model.cpp:48-86, 274-325).
//
// Usage: ref_workload <workload-file | ->
#include <nixie_workload/workload_sim.hpp>

#include <fstream>
#include <iostream>
#include <sstream>

int main(int argc, char** argv) {
  try {
    std::stringstream ss;
    if (argc < 2 || std::string(argv[1]) == "-") {
      ss << std::cin.rdbuf();
    } else {
      std::ifstream f(argv[1]);
      if (!f) {
        std::cerr << "cannot open " << argv[1] << "\n";
        return 2;
      }
      ss << f.rdbuf();
    }
    const nixie::workload::Spec spec = nixie::workload::parse(ss.str());
    nixie::MemState mem;
    spec.hw.apply_to(mem);
    nixie::workload::Engine eng(spec, mem);
    std::cout << eng.run().trace;
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "ref_workload: " << e.what() << "\n";
    return 1;
  }
}
