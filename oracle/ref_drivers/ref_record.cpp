// Reads a run-record CSV with the REFERENCE's parser (accelfwd::prof::
// read_cycle_csv, proj/src/profiler.cpp:148-220), checks the time
// decomposition (decomposition_holds, profiler.cpp:17-21), and prints the
// reference's own summary markdown (write_summary_markdown) to stdout, then a
// final JSON status line. TEST INFRASTRUCTURE ONLY: used to show that records
// written by avec-loadgen are consumable by the reference tooling.
#include <fstream>
#include <iostream>
#include <sstream>

#include "accelfwd/error.hpp"
#include "accelfwd/profiler.hpp"
#include "ref_common.hpp"

using namespace accelfwd;

int main(int argc, char** argv) {
  try {
    auto a = refdrv::parse_args(argc, argv);
    std::ifstream in(refdrv::get(a, "csv", "record.csv"));
    if (!in) throw std::runtime_error("cannot open csv");
    prof::RunRecord rec = prof::read_cycle_csv(in);
    const double tol = std::stod(refdrv::get(a, "tol", "0.01"));
    const bool holds = prof::decomposition_holds(rec.breakdown(), tol);
    std::ostringstream md;
    prof::write_summary_markdown(rec, nullptr, md);
    std::cout << md.str();
    std::printf("{\"ok\": true, \"frames\": %zu, \"decomposition_holds\": %s, \"bytes_sent\": %llu, "
                "\"bytes_received\": %llu}\n",
                rec.frame_count(), holds ? "true" : "false",
                static_cast<unsigned long long>(rec.bytes_sent()),
                static_cast<unsigned long long>(rec.bytes_received()));
    return 0;
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
}
