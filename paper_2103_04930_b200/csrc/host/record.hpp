// Per-cycle run records in the reference's report formats, so a B200 run can
// be fed to the reference tooling (`accelfwd-bench compare`, which reads
// records with proj/src/profiler.cpp read_cycle_csv):
//   * cycle CSV: "# key=value" metadata lines, then
//     index,gpu_s,communication_s,other_s,bytes_sent,bytes_received
//     (proj/src/profiler.cpp:88-110 write_cycle_csv; %.9f seconds)
//   * run summary markdown (proj/src/profiler.cpp:222-261)
// Cycle timing follows the reference client's decomposition
// (proj/src/client.cpp:160-195): gpu = min(server compute_s, wait),
// communication = send + (wait - gpu), other = the rest of the cycle.
#pragma once

#include <cstdint>
#include <ostream>
#include <string>
#include <vector>

namespace avec::record {

struct CycleTiming {
  double communication_s = 0;
  double gpu_s = 0;
  double other_s = 0;
  std::uint64_t bytes_sent = 0;
  std::uint64_t bytes_received = 0;
  double compute_s = 0;  // server-reported compute window (not a CSV column)
};

struct RunMeta {
  std::string label = "run";
  std::string mode = "offload";  // "native" | "offload" (profiler.hpp RunMode)
  std::string host = "host";
  std::string destination = "local";
  std::string workload;
  std::string model;
  double output_divisor = 0;
  double scale_factor = 1.0;
  std::string result_digest;
};

class RunRecord {
 public:
  explicit RunRecord(RunMeta meta) : meta_(std::move(meta)) {}
  void record(const CycleTiming& c);           // throws after finalize
  void finalize(double setup_s, double total_wall_s);
  const RunMeta& meta() const { return meta_; }
  const std::vector<CycleTiming>& cycles() const { return cycles_; }
  double setup_s() const { return setup_s_; }
  double total_wall_s() const { return total_wall_s_; }
  double processing_s() const { return total_wall_s_ - setup_s_; }
  std::uint64_t bytes_sent() const;
  std::uint64_t bytes_received() const;
  double gpu_s() const;
  double communication_s() const;
  double other_s() const;

 private:
  RunMeta meta_;
  std::vector<CycleTiming> cycles_;
  double setup_s_ = 0, total_wall_s_ = 0;
  bool finalized_ = false;
};

void write_cycle_csv(const RunRecord& r, std::ostream& out);
void write_summary_markdown(const RunRecord& r, std::ostream& out);

}  // namespace avec::record
