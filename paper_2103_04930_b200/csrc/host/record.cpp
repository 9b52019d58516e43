#include "record.hpp"

#include <cstdio>
#include <stdexcept>

namespace avec::record {

void RunRecord::record(const CycleTiming& c) {
  if (finalized_) throw std::logic_error("record after finalize");
  cycles_.push_back(c);
}

void RunRecord::finalize(double setup_s, double total_wall_s) {
  if (finalized_) throw std::logic_error("finalize called twice");
  if (setup_s < 0 || total_wall_s < 0) throw std::invalid_argument("negative time on finalize");
  setup_s_ = setup_s;
  total_wall_s_ = total_wall_s;
  finalized_ = true;
}

// sums accumulate in recording order, like the reference's running totals
std::uint64_t RunRecord::bytes_sent() const {
  std::uint64_t s = 0;
  for (const auto& c : cycles_) s += c.bytes_sent;
  return s;
}
std::uint64_t RunRecord::bytes_received() const {
  std::uint64_t s = 0;
  for (const auto& c : cycles_) s += c.bytes_received;
  return s;
}
double RunRecord::gpu_s() const {
  double s = 0;
  for (const auto& c : cycles_) s += c.gpu_s;
  return s;
}
double RunRecord::communication_s() const {
  double s = 0;
  for (const auto& c : cycles_) s += c.communication_s;
  return s;
}
double RunRecord::other_s() const {
  double s = 0;
  for (const auto& c : cycles_) s += c.other_s;
  return s;
}

namespace {

std::string f9(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.9f", v);
  return b;
}

std::string f3(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.3f", v);
  return b;
}

}  // namespace

void write_cycle_csv(const RunRecord& r, std::ostream& out) {
  const RunMeta& m = r.meta();
  const std::pair<const char*, std::string> meta[] = {
      {"label", m.label},
      {"mode", m.mode},
      {"host", m.host},
      {"destination", m.destination},
      {"workload", m.workload},
      {"model", m.model},
      {"output_divisor", f9(m.output_divisor)},
      {"scale_factor", f9(m.scale_factor)},
      {"frames", std::to_string(r.cycles().size())},
      {"setup_s", f9(r.setup_s())},
      {"total_wall_s", f9(r.total_wall_s())},
      {"bytes_sent", std::to_string(r.bytes_sent())},
      {"bytes_received", std::to_string(r.bytes_received())},
      {"result_digest", m.result_digest},
  };
  for (const auto& kv : meta) out << "# " << kv.first << "=" << kv.second << "\n";
  out << "index,gpu_s,communication_s,other_s,bytes_sent,bytes_received\n";
  for (std::size_t i = 0; i < r.cycles().size(); ++i) {
    const CycleTiming& c = r.cycles()[i];
    out << i << ',' << f9(c.gpu_s) << ',' << f9(c.communication_s) << ',' << f9(c.other_s) << ','
        << c.bytes_sent << ',' << c.bytes_received << "\n";
  }
}

void write_summary_markdown(const RunRecord& r, std::ostream& out) {
  const RunMeta& m = r.meta();
  const std::size_t n = r.cycles().size();
  const double nn = n ? double(n) : 1.0;
  const double gpu = r.gpu_s(), comm = r.communication_s(), other = r.other_s();
  out << "# Run summary: " << m.label << "\n\n"
      << "- mode: " << m.mode << "\n"
      << "- host: " << m.host << "\n"
      << "- destination: " << m.destination << "\n"
      << "- workload: " << m.workload << "\n"
      << "- model: " << m.model << " (output divisor " << f9(m.output_divisor) << ")\n"
      << "- scale factor: " << f9(m.scale_factor) << "\n"
      << "- frames: " << n << "\n";
  if (!m.result_digest.empty()) out << "- result digest: " << m.result_digest << "\n";
  out << "\n| phase | total s | per frame s |\n|---|---|---|\n"
      << "| gpu | " << f9(gpu) << " | " << f9(gpu / nn) << " |\n"
      << "| communication | " << f9(comm) << " | " << f9(comm / nn) << " |\n"
      << "| other | " << f9(other) << " | " << f9(other / nn) << " |\n"
      << "| setup (one-time) | " << f9(r.setup_s()) << " | - |\n"
      << "| total wall | " << f9(r.total_wall_s()) << " | - |\n\n"
      << "- bytes sent: " << r.bytes_sent() << ", received: " << r.bytes_received() << "\n";
  if (n > 0 && r.processing_s() > 0) out << "- fps (setup excluded): " << f3(double(n) / r.processing_s()) << "\n";
}

}  // namespace avec::record
