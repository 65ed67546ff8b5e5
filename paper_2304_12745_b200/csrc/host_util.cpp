// Host utilities of the reference core kept for source compatibility:
// parallel_for / default_thread_count (parallel.cpp:13-59) and trace CSV +
// atomic file I/O (trace_io.cpp). Not on the solver path.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ufpgd/channel.hpp"
#include "ufpgd/errors.hpp"
#include "ufpgd/parallel.hpp"
#include "ufpgd/trace_io.hpp"

namespace ufpgd {

ComplexVector simulate_received(const ChannelMatrix& channel, const PrecoderMatrix& precoder,
                                const ComplexVector& symbols, const SystemConfig& cfg, Rng& rng) {
  cfg.validate();
  if (channel.rows() != cfg.K || channel.cols() != cfg.M || precoder.rows() != cfg.K || precoder.cols() != cfg.M ||
      static_cast<int>(symbols.size()) != cfg.K)
    throw std::invalid_argument("simulate_received: shape mismatch");
  ComplexVector x(static_cast<std::size_t>(cfg.M), Complex(0.0, 0.0));  // transmit vector W^T s
  for (int m = 0; m < cfg.M; ++m)
    for (int k = 0; k < cfg.K; ++k) x[m] += precoder(k, m) * symbols[k];
  ComplexVector r(static_cast<std::size_t>(cfg.K), Complex(0.0, 0.0));
  for (int k = 0; k < cfg.K; ++k) {
    for (int m = 0; m < cfg.M; ++m) r[k] += channel(k, m) * x[m];
    r[k] += cfg.sigma_nu * rng.complex_gaussian();
  }
  return r;
}

int default_thread_count() {
  if (const char* v = std::getenv("UFPGD_THREADS")) {
    char* end = nullptr;
    const long n = std::strtol(v, &end, 10);
    if (end && *end == '\0' && n > 0) return static_cast<int>(n);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

void parallel_for(std::size_t n, const std::function<void(std::size_t)>& body, int threads) {
  if (n == 0) return;
  const std::size_t workers = std::min<std::size_t>(n, static_cast<std::size_t>(threads > 0 ? threads : default_thread_count()));
  std::atomic<std::size_t> next{0};
  std::exception_ptr first;
  std::mutex mu;
  auto run = [&] {
    for (;;) {
      const std::size_t i = next.fetch_add(1);
      if (i >= n) return;
      try {
        body(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!first) first = std::current_exception();
        next.store(n);  // stop handing out work
      }
    }
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < workers; ++t) pool.emplace_back(run);
  run();
  for (std::thread& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}

namespace {

constexpr const char* kHeader = "run_id,index,lagrangian,residual,pcg,sum_rate,active_columns";

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

double cell_double(const std::string& s) {
  std::size_t used = 0;
  const double v = std::stod(s, &used);
  if (used != s.size()) throw DataFormatError("trace CSV: bad numeric cell '" + s + "'");
  return v;
}

}  // namespace

std::string format_trace_csv(const std::vector<TraceRow>& rows) {
  std::string out = std::string(kHeader) + "\n";
  for (const TraceRow& r : rows) {
    out += r.run_id + "," + std::to_string(r.record.index) + "," + g17(r.record.lagrangian) + "," +
           g17(r.record.residual) + "," + g17(r.record.pcg) + "," + g17(r.record.sum_rate) + "," +
           g17(r.record.active_columns) + "\n";
  }
  return out;
}

void write_file_atomic(const std::string& path, const std::string& contents) {
  const std::filesystem::path target(path);
  std::filesystem::path temp = target;
  temp += ".tmp";
  {
    std::ofstream out(temp, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open for writing: " + temp.string());
    out << contents;
    out.flush();
    if (!out) throw std::runtime_error("write failed: " + temp.string());
  }
  std::filesystem::rename(temp, target);
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataFormatError("cannot open file: " + path);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

void write_trace_csv(const std::string& path, const std::vector<TraceRow>& rows) {
  write_file_atomic(path, format_trace_csv(rows));
}

std::vector<TraceRow> read_trace_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw DataFormatError("cannot open trace file: " + path);
  std::string line;
  if (!std::getline(in, line) || line != kHeader) throw DataFormatError("trace CSV: missing or wrong header in " + path);
  std::vector<TraceRow> rows;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::vector<std::string> f;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) f.push_back(cell);
    if (!line.empty() && line.back() == ',') f.push_back("");
    if (f.size() != 7) throw DataFormatError("trace CSV: expected 7 columns, got " + std::to_string(f.size()));
    TraceRow r;
    r.run_id = f[0];
    try {
      std::size_t used = 0;
      r.record.index = std::stol(f[1], &used);
      if (used != f[1].size()) throw DataFormatError("trace CSV: bad index cell '" + f[1] + "'");
      r.record.lagrangian = cell_double(f[2]);
      r.record.residual = cell_double(f[3]);
      r.record.pcg = cell_double(f[4]);
      r.record.sum_rate = cell_double(f[5]);
      r.record.active_columns = cell_double(f[6]);
    } catch (const std::logic_error&) {
      throw DataFormatError("trace CSV: unparsable row '" + line + "'");
    }
    rows.push_back(std::move(r));
  }
  return rows;
}

}  // namespace ufpgd
