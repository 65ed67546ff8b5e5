// ufpgd/trace_io.hpp of the reference (/root/reference/proj/core/include/ufpgd/trace_io.hpp:9-33):
// trace CSV files (schema run_id,index,lagrangian,residual,pcg,sum_rate,
// active_columns; 17 significant digits) and atomic file helpers.
#pragma once

#include <string>
#include <vector>

#include "ufpgd/pgd.hpp"

namespace ufpgd {

struct TraceRow {
  std::string run_id;
  TraceRecord record;
};

std::string format_trace_csv(const std::vector<TraceRow>& rows);
void write_trace_csv(const std::string& path, const std::vector<TraceRow>& rows);  // atomic
std::vector<TraceRow> read_trace_csv(const std::string& path);                     // DataFormatError
void write_file_atomic(const std::string& path, const std::string& contents);
std::string read_file(const std::string& path);

}  // namespace ufpgd
