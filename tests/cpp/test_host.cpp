// Host-only checks of the drop-in C++ API (no GPU needed; tests/test_cpp_api.py):
// model JSON files (unfolded.cpp:241-298), trace CSV files (trace_io.cpp) and
// parallel_for (parallel.cpp:25-59) — round trips, layouts, error cases.
#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "ufpgd/errors.hpp"
#include "ufpgd/parallel.hpp"
#include "ufpgd/trace_io.hpp"
#include "ufpgd/unfolded.hpp"

using namespace ufpgd;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                \
  do {                                                             \
    ++g_checks;                                                    \
    if (!(cond)) {                                                 \
      ++g_fail;                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                              \
  } while (0)

static bool rejects(const std::string& text) {
  try {
    network_from_json_string(text);
  } catch (const DataFormatError&) {
    return true;
  } catch (...) {
  }
  return false;
}

int main() {
  UnfoldedNetwork net = UnfoldedNetwork::pgd_init(8, 64, 20, 1.0 / 15.0);
  net.layers[3].lambda_i = 0.1;
  net.layers[7].eta_i *= 0.75;
  const std::string text = to_json_string(net);
  CHECK(text.rfind("{\n  \"I\": 20,\n  \"K\": 8,\n  \"M\": 64,\n  \"layers\": [\n    {\n      \"eta\": ", 0) == 0);
  CHECK(text.find("\"lambda\": 0.1\n") != std::string::npos);
  CHECK(text.find("\"version\": 1\n}\n") != std::string::npos);
  const UnfoldedNetwork back = network_from_json_string(text);
  bool same = back.num_users == 8 && back.num_antennas == 64 && back.mp_bound == net.mp_bound &&
              back.layers.size() == net.layers.size();
  for (std::size_t i = 0; same && i < net.layers.size(); ++i)
    same = back.layers[i].lambda_i == net.layers[i].lambda_i && back.layers[i].eta_i == net.layers[i].eta_i;
  CHECK(same);
  const std::string path = "/tmp/ufpgd_model_test.json";
  save_network(net, path);
  const UnfoldedNetwork loaded = load_network(path);
  CHECK(loaded.layers.size() == 20 && loaded.layers[7].eta_i == net.layers[7].eta_i);
  std::remove(path.c_str());
  CHECK(rejects("not json"));
  CHECK(rejects("{\"version\": 2, \"K\": 1, \"M\": 1, \"I\": 1, \"mp_bound\": 4.0, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 2, \"mp_bound\": 4.0, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 0, \"mp_bound\": 4.0, \"layers\": []}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 1, \"mp_bound\": 5.0, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 1, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 1, \"mp_bound\": 4.0, \"layers\": [{\"lambda\": 0.1}]}"));
  CHECK(rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 1, \"mp_bound\": 4.0, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]} x"));
  CHECK(!rejects("{\"version\": 1, \"K\": 1, \"M\": 1, \"I\": 1, \"mp_bound\": 4.0, \"layers\": [{\"lambda\": 0.1, \"eta\": 0.2}]}"));
  bool threw = false;
  try {
    load_network("/tmp/no_such_model.json");
  } catch (const DataFormatError&) {
    threw = true;
  }
  CHECK(threw);
  {  // trace CSV round trip and corruption (test_trace_io.cpp)
    std::vector<TraceRow> rows(3);
    for (int i = 0; i < 3; ++i) {
      rows[i].run_id = i == 2 ? "" : "run" + std::to_string(i);
      rows[i].record.index = 10 * i;
      rows[i].record.lagrangian = 0.1 + i / 3.0;
      rows[i].record.residual = 1e-17 * (i + 1);
      rows[i].record.pcg = 1.0915;
      rows[i].record.sum_rate = 27.68 + i;
      rows[i].record.active_columns = 63.5;
    }
    const std::string text = format_trace_csv(rows);
    CHECK(text.rfind("run_id,index,lagrangian,residual,pcg,sum_rate,active_columns\nrun0,0,", 0) == 0);
    const std::string path = "/tmp/ufpgd_trace_test.csv";
    write_trace_csv(path, rows);
    CHECK(read_file(path) == text);
    const std::vector<TraceRow> back = read_trace_csv(path);
    bool same = back.size() == 3;
    for (std::size_t i = 0; same && i < 3; ++i)
      same = back[i].run_id == rows[i].run_id && back[i].record.index == rows[i].record.index &&
             back[i].record.lagrangian == rows[i].record.lagrangian && back[i].record.residual == rows[i].record.residual &&
             back[i].record.sum_rate == rows[i].record.sum_rate && back[i].record.active_columns == rows[i].record.active_columns;
    CHECK(same);
    write_file_atomic(path, "run_id,index\n");
    bool threw = false;
    try {
      read_trace_csv(path);
    } catch (const DataFormatError&) {
      threw = true;
    }
    CHECK(threw);
    write_file_atomic(path, std::string("run_id,index,lagrangian,residual,pcg,sum_rate,active_columns\n") + "a,1,2,x,4,5,6\n");
    threw = false;
    try {
      read_trace_csv(path);
    } catch (const DataFormatError&) {
      threw = true;
    }
    CHECK(threw);
    std::remove(path.c_str());
  }
  {  // parallel_for: every index once, first exception rethrown (parallel.cpp:25-59)
    std::vector<std::atomic<int>> hits(1000);
    parallel_for(hits.size(), [&](std::size_t i) { hits[i].fetch_add(1); }, 7);
    bool once = true;
    for (auto& h : hits) once = once && h.load() == 1;
    CHECK(once);
    bool threw = false;
    try {
      parallel_for(100, [](std::size_t i) { if (i == 37) throw std::runtime_error("boom"); }, 4);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
    CHECK(default_thread_count() >= 1);
    parallel_for(0, [](std::size_t) { throw std::runtime_error("never"); });
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
