// Host-only checks of the model JSON files (unfolded.cpp:241-298) of the
// drop-in C++ API: round trip, layout and the DataFormatError cases. Runs
// without a GPU (tests/test_cpp_api.py).
#include <cstdio>
#include <string>

#include "ufpgd/errors.hpp"
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
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
