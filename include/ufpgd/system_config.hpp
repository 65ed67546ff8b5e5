// /root/reference/proj/core/include/ufpgd/system_config.hpp:12-32.
#pragma once

#include "ufpgd/types.hpp"

namespace ufpgd {

struct SystemConfig {
  int K = 0;
  int M = 0;
  double sigma_nu = 1.0;
  RealVector gamma;
  double alpha = 1.0;

  static SystemConfig uniform(int num_users, int num_antennas, double sinr_target,
                              double noise_std = 1.0, double pa_scale = 1.0);
  void validate() const;              // system_config.cpp:22-43
  RealVector constraint_diag() const;  // sigma_nu * sqrt(gamma), system_config.cpp:45-47
};

}  // namespace ufpgd
