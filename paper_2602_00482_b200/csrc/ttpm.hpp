// TTPM reader (model_io.cpp:73-105) and the canonical tensor table (model.hpp:42-59).
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/treetrain_b200.h"

namespace ttb {

std::vector<std::pair<std::string, std::vector<uint64_t>>> tensor_specs(const tt_model_config& c);

struct TtpmFile {
  tt_model_config config;
  std::vector<double> values;  // for_each_tensor order
};
TtpmFile read_ttpm(const std::string& path);

}  // namespace ttb
