// TEST-ONLY stub of proj/include/catsim/cost_model.hpp, used for ONE purpose:
// compiling the reference's acceptance gate (proj/tests/acceptance.cpp)
// unmodified against this repo's headers (tests/cpp/ref_suites.mk).  The
// analytical PRAM cost model (paper Eqs. 8-19, Table II) is out of scope for
// this build (no runtime role); every speedup here is 0,
// so acceptance criterion 2 ("analytical speedup table reproduction") reports
// FAIL explicitly instead of passing vacuously.  Criteria 1 and 3-7 -- the
// parity contract -- run against the B200 engines.
#pragma once

#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace catsim {

struct CostParams {};

struct Scenario {
  std::string name;
  std::vector<std::pair<std::string, std::string>> overrides;
};

struct SpeedupTable {
  std::vector<int> radii;
  std::vector<std::string> scenario_names;
  std::vector<std::vector<double>> speedups;
};

inline std::vector<Scenario> reference_scenarios(const CostParams&) {
  return std::vector<Scenario>(6, Scenario{"cost model not built", {}});
}

inline SpeedupTable scenario_table(const CostParams&, const std::vector<Scenario>& scenarios,
                                   const std::vector<int>& radii) {
  SpeedupTable t;
  t.radii = radii;
  for (const Scenario& s : scenarios) t.scenario_names.push_back(s.name);
  t.speedups.assign(scenarios.size(), std::vector<double>(radii.size(), 0.0));
  return t;
}

}  // namespace catsim
