// capi_rule.cpp -- C-ABI wrappers of the host-side rule helpers
// (ltl_parse_rule / ltl_format_rule / presets / VN probe, include/ltl_b200.h).
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "host/internal.hpp"

extern "C" {

int ltl_parse_rule(const char* text, ltl_rule_c* out, char* err, int32_t err_len) {
  return ltl_parse_rule_ext(text, catsim::kMaxRadius, out, err, err_len);
}

int ltl_parse_rule_ext(const char* text, int32_t max_radius, ltl_rule_c* out, char* err,
                       int32_t err_len) {
  try {
    if (!text || !out) throw std::invalid_argument("rule parse error: field R: null input");
    *out = catsim::to_c(catsim::parse_ltl_rule(text, max_radius));
    if (err && err_len > 0) err[0] = '\0';
    return LTL_OK;
  } catch (const std::exception& e) {
    if (err && err_len > 0) {
      std::strncpy(err, e.what(), static_cast<size_t>(err_len) - 1);
      err[err_len - 1] = '\0';
    }
    return LTL_ERR_INVALID_ARGUMENT;
  }
}

int32_t ltl_format_rule(const ltl_rule_c* rule, char* buf, int32_t buf_len) {
  if (!rule) return -1;
  const std::string s = catsim::format_ltl_rule(catsim::from_c(*rule));
  if (buf && buf_len > 0) {
    std::strncpy(buf, s.c_str(), static_cast<size_t>(buf_len) - 1);
    buf[buf_len - 1] = '\0';
  }
  return static_cast<int32_t>(s.size());
}

int32_t ltl_preset_count(void) { return static_cast<int32_t>(catsim::ltl_presets().size()); }

int ltl_preset(int32_t index, const char** name, const char** rule, double* density) {
  const auto& all = catsim::ltl_presets();
  if (index < 0 || index >= static_cast<int32_t>(all.size())) return LTL_ERR_INVALID_ARGUMENT;
  if (name) *name = all[index].name;
  if (rule) *rule = all[index].rule;
  if (density) *density = all[index].density;
  return LTL_OK;
}

void ltl_von_neumann_probe_rule(int32_t r, ltl_rule_c* out) {
  if (out) *out = catsim::to_c(catsim::von_neumann_probe_rule(r));
}

}  // extern "C"
