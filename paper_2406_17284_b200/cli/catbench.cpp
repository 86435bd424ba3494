// catbench -- the reference's command-line front end (proj/tools/catbench.cpp,
// subcommands run / verify / bench / sweep-tiles / cost-model), rebuilt over
// this repo's catsim C++ API (include/catsim/) and therefore over the B200
// library: `cat` is the tcgen05 banded-MMA engine, `base` / `pack` the
// CUDA-core ablations standing in for the reference's BASE / PACK.  Same
// options, defaults, output lines, CSV and exit codes (0 ok, 1 verify
// failures, 2 any error; `--engine gpu` stays an unknown engine).  CLI11 is
// absent here (proj/.gitignore:2), so options are parsed by hand:
// `--name value`, `--name=value`, flags, CAT_WORKERS for --workers.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "catsim/bench.hpp"
#include "catsim/engines.hpp"
#include "catsim/grid.hpp"
#include "catsim/rule.hpp"
#include "catsim/snapshot.hpp"
#if __has_include("catsim/cost_model.hpp")
#include "catsim/cost_model.hpp"
#define CATBENCH_COST_MODEL 1
#endif

using namespace catsim;

namespace {

[[noreturn]] void config_fail(const std::string& why) {
  throw std::invalid_argument("config error: " + why);
}

// Command-line usage errors, with CLI11's exit codes: 104 conversion (not a
// number), 105 validation (--f not in {4,8,16}), 106 required (no
// subcommand), 109 extras (unknown option / argument), 114 argument mismatch
// (an option without its value).
struct UsageError : std::runtime_error {
  int code;
  UsageError(const std::string& what, int code_) : std::runtime_error(what), code(code_) {}
};

int parse_int_token(const std::string& tok) {
  std::size_t used = 0;
  long v = 0;
  try {
    v = std::stol(tok, &used, 10);
  } catch (const std::exception&) {
    used = 0;
  }
  if (tok.empty() || used != tok.size() || v < INT32_MIN || v > INT32_MAX)
    config_fail("bad integer '" + tok + "'");
  return static_cast<int>(v);
}

std::vector<std::string> split_list(const std::string& text) {
  std::vector<std::string> out;
  std::string tok;
  std::istringstream ss(text);
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) out.push_back(tok);
  return out;
}

// "1,3-5,16" -> {1,3,4,5,16}
std::vector<int> parse_int_list(const std::string& text) {
  std::vector<int> out;
  for (const std::string& tok : split_list(text)) {
    const auto dash = tok.find('-', 1);
    if (dash == std::string::npos) {
      out.push_back(parse_int_token(tok));
      continue;
    }
    const int a = parse_int_token(tok.substr(0, dash)), b = parse_int_token(tok.substr(dash + 1));
    if (b < a) config_fail("descending range '" + tok + "'");
    for (int v = a; v <= b; ++v) out.push_back(v);
  }
  return out;
}

std::vector<std::pair<int, int>> parse_shape_list(const std::string& text) {
  std::vector<std::pair<int, int>> out;
  for (const std::string& tok : split_list(text)) {
    const auto x = tok.find('x');
    if (x == std::string::npos || x == 0 || x + 1 == tok.size())
      config_fail("bad tile shape '" + tok + "' (expected WxH)");
    out.emplace_back(parse_int_token(tok.substr(0, x)), parse_int_token(tok.substr(x + 1)));
  }
  return out;
}

// ---- option parsing ----------------------------------------------------------
class Options {
 public:
  // spec: option -> number of values it takes (0: a flag)
  Options(std::vector<std::string> args, std::map<std::string, int> spec)
      : spec_(std::move(spec)) {
    for (std::size_t i = 0; i < args.size(); ++i) {
      std::string a = args[i];
      if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a, 109);
      std::string value;
      bool has_value = false;
      const auto eq = a.find('=');
      if (eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_value = true;
      }
      const auto it = spec_.find(a);
      if (it == spec_.end()) throw UsageError("The following argument was not expected: " + a, 109);
      if (it->second > 0) {  // takes values
        auto& vals = values_[a];
        for (int k = 0; k < it->second; ++k) {
          if (k == 0 && has_value) {
            vals.push_back(value);
            continue;
          }
          if (i + 1 >= args.size())
            throw UsageError(a + ": " + std::to_string(it->second) + " value(s) required", 114);
          vals.push_back(args[++i]);
        }
      } else {
        if (has_value) throw UsageError(a + ": takes no value", 114);
        values_[a].push_back("1");
      }
    }
  }
  bool has(const std::string& k) const { return values_.count(k) > 0; }
  std::string str(const std::string& k, const std::string& dflt) const {
    return has(k) ? values_.at(k).back() : dflt;
  }
  std::vector<std::string> all(const std::string& k) const {
    return has(k) ? values_.at(k) : std::vector<std::string>{};
  }
  int integer(const std::string& k, int dflt) const {
    if (!has(k)) return dflt;
    try {
      return parse_int_token(str(k, ""));
    } catch (const std::invalid_argument&) {
      throw UsageError(k + ": '" + str(k, "") + "' is not an integer", 104);
    }
  }
  double real(const std::string& k, double dflt) const {
    if (!has(k)) return dflt;
    const std::string v = str(k, "");
    std::size_t used = 0;
    double d = 0;
    try {
      d = std::stod(v, &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used != v.size() || v.empty()) throw UsageError(k + ": '" + v + "' is not a number", 104);
    return d;
  }
  uint64_t u64(const std::string& k, uint64_t dflt) const {
    if (!has(k)) return dflt;
    const std::string v = str(k, "");
    std::size_t used = 0;
    unsigned long long d = 0;
    try {
      d = std::stoull(v, &used, 10);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used != v.size() || v.empty() || v[0] == '-')
      throw UsageError(k + ": '" + v + "' is not an unsigned integer", 104);
    return d;
  }

 private:
  std::map<std::string, int> spec_;
  std::map<std::string, std::vector<std::string>> values_;
};

// Shared engine / geometry options (catbench.cpp:133-157).
struct EngineOpts {
  int f = kDefaultFragmentSide;
  int tile_w = 1;
  int tile_h = 14;
  int workers = 1;
};

void add_engine_spec(std::map<std::string, int>& spec) {
  for (const char* k : {"--f", "--tile-w", "--tile-h", "--workers"}) spec[k] = 1;
}

EngineOpts engine_opts(const Options& o) {
  EngineOpts e;
  e.f = o.integer("--f", e.f);
  if (e.f != 4 && e.f != 8 && e.f != 16)
    throw UsageError("--f: value " + std::to_string(e.f) + " not in {4,8,16}", 105);
  e.tile_w = o.integer("--tile-w", e.tile_w);
  e.tile_h = o.integer("--tile-h", e.tile_h);
  if (o.has("--workers")) {
    e.workers = o.integer("--workers", e.workers);
  } else if (const char* env = std::getenv("CAT_WORKERS")) {
    try {
      e.workers = parse_int_token(env);
    } catch (const std::invalid_argument&) {
      throw UsageError(std::string("CAT_WORKERS: '") + env + "' is not an integer", 104);
    }
  }
  return e;
}

CatConfig make_config(const EngineOpts& opts, NeighborhoodKind kind) {
  CatConfig cfg;
  cfg.f = opts.f;
  cfg.tile_w = opts.tile_w;
  cfg.tile_h = opts.tile_h;
  cfg.workers = opts.workers;
  cfg.kind = kind;
  return cfg;
}

struct RuleChoice {
  LtlRule rule;
  double density = 0.25;
};

// Exactly one of --rule / --preset; the preset brings its published density.
RuleChoice resolve_rule(const std::string& rule_text, const std::string& preset_name,
                        double density, bool density_set) {
  RuleChoice rc;
  if (!rule_text.empty() && !preset_name.empty())
    config_fail("--rule and --preset are mutually exclusive");
  if (!rule_text.empty()) {
    rc.rule = parse_ltl_rule(rule_text);
  } else {
    const std::string name = preset_name.empty() ? "life" : preset_name;
    const LtlPreset* preset = find_preset(name);
    if (!preset) {
      std::string known;
      for (const LtlPreset& p : ltl_presets()) known += (known.empty() ? "" : ", ") + std::string(p.name);
      config_fail("unknown preset '" + name + "' (known: " + known + ")");
    }
    rc.rule = parse_ltl_rule(preset->rule);
    rc.density = preset->density;
  }
  if (density_set) rc.density = density;
  if (rc.density < 0.0 || rc.density > 1.0) config_fail("density must be in [0, 1]");
  return rc;
}

int round_up(int n, int f) { return (n + f - 1) / f * f; }

// n rounded up to a multiple of f; only the requested n x n block is seeded.
Grid make_initial(int n, int f, double density, uint64_t seed) {
  const int rounded = round_up(n, f);
  return init_random(rounded, density, seed, f, rounded == n ? -1 : n);
}

double time_run_ms(EngineKind kind, const Grid& initial, const LtlRule& rule,
                   const CatConfig& cfg, int steps, RunStats* stats = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  const Grid out = run_engine(kind, initial, rule, cfg, steps, stats);
  const auto t1 = std::chrono::steady_clock::now();
  (void)out;
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

// ---- subcommands -------------------------------------------------------------
int cmd_run(const Options& o) {
  const RuleChoice rc = resolve_rule(o.str("--rule", ""), o.str("--preset", ""),
                                     o.real("--density", 0.25), o.has("--density"));
  const EngineOpts opts = engine_opts(o);
  const int n = o.integer("--n", 256), steps = o.integer("--steps", 1);
  const uint64_t seed = o.u64("--seed", 1);
  const std::string engine = o.str("--engine", "cat"), out_path = o.str("--out", "");
  const EngineKind kind = parse_engine(engine);
  const CatConfig cfg = make_config(opts, rc.rule.kind);
  const int rounded = round_up(n, opts.f);
  const Grid initial = make_initial(n, opts.f, rc.density, seed);

  RunStats stats;
  const auto t0 = std::chrono::steady_clock::now();
  const Grid final_grid = run_engine(kind, initial, rc.rule, cfg, steps, &stats);
  const auto t1 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();

  std::cout << "engine " << engine_name(kind) << " rule " << format_ltl_rule(rc.rule) << " n "
            << rounded;
  if (rounded != n) std::cout << " (requested " << n << ", padded to fit f)";
  std::cout << " f " << opts.f << " steps " << steps << " seed " << seed << " density "
            << rc.density << '\n';
  std::cout << "alive " << count_alive(final_grid) << '\n';
  const double per_step = steps > 0 ? ms / steps : ms;
  char line[160];
  std::snprintf(line, sizeof line, "elapsed_ms %.3f ms_per_step %.4f cells_per_sec %.4g", ms,
                per_step,
                per_step > 0 ? static_cast<double>(rounded) * rounded * 1000.0 / per_step : 0.0);
  std::cout << line << '\n';
  if (kind == EngineKind::Cat)
    std::cout << "mma_count " << stats.cat.mma_count << " max_h " << stats.cat.max_h
              << " max_r " << stats.cat.max_r << '\n';
  if (kind == EngineKind::Base) std::cout << "memory_accesses " << stats.base.accesses() << '\n';
  if (!out_path.empty()) {
    snapshot_write(final_grid, out_path);
    std::cout << "snapshot " << out_path << '\n';
  }
  return 0;
}

// cat vs base (vs pack when its word gathers fit) per (r, kind, n, seed, steps):
// three independent device implementations must agree cell for cell; with
// --inject-fault the faulted cat run must diverge or abort.
int cmd_verify(const Options& o) {
  const std::vector<int> radii = parse_int_list(o.str("--radii", "1-16"));
  const std::vector<int> sizes = parse_int_list(o.str("--sizes", "32,64"));
  const std::vector<int> seeds = parse_int_list(o.str("--seeds", "1,2"));
  const std::vector<int> steps_list = parse_int_list(o.str("--steps", "1,25"));
  const std::vector<std::string> kinds = split_list(o.str("--kinds", "moore,vn"));
  const bool inject_fault = o.has("--inject-fault");
  const EngineOpts opts = engine_opts(o);
  if (radii.empty() || sizes.empty() || seeds.empty() || steps_list.empty() || kinds.empty()) {
    std::cout << "nothing to verify\n";
    return 0;
  }
  int pass = 0, fail = 0;
  for (const int r : radii) {
    if (r < 1 || r > 16) config_fail("radius must be in 1..16");
    for (const std::string& kind_name : kinds) {
      LtlRule rule;
      double density = 0.25;
      if (kind_name == "moore") {
        const LtlPreset& preset = ltl_presets()[static_cast<std::size_t>(r - 1)];
        rule = parse_ltl_rule(preset.rule);
        density = preset.density;
      } else if (kind_name == "vn") {
        rule = von_neumann_probe_rule(r);
      } else {
        config_fail("unknown kind '" + kind_name + "' (moore, vn)");
      }
      const bool pack_fits = opts.f >= 8 * ((r + 7) / 8);
      for (const int n : sizes)
        for (const int seed : seeds)
          for (const int steps : steps_list) {
            if (n % opts.f != 0) config_fail("size " + std::to_string(n) + " is not a multiple of f");
            const Grid initial = make_initial(n, opts.f, density, static_cast<uint64_t>(seed));
            CatConfig cfg = make_config(opts, rule.kind);
            cfg.inject_band_fault = inject_fault;
            std::optional<Grid> cat_out;
            try {
              cat_out = run_engine(EngineKind::Cat, initial, rule, cfg, steps);
            } catch (const std::exception&) {
              if (!inject_fault) throw;  // a faulted band may trip the guard: detected
            }
            cfg.inject_band_fault = false;
            const Grid base_out = run_engine(EngineKind::Base, initial, rule, cfg, steps);
            std::optional<CellCoord> diff;
            if (cat_out) diff = first_interior_difference(base_out, *cat_out);
            std::string label = "r=" + std::to_string(r) + " kind=" + kind_name +
                                " n=" + std::to_string(n) + " seed=" + std::to_string(seed) +
                                " steps=" + std::to_string(steps);
            bool ok;
            if (inject_fault) {
              ok = !cat_out || diff.has_value();
              label += !ok ? " (fault missed)"
                           : !cat_out ? " (fault detected: engine aborted)"
                                      : " (fault detected: grid diverged)";
            } else {
              ok = !diff.has_value();
              if (ok && pack_fits) {
                const Grid pack_out = run_engine(EngineKind::Pack, initial, rule, cfg, steps);
                const auto pd = first_interior_difference(base_out, pack_out);
                if (pd) {
                  ok = false;
                  label += " pack first-diff=(" + std::to_string(pd->y) + "," +
                           std::to_string(pd->x) + ")";
                } else {
                  label += " engines=cat,base,pack";
                }
              } else if (ok) {
                label += " engines=cat,base";
              }
              if (!ok && diff)
                label += " first-diff=(" + std::to_string(diff->y) + "," + std::to_string(diff->x) +
                         ") base=" + std::to_string(base_out.interior(diff->y, diff->x)) +
                         " cat=" + std::to_string(cat_out->interior(diff->y, diff->x));
            }
            std::cout << (ok ? "PASS " : "FAIL ") << label << '\n';
            ++(ok ? pass : fail);
          }
    }
  }
  std::cout << "verified " << (pass + fail) << " combinations: " << pass << " pass, " << fail
            << " fail\n";
  return fail == 0 ? 0 : 1;
}

// Realizations of whole run_engine calls until the stderr of the mean is
// below --target-stderr percent (or --max-realizations), one CSV row per engine.
int cmd_bench(const Options& o) {
  const RuleChoice rc = resolve_rule(o.str("--rule", ""), o.str("--preset", ""),
                                     o.real("--density", 0.25), o.has("--density"));
  const EngineOpts opts = engine_opts(o);
  const int n = o.integer("--n", 1024), steps = o.integer("--steps", 10);
  const uint64_t seed = o.u64("--seed", 1);
  const int max_realizations = o.integer("--max-realizations", 16);
  const double target_stderr = o.real("--target-stderr", 1.0);
  const std::string csv_path = o.str("--csv", "");
  const CatConfig cfg = make_config(opts, rc.rule.kind);
  const Grid initial = make_initial(n, opts.f, rc.density, seed);
  const int rounded = round_up(n, opts.f);
  if (steps < 1) config_fail("bench needs steps >= 1");
  if (max_realizations < 3) config_fail("bench needs at least 3 realizations");
  std::ostringstream out;
  out << bench_csv_header() << '\n';
  for (const std::string& name : split_list(o.str("--engines", "cat,base,pack"))) {
    const EngineKind kind = parse_engine(name);
    time_run_ms(kind, initial, rc.rule, cfg, 1);  // warm: device context, code paths
    BenchAccumulator acc;
    while (acc.count() < max_realizations && !acc.converged(target_stderr, 3))
      acc.add(time_run_ms(kind, initial, rc.rule, cfg, steps) / steps);
    out << bench_csv_row(engine_name(kind), rounded, rc.rule.r, steps, acc) << '\n';
  }
  if (csv_path.empty()) {
    std::cout << out.str();
  } else {
    std::ofstream file(csv_path);
    if (!file) config_fail("cannot open '" + csv_path + "' for writing");
    file << out.str();
    std::cout << "wrote " << csv_path << '\n';
  }
  return 0;
}

// Tile shapes are accepted and validated as the reference's; on the device
// they do not change the schedule (nor, as in the reference, the bytes).
int cmd_sweep_tiles(const Options& o) {
  const RuleChoice rc = resolve_rule(o.str("--rule", ""), o.str("--preset", ""),
                                     o.real("--density", 0.25), o.has("--density"));
  const EngineOpts opts = engine_opts(o);
  const int n = o.integer("--n", 1024), steps = o.integer("--steps", 5);
  const int realizations = o.integer("--realizations", 3);
  const Grid initial = make_initial(n, opts.f, rc.density, o.u64("--seed", 1));
  if (realizations < 1) config_fail("sweep needs realizations >= 1");
  std::cout << "tile_w,tile_h,ms_per_step\n";
  for (const auto& [tw, th] : parse_shape_list(o.str("--shapes", "1x1,1x14,14x1,2x7,7x2,4x4,8x8,16x16"))) {
    EngineOpts shaped = opts;
    shaped.tile_w = tw;
    shaped.tile_h = th;
    const CatConfig cfg = make_config(shaped, rc.rule.kind);
    time_run_ms(EngineKind::Cat, initial, rc.rule, cfg, 1);
    BenchAccumulator acc;
    for (int i = 0; i < realizations; ++i)
      acc.add(time_run_ms(EngineKind::Cat, initial, rc.rule, cfg, steps) / steps);
    char line[64];
    std::snprintf(line, sizeof line, "%d,%d,%.6g", tw, th, acc.mean());
    std::cout << line << '\n';
  }
  return 0;
}

int cmd_cost_model(const Options& o) {
#ifdef CATBENCH_COST_MODEL
  CostParams base;
  bool customized = false;
  const std::string params_path = o.str("--params", "");
  if (!params_path.empty()) {
    std::ifstream file(params_path);
    if (!file) config_fail("cannot open '" + params_path + "'");
    std::string line;
    while (std::getline(file, line)) {
      const auto start = line.find_first_not_of(" \t");
      if (start == std::string::npos || line[start] == '#') continue;
      const auto end = line.find_last_not_of(" \t\r");
      apply_override_line(base, line.substr(start, end - start + 1));
      customized = true;
    }
  }
  for (const std::string& kv : o.all("--set")) {
    apply_override_line(base, kv);
    customized = true;
  }
  std::vector<std::string> derive = o.all("--derive-e");
  if (!derive.empty()) {
    derive.erase(derive.begin(), derive.end() - 2);  // the last occurrence wins
    const int r = parse_int_token(derive[0]);
    double target = 0.0;
    try {
      target = std::stod(derive[1]);
    } catch (const std::exception&) {
      config_fail("bad speedup target '" + derive[1] + "'");
    }
    char buf[48];
    std::snprintf(buf, sizeof buf, "%.17g", derive_e(base, r, target));
    std::cout << "E=" << buf << '\n';
    return 0;
  }
  const std::vector<int> radii = parse_int_list(o.str("--radii", "1,4,8,16"));
  if (radii.empty()) config_fail("no radii given");
  const std::vector<Scenario> scenarios =
      customized ? std::vector<Scenario>{{"custom", {}}} : reference_scenarios(base);
  const SpeedupTable table = scenario_table(base, scenarios, radii);
  std::cout << (o.has("--csv") ? format_table_csv(table) : format_table_text(table));
  return 0;
#else
  (void)o;
  config_fail("cost-model is not part of this build");
#endif
}

const char* kUsage =
    "banded matrix-multiply cellular automata toolkit (B200 engines)\n"
    "usage: catbench <run|verify|bench|sweep-tiles|cost-model> [options]\n"
    "  run          --rule R --preset P --density D --n N --steps S --seed X --engine cat|base|pack\n"
    "               --out FILE --f 4|8|16 --tile-w W --tile-h H --workers K\n"
    "  verify       --radii 1-16 --sizes 32,64 --seeds 1,2 --kinds moore,vn --steps 1,25\n"
    "               --inject-fault [engine options]\n"
    "  bench        --rule/--preset --density --n 1024 --steps 10 --seed --engines cat,base,pack\n"
    "               --max-realizations 16 --target-stderr 1 --csv FILE [engine options]\n"
    "  sweep-tiles  --rule/--preset --density --n 1024 --steps 5 --seed --shapes WxH,...\n"
    "               --realizations 3 [engine options]\n"
    "  cost-model   --params FILE --set k=v --radii 1,4,8,16 --csv --derive-e R TARGET\n";

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty()) {
    std::cerr << "A subcommand is required\n" << kUsage;
    return 106;
  }
  if (args[0] == "--help" || args[0] == "-h") {
    std::cout << kUsage;
    return 0;
  }
  const std::string sub = args[0];
  args.erase(args.begin());
  std::map<std::string, int> spec;
  int (*fn)(const Options&) = nullptr;
  if (sub == "run") {
    for (const char* k : {"--rule", "--preset", "--density", "--n", "--steps", "--seed", "--engine", "--out"})
      spec[k] = 1;
    add_engine_spec(spec);
    fn = cmd_run;
  } else if (sub == "verify") {
    for (const char* k : {"--radii", "--sizes", "--seeds", "--kinds", "--steps"}) spec[k] = 1;
    spec["--inject-fault"] = 0;
    add_engine_spec(spec);
    fn = cmd_verify;
  } else if (sub == "bench") {
    for (const char* k : {"--rule", "--preset", "--density", "--n", "--steps", "--seed", "--engines",
                          "--max-realizations", "--target-stderr", "--csv"})
      spec[k] = 1;
    add_engine_spec(spec);
    fn = cmd_bench;
  } else if (sub == "sweep-tiles") {
    for (const char* k : {"--rule", "--preset", "--density", "--n", "--steps", "--seed", "--shapes",
                          "--realizations"})
      spec[k] = 1;
    add_engine_spec(spec);
    fn = cmd_sweep_tiles;
  } else if (sub == "cost-model") {
    for (const char* k : {"--params", "--set", "--radii"}) spec[k] = 1;
    spec["--derive-e"] = 2;
    spec["--csv"] = 0;
    fn = cmd_cost_model;
  } else {
    std::cerr << "unknown subcommand '" << sub << "'\n" << kUsage;
    return 109;
  }
  try {
    const Options opts(args, spec);
    return fn(opts);
  } catch (const UsageError& ex) {
    std::cerr << ex.what() << "\n" << kUsage;
    return ex.code;
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << '\n';
    return 2;
  }
}
