// tuning_db.cu -- see tuning_db.cuh.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "tuning_db.cuh"

namespace tkb {

namespace {

std::mutex g_mu;
std::map<std::string, TunedKnobs>& db() {
  static std::map<std::string, TunedKnobs> m;
  return m;
}

// Value of "key": in one flat JSON object line (strings unescaped simply;
// the DB's values are plain identifiers and numbers).
bool field(const std::string& line, const char* key, std::string* out) {
  const std::string pat = std::string("\"") + key + "\"";
  size_t p = line.find(pat);
  if (p == std::string::npos) return false;
  p = line.find(':', p + pat.size());
  if (p == std::string::npos) return false;
  ++p;
  while (p < line.size() && (line[p] == ' ' || line[p] == '\t')) ++p;
  if (p < line.size() && line[p] == '"') {
    const size_t e = line.find('"', p + 1);
    if (e == std::string::npos) return false;
    *out = line.substr(p + 1, e - p - 1);
    return true;
  }
  size_t e = p;
  while (e < line.size() && line[e] != ',' && line[e] != '}') ++e;
  *out = line.substr(p, e - p);
  while (!out->empty() && (out->back() == ' ' || out->back() == '\r')) out->pop_back();
  return true;
}

int precision_of_name(const std::string& s) {
  if (s == "tf32") return TK_PREC_TF32;
  if (s == "bf16") return TK_PREC_BF16;
  if (s == "3xtf32") return TK_PREC_3XTF32;
  if (s == "fp32") return TK_PREC_FP32_EXACT;
  return -1;
}

// "<family>@<precision><suffix>" with suffix tokens _n<N> _s<S> _c<C>
// _halo|_pixn|_pixm|_gather|_pointwise|_im2col _nosplit _k<K>
// (tilekit::b200::ExecOptions::suffix).
bool parse_config(const std::string& cfg, std::string* family, int* prec, TunedKnobs* k) {
  const size_t at = cfg.find('@');
  if (at == std::string::npos) return false;
  *family = cfg.substr(0, at);
  std::string rest = cfg.substr(at + 1);
  const size_t us = rest.find('_');
  *prec = precision_of_name(rest.substr(0, us));
  if (*prec < 0) return false;
  static const char* modes[] = {"", "halo", "pixn", "pixm", "gather", "pointwise", "im2col"};
  size_t p = us;
  while (p != std::string::npos && p < rest.size()) {
    size_t e = rest.find('_', p + 1);
    const std::string tok = rest.substr(p + 1, e == std::string::npos ? std::string::npos : e - p - 1);
    p = e;
    if (tok.empty()) continue;
    bool is_mode = false;
    for (int m = 1; m < 7; ++m)
      if (tok == modes[m]) {
        k->mode = m;
        is_mode = true;
      }
    if (is_mode) continue;
    if (tok == "nosplit") {
      k->split = 1;
      continue;
    }
    const int v = std::atoi(tok.c_str() + 1);
    switch (tok[0]) {
      case 'n': k->tile_n = v; break;
      case 's': k->stages = v; break;
      case 'c': k->cluster = v; break;
      case 'k': k->split = v; break;
      default: return false;
    }
  }
  return true;
}

std::string db_key(const std::string& problem, const std::string& family, int prec) {
  return problem + "|" + family + "|" + std::to_string(prec);
}

}  // namespace

size_t tuning_db_load(const std::string& path, const std::string& device) {
  std::ifstream in(path);
  if (!in) fail(TK_ERR_IO, "tuning_db_load: cannot open \"" + path + "\"");
  std::string line;
  size_t kept = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  while (std::getline(in, line)) {
    if (line.find('{') == std::string::npos) continue;
    std::string problem, config, dev, ns, valid;
    if (!field(line, "problem", &problem) || !field(line, "config", &config) ||
        !field(line, "median_ns", &ns))
      fail(TK_ERR_PARSE, "tuning_db_load: record without problem/config/median_ns: " + line);
    if (field(line, "valid", &valid) && valid != "true") continue;
    if (!device.empty() && field(line, "device", &dev) && dev != device) continue;
    std::string family;
    int prec = -1;
    TunedKnobs k;
    if (!parse_config(config, &family, &prec, &k)) continue;  // exact-FP32 names: no knobs
    k.median_ns = std::atoll(ns.c_str());
    k.config = config;
    if (k.median_ns <= 0) continue;
    auto& m = db();
    const std::string key = db_key(problem, family, prec);
    auto it = m.find(key);
    // fastest record wins; equal times: the lexically smaller name (stable)
    if (it == m.end() || k.median_ns < it->second.median_ns ||
        (k.median_ns == it->second.median_ns && k.config < it->second.config)) {
      m[key] = k;
      ++kept;
    }
  }
  return kept;
}

void tuning_db_clear() {
  std::lock_guard<std::mutex> lk(g_mu);
  db().clear();
}

size_t tuning_db_size() {
  std::lock_guard<std::mutex> lk(g_mu);
  return db().size();
}

bool tuning_db_lookup(const std::string& problem, const std::string& family, int precision,
                      TunedKnobs* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  const auto& m = db();
  if (m.empty()) return false;
  auto it = m.find(db_key(problem, family, precision));
  if (it == m.end()) return false;
  *out = it->second;
  return true;
}

}  // namespace tkb
