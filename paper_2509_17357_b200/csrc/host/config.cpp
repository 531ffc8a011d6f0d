// cronus/model.hpp implementation: link model, policy names, validation and the
// `key = value` config codec. Behaviour (accepted keys, error text, %.17g
// round-trip, unknown keys rejected) follows reference proj/src/model.cpp:11-217;
// the codec here is table driven so the serializer and parser share one key list.
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>

#include "cronus/model.hpp"

namespace cronus {

double transfer_time(const LinkModel& link, long long tokens) {
    // Same expression order as the oracle (model.cpp:12); built with -ffp-contract=off.
    return link.latency + link.kv_cost_per_token * static_cast<double>(tokens) / link.bandwidth;
}

namespace {

struct PolicyName {
    Policy p;
    const char* name;
};
constexpr PolicyName kPolicyNames[] = {
    {Policy::Cronus, "cronus"},
    {Policy::DpChunked, "dp"},
    {Policy::PpChunked, "pp"},
    {Policy::DisaggHighLow, "disagg-hl"},
    {Policy::DisaggLowHigh, "disagg-lh"},
};

}  // namespace

const char* policy_name(Policy p) {
    for (const auto& e : kPolicyNames)
        if (e.p == p) return e.name;
    return "?";
}

bool parse_policy(const std::string& s, Policy& out) {
    for (const auto& e : kPolicyNames)
        if (s == e.name) {
            out = e.p;
            return true;
        }
    return false;
}

namespace {

void validate_profile(const GpuProfile& g, const std::string& who, std::vector<std::string>& out) {
    auto need = [&](bool ok, const char* what) {
        if (!ok) out.push_back(who + what);
    };
    need(g.kv_blocks_capacity >= 1, ".kv_blocks_capacity must be >= 1");
    need(g.kv_block_size >= 1, ".kv_block_size must be >= 1");
    need(g.prefill_k >= 0, ".prefill_k must be >= 0");
    need(g.prefill_b >= 0, ".prefill_b must be >= 0");
    need(g.chunked_k_ctxp >= 0, ".chunked_k_ctxp must be >= 0");
    need(g.chunked_k_ctxd >= 0, ".chunked_k_ctxd must be >= 0");
    need(g.chunked_b >= 0, ".chunked_b must be >= 0");
    need(g.total_layers >= 1, ".total_layers must be >= 1");
    need(g.bf16_tflops > 0, ".bf16_tflops must be positive");
}

}  // namespace

std::vector<std::string> validate_config(const ClusterConfig& c) {
    std::vector<std::string> out;
    validate_profile(c.high_gpu, "high", out);
    validate_profile(c.low_gpu, "low", out);
    auto need = [&](bool ok, const std::string& what) {
        if (!ok) out.push_back(what);
    };
    need(c.link.bandwidth > 0, "link.bandwidth must be positive");
    need(c.link.latency >= 0, "link.latency must be >= 0");
    need(c.link.kv_cost_per_token >= 0, "link.kv_cost_per_token must be >= 0");
    need(c.max_batched_tokens_high >= 1, "max_batched_tokens_high must be >= 1");
    need(c.max_batched_tokens_low >= 1, "max_batched_tokens_low must be >= 1");
    need(c.dp_weight_high >= 1, "dp_weight_high must be >= 1");
    need(c.dp_weight_low >= 0, "dp_weight_low must be >= 0");
    need(c.dp_queue_cap_high >= 1, "dp_queue_cap_high must be >= 1");
    need(c.dp_queue_cap_low >= 1, "dp_queue_cap_low must be >= 1");
    need(c.ppi_max_inflight >= 1, "ppi_max_inflight must be >= 1");
    need(c.pp_comm_ms >= 0, "pp_comm_ms must be >= 0");
    const bool pp_split_given = c.pp_layers_high != 0 || c.pp_layers_low != 0;
    if (pp_split_given) {
        need(c.high_gpu.total_layers == c.low_gpu.total_layers,
             "high.total_layers/low.total_layers: profiles disagree on model depth");
        if (c.pp_layers_high < 1 || c.pp_layers_low < 1) {
            out.push_back("pp_layers_high/pp_layers_low must be >= 1");
        } else if (c.pp_layers_high + c.pp_layers_low != c.high_gpu.total_layers) {
            out.push_back("pp_layers_high/pp_layers_low: layer split mismatch (" +
                          std::to_string(c.pp_layers_high) + "+" +
                          std::to_string(c.pp_layers_low) + " != " +
                          std::to_string(c.high_gpu.total_layers) + ")");
        }
    } else if (c.policy == Policy::PpChunked) {
        out.push_back("pp_layers_high/pp_layers_low required for the pp policy");
    }
    return out;
}

namespace {

std::string g17(double v) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

// One entry per config key, in canonical serialization order. `get` renders the
// value; `set` parses it (throwing through `fail` on malformed input).
struct Key {
    std::string name;
    std::function<std::string(const ClusterConfig&)> get;
    std::function<void(ClusterConfig&, const std::string&)> set;
};

[[noreturn]] void fail_line(int line, const std::string& msg) {
    throw std::runtime_error("config line " + std::to_string(line) + ": " + msg);
}

thread_local int g_line = 0;  // line being parsed, for error messages

long long to_int(const std::string& key, const std::string& v) {
    try {
        return std::stoll(v);
    } catch (...) {
        fail_line(g_line, "bad integer for " + key);
    }
}

double to_dbl(const std::string& key, const std::string& v) {
    try {
        return std::stod(v);
    } catch (...) {
        fail_line(g_line, "bad number for " + key);
    }
}

template <class T>
Key int_key(const std::string& name, T ClusterConfig::*m) {
    return {name, [m](const ClusterConfig& c) { return std::to_string(c.*m); },
            [m, name](ClusterConfig& c, const std::string& v) {
                c.*m = static_cast<T>(to_int(name, v));
            }};
}

Key dbl_key(const std::string& name, std::function<double&(ClusterConfig&)> ref) {
    return {name, [ref](const ClusterConfig& c) { return g17(ref(const_cast<ClusterConfig&>(c))); },
            [ref, name](ClusterConfig& c, const std::string& v) { ref(c) = to_dbl(name, v); }};
}

void add_profile_keys(std::vector<Key>& keys, const std::string& pfx,
                      GpuProfile ClusterConfig::*gp) {
    auto P = [gp](ClusterConfig& c) -> GpuProfile& { return c.*gp; };
    keys.push_back({pfx + ".name", [gp](const ClusterConfig& c) { return (c.*gp).name; },
                    [P](ClusterConfig& c, const std::string& v) { P(c).name = v; }});
    keys.push_back({pfx + ".kv_blocks_capacity",
                    [gp](const ClusterConfig& c) { return std::to_string((c.*gp).kv_blocks_capacity); },
                    [P, pfx](ClusterConfig& c, const std::string& v) {
                        P(c).kv_blocks_capacity = to_int(pfx + ".kv_blocks_capacity", v);
                    }});
    keys.push_back({pfx + ".kv_block_size",
                    [gp](const ClusterConfig& c) { return std::to_string((c.*gp).kv_block_size); },
                    [P, pfx](ClusterConfig& c, const std::string& v) {
                        P(c).kv_block_size = static_cast<int>(to_int(pfx + ".kv_block_size", v));
                    }});
    keys.push_back(dbl_key(pfx + ".prefill_k", [P](ClusterConfig& c) -> double& { return P(c).prefill_k; }));
    keys.push_back(dbl_key(pfx + ".prefill_b", [P](ClusterConfig& c) -> double& { return P(c).prefill_b; }));
    keys.push_back(dbl_key(pfx + ".chunked_k_ctxp", [P](ClusterConfig& c) -> double& { return P(c).chunked_k_ctxp; }));
    keys.push_back(dbl_key(pfx + ".chunked_k_ctxd", [P](ClusterConfig& c) -> double& { return P(c).chunked_k_ctxd; }));
    keys.push_back(dbl_key(pfx + ".chunked_b", [P](ClusterConfig& c) -> double& { return P(c).chunked_b; }));
    keys.push_back({pfx + ".total_layers",
                    [gp](const ClusterConfig& c) { return std::to_string((c.*gp).total_layers); },
                    [P, pfx](ClusterConfig& c, const std::string& v) {
                        P(c).total_layers = static_cast<int>(to_int(pfx + ".total_layers", v));
                    }});
    keys.push_back(dbl_key(pfx + ".bf16_tflops", [P](ClusterConfig& c) -> double& { return P(c).bf16_tflops; }));
}

const std::vector<Key>& key_table() {
    static const std::vector<Key> keys = [] {
        std::vector<Key> k;
        k.push_back({"policy", [](const ClusterConfig& c) { return std::string(policy_name(c.policy)); },
                     [](ClusterConfig& c, const std::string& v) {
                         if (!parse_policy(v, c.policy)) fail_line(g_line, "unknown policy '" + v + "'");
                     }});
        k.push_back(int_key("seed", &ClusterConfig::seed));
        k.push_back(int_key("max_batched_tokens_high", &ClusterConfig::max_batched_tokens_high));
        k.push_back(int_key("max_batched_tokens_low", &ClusterConfig::max_batched_tokens_low));
        k.push_back(int_key("dp_weight_high", &ClusterConfig::dp_weight_high));
        k.push_back(int_key("dp_weight_low", &ClusterConfig::dp_weight_low));
        k.push_back(int_key("dp_queue_cap_high", &ClusterConfig::dp_queue_cap_high));
        k.push_back(int_key("dp_queue_cap_low", &ClusterConfig::dp_queue_cap_low));
        k.push_back(int_key("pp_layers_high", &ClusterConfig::pp_layers_high));
        k.push_back(int_key("pp_layers_low", &ClusterConfig::pp_layers_low));
        k.push_back(dbl_key("pp_comm_ms", [](ClusterConfig& c) -> double& { return c.pp_comm_ms; }));
        k.push_back(int_key("ppi_max_inflight", &ClusterConfig::ppi_max_inflight));
        k.push_back(dbl_key("link.bandwidth", [](ClusterConfig& c) -> double& { return c.link.bandwidth; }));
        k.push_back(dbl_key("link.latency", [](ClusterConfig& c) -> double& { return c.link.latency; }));
        k.push_back(dbl_key("link.kv_cost_per_token",
                            [](ClusterConfig& c) -> double& { return c.link.kv_cost_per_token; }));
        add_profile_keys(k, "high", &ClusterConfig::high_gpu);
        add_profile_keys(k, "low", &ClusterConfig::low_gpu);
        return k;
    }();
    return keys;
}

std::string strip(const std::string& s) {
    const char* ws = " \t\r";
    size_t a = s.find_first_not_of(ws);
    if (a == std::string::npos) return {};
    return s.substr(a, s.find_last_not_of(ws) - a + 1);
}

}  // namespace

std::string serialize_config(const ClusterConfig& cfg) {
    std::string out;
    for (const auto& k : key_table()) out += k.name + " = " + k.get(cfg) + "\n";
    return out;
}

ClusterConfig parse_config(const std::string& text) {
    ClusterConfig cfg;
    std::istringstream in(text);
    std::string raw;
    g_line = 0;
    while (std::getline(in, raw)) {
        ++g_line;
        const std::string s = strip(raw);
        if (s.empty() || s[0] == '#') continue;
        const size_t eq = s.find('=');
        if (eq == std::string::npos) fail_line(g_line, "expected 'key = value'");
        const std::string key = strip(s.substr(0, eq));
        const std::string val = strip(s.substr(eq + 1));
        bool known = false;
        for (const auto& k : key_table())
            if (k.name == key) {
                k.set(cfg, val);
                known = true;
                break;
            }
        if (!known) fail_line(g_line, "unknown key " + key);
    }
    return cfg;
}

ClusterConfig load_config(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot open config file: " + path);
    std::ostringstream ss;
    ss << f.rdbuf();
    return parse_config(ss.str());
}

void save_config(const ClusterConfig& cfg, const std::string& path) {
    std::ofstream f(path);
    if (!f) throw std::runtime_error("cannot write config file: " + path);
    f << serialize_config(cfg);
}

}  // namespace cronus
