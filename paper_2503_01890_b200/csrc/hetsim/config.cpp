// [model]/[hardware] key = value configuration. Behaviour (accepted grammar, unit
// conversions, diagnostics "origin:line: message") follows
// /root/reference/proj/core/src/config.cpp:17-209: '#' comments, unknown sections/keys and
// duplicates rejected, GiB -> bytes via llround, TFLOPS x1e12, GB/s x1e9, Mparams/s x1e6.
#include "hetsim/config.hpp"

#include <cmath>
#include <cstdint>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

namespace hetsim {

namespace {

struct Value {
    std::string text;
    int line = 0;
};

class Ini {
public:
    Ini(const std::string& text, std::string origin) : origin_(std::move(origin)) {
        std::istringstream in(text);
        std::string raw, section;
        for (int ln = 1; std::getline(in, raw); ++ln) {
            std::string line = strip(raw.substr(0, raw.find('#')));
            if (line.empty()) continue;
            if (line[0] == '[') {
                if (line.back() != ']') die(ln, "malformed section header '" + line + "'");
                section = strip(line.substr(1, line.size() - 2));
                if (section != "model" && section != "hardware")
                    die(ln, "unknown section '" + section + "' (expected [model] or [hardware])");
                sections_[section];
                continue;
            }
            const std::size_t eq = line.find('=');
            if (eq == std::string::npos) die(ln, "expected 'key = value', got '" + line + "'");
            if (section.empty()) die(ln, "key before any [model]/[hardware] section");
            const std::string key = strip(line.substr(0, eq));
            const std::string val = strip(line.substr(eq + 1));
            if (key.empty() || val.empty()) die(ln, "empty key or value");
            auto& sec = sections_[section];
            auto found = sec.find(key);
            if (found != sec.end())
                die(ln, "duplicate key '" + key + "' in [" + section + "] (first on line " +
                            std::to_string(found->second.line) + ")");
            sec[key] = Value{val, ln};
        }
    }

    [[noreturn]] void die(int line, const std::string& msg) const {
        std::string where = origin_;
        if (line > 0) where += ":" + std::to_string(line);
        throw ConfigError(where + ": " + msg);
    }

    const std::map<std::string, Value>* section(const std::string& name) const {
        auto it = sections_.find(name);
        return it == sections_.end() ? nullptr : &it->second;
    }

    static std::string strip(const std::string& s) {
        const char* ws = " \t\r";
        const std::size_t a = s.find_first_not_of(ws);
        if (a == std::string::npos) return "";
        return s.substr(a, s.find_last_not_of(ws) - a + 1);
    }

private:
    std::string origin_;
    std::map<std::string, std::map<std::string, Value>> sections_;
};

// Reads typed fields out of one section and remembers which keys were consumed, so
// leftovers can be reported as unknown.
class Fields {
public:
    Fields(const Ini& ini, const std::string& name) : ini_(ini), name_(name) {
        sec_ = ini.section(name);
        if (!sec_) ini.die(0, "missing required section [" + name + "]");
    }

    double real(const std::string& key) { return parse(need(key), key); }
    double real(const std::string& key, double dflt) {
        const Value* v = get(key);
        return v ? parse(*v, key) : dflt;
    }
    std::int64_t whole(const std::string& key) { return integral(need(key), key); }
    std::optional<std::int64_t> maybe_whole(const std::string& key) {
        const Value* v = get(key);
        if (!v) return std::nullopt;
        return integral(*v, key);
    }
    void done() const {
        for (const auto& kv : *sec_)
            if (!used_.count(kv.first))
                ini_.die(kv.second.line, "unknown field '" + kv.first + "' in [" + name_ + "]");
    }

private:
    const Value* get(const std::string& key) {
        used_.insert(key);
        auto it = sec_->find(key);
        return it == sec_->end() ? nullptr : &it->second;
    }
    const Value& need(const std::string& key) {
        const Value* v = get(key);
        if (!v) ini_.die(0, "missing required field '" + key + "' in [" + name_ + "]");
        return *v;
    }
    double parse(const Value& v, const std::string& key) const {
        std::size_t used = 0;
        double x = 0.0;
        bool ok = true;
        try {
            x = std::stod(v.text, &used);
        } catch (const std::exception&) {
            ok = false;
        }
        if (!ok || used != v.text.size())
            ini_.die(v.line, "field '" + key + "': cannot parse '" + v.text + "' as a number");
        return x;
    }
    std::int64_t integral(const Value& v, const std::string& key) const {
        const double x = parse(v, key);
        if (x != std::floor(x)) ini_.die(v.line, "field '" + key + "' must be an integer");
        return static_cast<std::int64_t>(x);
    }

    const Ini& ini_;
    std::string name_;
    const std::map<std::string, Value>* sec_ = nullptr;
    std::set<std::string> used_;
};

std::int64_t gib_to_bytes(double gib) {
    return static_cast<std::int64_t>(std::llround(gib * (1024.0 * 1024.0 * 1024.0)));
}

}  // namespace

RunConfig parse_config(const std::string& text, const std::string& origin) {
    const Ini ini(text, origin);
    RunConfig cfg;

    Fields m(ini, "model");
    cfg.model.num_blocks = static_cast<int>(m.whole("num_blocks"));
    cfg.model.hidden_size = m.whole("hidden_size");
    cfg.model.seq_len = m.whole("seq_len");
    cfg.model.batch_size = m.whole("batch_size");
    cfg.model.vocab_size = m.whole("vocab_size");
    cfg.model.activation_coef = m.real("activation_coef", 16.0);
    cfg.model.bwd_fwd_ratio = m.real("bwd_fwd_ratio", 2.0);
    cfg.overrides.m_gc = m.maybe_whole("m_gc_bytes");
    cfg.overrides.m_cc = m.maybe_whole("m_cc_bytes");
    m.done();

    Fields h(ini, "hardware");
    cfg.hardware.gpu_mem = gib_to_bytes(h.real("gpu_mem_gib"));
    cfg.hardware.cpu_mem = gib_to_bytes(h.real("cpu_mem_gib"));
    cfg.hardware.gpu_compute_rate = h.real("gpu_tflops") * 1e12;
    cfg.hardware.h2d_bandwidth = h.real("h2d_gbps") * 1e9;
    cfg.hardware.d2h_bandwidth = h.real("d2h_gbps") * 1e9;
    cfg.hardware.cpu_optim_rate = h.real("cpu_optim_mparams_s") * 1e6;
    cfg.hardware.gpu_optim_rate = h.real("gpu_optim_mparams_s") * 1e6;
    h.done();

    try {
        cfg.model.validate();
        cfg.hardware.validate();
    } catch (const std::invalid_argument& e) {
        throw ConfigError(origin + ": " + e.what());
    }
    return cfg;
}

RunConfig load_config(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw ConfigError(path + ": cannot open config file");
    std::stringstream ss;
    ss << f.rdbuf();
    return parse_config(ss.str(), path);
}

}  // namespace hetsim
