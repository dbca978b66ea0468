// Plan / strategy / manifest documents (reference: proj/core/src/plan_io.cpp:15-105).
//
// The reference serialises through nlohmann::json dump(2). We carry our own small JSON
// tree with the same observable output: object keys sorted, two-space indent, doubles in
// shortest round-trip form with nlohmann's notation rules (".0" on integral values,
// exponent form outside 1e-5 < |x| < 1e15, two-digit exponents), and integer arrays
// written inline as the in-container nlohmann 3.11.3 build does. read_strategy_json
// accepts a full plan or a bare strategy object, like the reference.
#include "hetsim/plan_io.hpp"

#include <charconv>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <ostream>
#include <sstream>
#include <variant>

#include "hetsim/version.hpp"

namespace hetsim {

namespace {

struct Json;
using JsonObject = std::map<std::string, Json>;
using JsonArray = std::vector<Json>;

struct Json {
    enum Kind { Null, Bool, Int, Real, Str, Arr, Obj } kind = Null;
    bool b = false;
    std::int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::shared_ptr<JsonArray> arr;
    std::shared_ptr<JsonObject> obj;

    static Json integer(std::int64_t v) { Json j; j.kind = Int; j.i = v; return j; }
    static Json real(double v) { Json j; j.kind = Real; j.d = v; return j; }
    static Json text(std::string v) { Json j; j.kind = Str; j.s = std::move(v); return j; }
    static Json array() { Json j; j.kind = Arr; j.arr = std::make_shared<JsonArray>(); return j; }
    static Json object() { Json j; j.kind = Obj; j.obj = std::make_shared<JsonObject>(); return j; }
    Json& operator[](const std::string& k) { return (*obj)[k]; }
};

// nlohmann-compatible double text from the shortest round-trip digits.
std::string format_double(double x) {
    if (!std::isfinite(x)) return "null";
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    std::string sci(buf, res.ptr);  // e.g. "-1.2345e+03"
    std::string out;
    std::size_t pos = 0;
    if (sci[0] == '-') { out.push_back('-'); pos = 1; }
    const std::size_t epos = sci.find('e');
    std::string digits;
    for (std::size_t q = pos; q < epos; ++q)
        if (sci[q] != '.') digits.push_back(sci[q]);
    const int exp10 = std::atoi(sci.c_str() + epos + 1);
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // value = 0.d1d2... x 10^n
    if (k <= n && n <= 15) {
        out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, static_cast<std::size_t>(n)) + "." +
               digits.substr(static_cast<std::size_t>(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        out += e < 0 ? "e-" : "e+";
        const int ae = e < 0 ? -e : e;
        if (ae < 10) out += "0";
        out += std::to_string(ae);
    }
    return out;
}

std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            case '\r': o += "\\r"; break;
            default: o.push_back(c);
        }
    }
    return o + "\"";
}

void dump(std::ostream& out, const Json& j, int indent) {
    const std::string pad(static_cast<std::size_t>(indent), ' ');
    const std::string pad2(static_cast<std::size_t>(indent + 2), ' ');
    switch (j.kind) {
        case Json::Null: out << "null"; break;
        case Json::Bool: out << (j.b ? "true" : "false"); break;
        case Json::Int: out << j.i; break;
        case Json::Real: out << format_double(j.d); break;
        case Json::Str: out << quote(j.s); break;
        case Json::Arr: {
            if (j.arr->empty()) { out << "[]"; break; }
            if ((*j.arr)[0].kind == Json::Int) {  // integer arrays inline
                out << "[";
                for (std::size_t q = 0; q < j.arr->size(); ++q) {
                    if (q) out << ",";
                    dump(out, (*j.arr)[q], indent);
                }
                out << "]";
                break;
            }
            out << "[\n";
            for (std::size_t q = 0; q < j.arr->size(); ++q) {
                out << pad2;
                dump(out, (*j.arr)[q], indent + 2);
                out << (q + 1 < j.arr->size() ? ",\n" : "\n");
            }
            out << pad << "]";
            break;
        }
        case Json::Obj: {
            if (j.obj->empty()) { out << "{}"; break; }
            out << "{\n";
            std::size_t q = 0;
            for (const auto& kv : *j.obj) {
                out << pad2 << quote(kv.first) << ": ";
                dump(out, kv.second, indent + 2);
                out << (++q < j.obj->size() ? ",\n" : "\n");
            }
            out << pad << "}";
            break;
        }
    }
}

// ---- minimal parser (enough for plan / strategy documents) ----
class Parser {
public:
    explicit Parser(const std::string& t) : t_(t) {}
    Json parse_document() {
        Json v = value();
        ws();
        if (p_ != t_.size()) fail("trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& m) const {
        throw std::runtime_error("parse error at byte " + std::to_string(p_) + ": " + m);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r'))
            ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < t_.size() && t_[p_] == c) { ++p_; return true; }
        return false;
    }
    Json value() {
        ws();
        if (p_ >= t_.size()) fail("unexpected end of input");
        const char c = t_[p_];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') return Json::text(string());
        if (t_.compare(p_, 4, "true") == 0) { p_ += 4; Json j; j.kind = Json::Bool; j.b = true; return j; }
        if (t_.compare(p_, 5, "false") == 0) { p_ += 5; Json j; j.kind = Json::Bool; return j; }
        if (t_.compare(p_, 4, "null") == 0) { p_ += 4; return Json{}; }
        return number();
    }
    Json object() {
        Json j = Json::object();
        eat('{');
        if (eat('}')) return j;
        do {
            ws();
            if (p_ >= t_.size() || t_[p_] != '"') fail("expected object key");
            std::string k = string();
            if (!eat(':')) fail("expected ':'");
            (*j.obj)[k] = value();
        } while (eat(','));
        if (!eat('}')) fail("expected '}'");
        return j;
    }
    Json array() {
        Json j = Json::array();
        eat('[');
        if (eat(']')) return j;
        do j.arr->push_back(value());
        while (eat(','));
        if (!eat(']')) fail("expected ']'");
        return j;
    }
    std::string string() {
        std::string s;
        ++p_;
        while (p_ < t_.size() && t_[p_] != '"') {
            if (t_[p_] == '\\' && p_ + 1 < t_.size()) {
                ++p_;
                const char e = t_[p_];
                s.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e);
            } else {
                s.push_back(t_[p_]);
            }
            ++p_;
        }
        if (p_ >= t_.size()) fail("unterminated string");
        ++p_;
        return s;
    }
    Json number() {
        const std::size_t a = p_;
        bool is_real = false;
        if (p_ < t_.size() && t_[p_] == '-') ++p_;
        while (p_ < t_.size()) {
            const char c = t_[p_];
            if (c >= '0' && c <= '9') { ++p_; continue; }
            if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { is_real = true; ++p_; continue; }
            break;
        }
        if (p_ == a) fail("unexpected character");
        const std::string tok = t_.substr(a, p_ - a);
        if (!is_real) return Json::integer(std::stoll(tok));
        return Json::real(std::stod(tok));
    }

    const std::string& t_;
    std::size_t p_ = 0;
};

const Json& member(const Json& obj, const std::string& key) {
    if (obj.kind != Json::Obj) throw std::runtime_error("type must be object");
    auto it = obj.obj->find(key);
    if (it == obj.obj->end()) throw std::runtime_error("key '" + key + "' not found");
    return it->second;
}

int as_int(const Json& j) {
    if (j.kind == Json::Int) return static_cast<int>(j.i);
    if (j.kind == Json::Real) return static_cast<int>(j.d);
    throw std::runtime_error("type must be number");
}

Json int_array(const std::vector<int>& v) {
    Json a = Json::array();
    for (int x : v) a.arr->push_back(Json::integer(x));
    return a;
}

}  // namespace

void write_plan_json(std::ostream& out, const PlanDocument& doc) {
    Json root = Json::object();
    Json st = Json::object();
    st["c_hat"] = Json::integer(doc.strategy.c_hat);
    st["p_hat"] = Json::integer(doc.strategy.p_hat);
    st["o_hat"] = Json::integer(doc.strategy.o_hat);
    st["prefetch_lookahead"] = int_array(doc.strategy.prefetch_lookahead);
    root["strategy"] = st;

    Json cost = Json::object();
    cost["t_fwd_s"] = Json::real(doc.cost.t_fwd);
    cost["t_bwd_s"] = Json::real(doc.cost.t_bwd);
    cost["t_sync_s"] = Json::real(doc.cost.t_sync);
    cost["v_hat"] = Json::integer(doc.cost.v_hat);
    cost["peak_gpu_bytes"] = Json::integer(doc.cost.peak_gpu);
    cost["cpu_bytes"] = Json::integer(doc.cost.cpu_bytes);
    cost["objective_s"] = Json::real(doc.cost.objective);
    root["cost"] = cost;

    Json margins = Json::object();
    margins["gpu_bytes"] = Json::integer(doc.gpu_margin);
    margins["cpu_bytes"] = Json::integer(doc.cpu_margin);
    root["margins"] = margins;

    Json search = Json::object();
    search["feasible_count"] = Json::integer(doc.feasible_count);
    root["search"] = search;

    dump(out, root, 0);
    out << "\n";
}

Strategy read_strategy_json(const std::string& path, int num_blocks) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error(path + ": cannot open strategy file");
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    Strategy s;
    try {
        const Json root = Parser(text).parse_document();
        const Json* src = &root;
        if (root.kind == Json::Obj && root.obj->count("strategy")) src = &root.obj->at("strategy");
        s.c_hat = as_int(member(*src, "c_hat"));
        s.p_hat = as_int(member(*src, "p_hat"));
        s.o_hat = as_int(member(*src, "o_hat"));
        if (src->obj->count("prefetch_lookahead")) {
            const Json& la = src->obj->at("prefetch_lookahead");
            if (la.kind != Json::Arr) throw std::runtime_error("prefetch_lookahead must be an array");
            for (const Json& e : *la.arr) s.prefetch_lookahead.push_back(as_int(e));
        }
    } catch (const std::runtime_error& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
    if (s.prefetch_lookahead.empty())
        s.prefetch_lookahead.assign(static_cast<std::size_t>(num_blocks), 1);
    s.validate(num_blocks);
    return s;
}

void write_manifest(std::ostream& out, const RunManifest& mf) {
    Json root = Json::object();
    root["command"] = Json::text(mf.command);
    Json model = Json::object();
    model["num_blocks"] = Json::integer(mf.model.num_blocks);
    model["hidden_size"] = Json::integer(mf.model.hidden_size);
    model["seq_len"] = Json::integer(mf.model.seq_len);
    model["batch_size"] = Json::integer(mf.model.batch_size);
    model["vocab_size"] = Json::integer(mf.model.vocab_size);
    model["activation_coef"] = Json::real(mf.model.activation_coef);
    model["bwd_fwd_ratio"] = Json::real(mf.model.bwd_fwd_ratio);
    root["model"] = model;
    Json hw = Json::object();
    hw["gpu_mem_bytes"] = Json::integer(mf.hardware.gpu_mem);
    hw["cpu_mem_bytes"] = Json::integer(mf.hardware.cpu_mem);
    hw["gpu_compute_flops"] = Json::real(mf.hardware.gpu_compute_rate);
    hw["h2d_bytes_s"] = Json::real(mf.hardware.h2d_bandwidth);
    hw["d2h_bytes_s"] = Json::real(mf.hardware.d2h_bandwidth);
    hw["cpu_optim_params_s"] = Json::real(mf.hardware.cpu_optim_rate);
    hw["gpu_optim_params_s"] = Json::real(mf.hardware.gpu_optim_rate);
    root["hardware"] = hw;
    Json outs = Json::array();
    for (const auto& o : mf.outputs) outs.arr->push_back(Json::text(o));
    root["outputs"] = outs;
    root["determinism"] = Json::text(
        "outputs are a pure function of the configuration; no seeds, timestamps, or machine "
        "state involved");
    root["version"] = Json::text(kVersion);
    dump(out, root, 0);
    out << "\n";
}

}  // namespace hetsim
