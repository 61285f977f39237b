// Host-side analysis API of the reference, over the
// B200 engine:
//   * RunReport aggregation + JSON/CSV emission  proj/src/report.cpp:51-173
//   * the ESPEC1 model file (load and save)       proj/src/model_io.cpp:18-190
//   * the fuzzy-vs-precise similarity probe       proj/src/draft_engine.cpp:291-372
// Host arithmetic follows the reference statement by statement (same sums in
// the same order, doubles where it uses doubles), so the numbers agree bit for
// bit given the same inputs; the probe's forward passes run on the GPU.
#include "host_api.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

namespace espec {

namespace {

[[noreturn]] void io_fail(const std::string& m) { throw Error(ST_IO, m); }

// ---- minimal JSON reader (the ESPEC1 header: objects, arrays, strings,
// numbers, literals) ----------------------------------------------------------
struct JVal {
    enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
    double num = 0;
    std::string raw;  // number text (integers are re-read exactly)
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal& at(const std::string& k) const {
        if (kind == OBJ)
            for (const auto& kv : obj)
                if (kv.first == k) return kv.second;
        throw std::out_of_range("key '" + k + "' not found");
    }
    long long as_int() const {
        if (kind != NUM) throw std::out_of_range("expected a number");
        long long v = 0;
        const auto r = std::from_chars(raw.data(), raw.data() + raw.size(), v);
        if (r.ec != std::errc() || r.ptr != raw.data() + raw.size()) throw std::out_of_range("expected an integer");
        return v;
    }
    unsigned long long as_u64() const {
        if (kind != NUM) throw std::out_of_range("expected a number");
        unsigned long long v = 0;
        const auto r = std::from_chars(raw.data(), raw.data() + raw.size(), v);
        if (r.ec != std::errc() || r.ptr != raw.data() + raw.size()) throw std::out_of_range("expected an integer");
        return v;
    }
};

struct JParser {
    const std::string& s;
    size_t i = 0;
    explicit JParser(const std::string& t) : s(t) {}
    [[noreturn]] void bad(const char* what) {
        throw std::invalid_argument(std::string(what) + " at byte " + std::to_string(i));
    }
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
    }
    JVal parse() {
        JVal v = value();
        ws();
        if (i != s.size()) bad("trailing characters");
        return v;
    }
    JVal value() {
        ws();
        if (i >= s.size()) bad("unexpected end of input");
        JVal v;
        const char c = s[i];
        if (c == '{') {
            v.kind = JVal::OBJ;
            ++i;
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                if (i >= s.size() || s[i] != '"') bad("expected a key");
                std::string k = string();
                ws();
                if (i >= s.size() || s[i] != ':') bad("expected ':'");
                ++i;
                v.obj.emplace_back(std::move(k), value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return v;
                }
                bad("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JVal::ARR;
            ++i;
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return v;
                }
                bad("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::STR;
            v.str = string();
            return v;
        }
        for (const char* lit : {"true", "false", "null"}) {
            const size_t n = std::strlen(lit);
            if (s.compare(i, n, lit) == 0) {
                i += n;
                v.kind = lit[0] == 'n' ? JVal::NUL : JVal::BOOL;
                v.num = lit[0] == 't';
                return v;
            }
        }
        const size_t b = i;
        while (i < s.size() && (std::isdigit((unsigned char)s[i]) || s[i] == '-' || s[i] == '+' || s[i] == '.' ||
                                s[i] == 'e' || s[i] == 'E'))
            ++i;
        if (i == b) bad("unexpected character");
        v.kind = JVal::NUM;
        v.raw = s.substr(b, i - b);
        const auto r = std::from_chars(v.raw.data(), v.raw.data() + v.raw.size(), v.num);
        if (r.ec != std::errc() || r.ptr != v.raw.data() + v.raw.size()) bad("malformed number");
        return v;
    }
    std::string string() {
        ++i;  // opening quote
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                if (++i >= s.size()) bad("bad escape");
                const char e = s[i++];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        if (i + 4 > s.size()) bad("bad \\u escape");
                        const unsigned cp = (unsigned)std::stoul(s.substr(i, 4), nullptr, 16);
                        i += 4;
                        if (cp < 0x80) out += (char)cp;
                        else if (cp < 0x800) {
                            out += (char)(0xC0 | (cp >> 6));
                            out += (char)(0x80 | (cp & 0x3F));
                        } else {
                            out += (char)(0xE0 | (cp >> 12));
                            out += (char)(0x80 | ((cp >> 6) & 0x3F));
                            out += (char)(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: bad("bad escape");
                }
            } else {
                out += s[i++];
            }
        }
        if (i >= s.size()) bad("unterminated string");
        ++i;
        return out;
    }
};

// nlohmann::json's number text for a float stored as double (shortest
// round-trip digits; decimal notation for exponents in [-4, 15), else
// d.ddde±XX) — what the reference's header.dump() writes for norm_eps.
std::string json_double(double x) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    std::string sci(buf, r.ptr);
    const size_t e = sci.find('e');
    std::string mant = sci.substr(0, e);
    const int exp10 = std::stoi(sci.substr(e + 1));
    std::string digits;
    bool neg = false;
    for (char c : mant) {
        if (c == '-') neg = true;
        else if (c != '.') digits += c;
    }
    const int n = (int)digits.size();
    const int k = exp10 + 1;  // decimal point position relative to the digits
    std::string out = neg ? "-" : "";
    if (k > 0 && k <= 15) {
        if (n <= k) out += digits + std::string(k - n, '0') + ".0";
        else out += digits.substr(0, k) + "." + digits.substr(k);
    } else if (k <= 0 && k > -4) {
        out += "0." + std::string(-k, '0') + digits;
    } else {
        out += digits.substr(0, 1);
        out += n > 1 ? "." + digits.substr(1) : "";
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
        out += eb;
    }
    return out;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

// manifest order (proj/src/model_io.cpp:27-45)
std::vector<ModelFileTensor> manifest(const ModelCfg& c) {
    std::vector<ModelFileTensor> m;
    const int d = c.d_model;
    m.push_back({"embedding", "embedding", -1, c.vocab_size, d});
    m.push_back({"final_norm_gain", "final_norm_gain", -1, 1, d});
    for (int l = 0; l < c.n_layers; ++l) {
        const std::string p = "layers." + std::to_string(l) + ".";
        m.push_back({p + "wq", "wq", l, d, d});
        m.push_back({p + "wk", "wk", l, d, d});
        m.push_back({p + "wv", "wv", l, d, d});
        m.push_back({p + "wo", "wo", l, d, d});
        m.push_back({p + "w_gate", "w_gate", l, d, c.d_mlp});
        m.push_back({p + "w_up", "w_up", l, d, c.d_mlp});
        m.push_back({p + "w_down", "w_down", l, c.d_mlp, d});
        m.push_back({p + "attn_norm_gain", "attn_norm_gain", l, 1, d});
        m.push_back({p + "mlp_norm_gain", "mlp_norm_gain", l, 1, d});
    }
    return m;
}

constexpr char kMagic[] = "ESPEC1\n";

}  // namespace

// ---------------------------------------------------------------------------
// RunReport (proj/src/report.cpp:51-95, 97-173)
// ---------------------------------------------------------------------------

ReportAgg aggregate_traces(const std::vector<IterationTrace>& traces, double vanilla_baseline_sim) {
    if (traces.empty()) throw Error(ST_CONFIG, "cannot aggregate an empty trace list");
    ReportAgg r;
    long emitted = 0, accepted = 0, attempted = 0;
    double d = 0, v = 0, c = 0, ds = 0, vs = 0, cs = 0;
    for (const auto& t : traces) {
        emitted += t.emitted;
        accepted += t.m;
        attempted += t.n;
        // the engine's device stage times (float ms) in seconds, the unit of
        // the reference's IterationTrace wall/sim fields
        d += (double)t.draft_ms / 1000.0;
        v += (double)t.verify_ms / 1000.0;
        c += (double)t.calibrate_ms / 1000.0;
        ds += t.draft_sim;
        vs += t.verify_sim;
        cs += t.calibrate_sim;
    }
    if (emitted <= 0) throw Error(ST_CONFIG, "traces emitted zero tokens");
    r.iterations = (int)traces.size();
    r.tokens_emitted = emitted;
    r.has_alpha = attempted > 0;
    r.alpha = attempted > 0 ? (double)accepted / attempted : 0.0;
    r.mean_accept_len = (double)emitted / (double)traces.size();
    const double per_token = 100.0 / (double)emitted;
    r.draft_per100 = d * per_token;
    r.verify_per100 = v * per_token;
    r.calibrate_per100 = c * per_token;
    r.draft_total_per100 = r.draft_per100 + r.calibrate_per100;
    r.total = d + v + c;
    r.tokens_per_s = r.total > 0.0 ? emitted / r.total : 0.0;
    // simulated units (report.cpp:83-90): the speed-up is the cost model's
    r.draft_per100_sim = ds * per_token;
    r.verify_per100_sim = vs * per_token;
    r.calibrate_per100_sim = cs * per_token;
    r.draft_total_per100_sim = r.draft_per100_sim + r.calibrate_per100_sim;
    r.total_sim = ds + vs + cs;
    r.speedup_vs_vanilla = r.total_sim > 0.0 ? vanilla_baseline_sim / r.total_sim : 1.0;
    return r;
}

std::string report_csv(const ReportAgg& r, const std::string& algorithm, int n, int lp_size) {
    // kReportCsvHeader + report_csv_row (proj/include/espec/report.hpp:64-65, report.cpp:163-171)
    std::ostringstream out;
    out << "algorithm,n,lp_size,alpha,d_per100,v_per100,c_per100,speedup\n";
    out << algorithm << ',' << n << ',' << lp_size << ',';
    if (r.has_alpha) out << r.alpha;
    out << ',' << r.draft_per100_sim << ',' << r.verify_per100_sim << ',' << r.calibrate_per100_sim << ','
        << r.speedup_vs_vanilla << "\n";
    return out.str();
}

std::string report_json(const ReportAgg& r, const std::vector<IterationTrace>& traces, const std::string& algorithm,
                        int n, const std::vector<int>& widths, int lp_size) {
    // emit_report's JSON layout (report.cpp:97-136): "sim" in the cost
    // model's units, "wall" in measured device seconds.
    std::ostringstream o;
    auto num = [](double x) { return json_double(x); };
    o << "{\n  \"algorithm\": " << json_string(algorithm) << ",\n  \"n\": " << n << ",\n  \"widths\": [";
    for (size_t i = 0; i < widths.size(); ++i) o << (i ? ", " : "") << widths[i];
    o << "],\n  \"lp_size\": " << lp_size << ",\n  \"alpha\": " << (r.has_alpha ? num(r.alpha) : "null")
      << ",\n  \"tokens_emitted\": " << r.tokens_emitted << ",\n  \"tokens_per_s_wall\": " << num(r.tokens_per_s);
    const char* blocks[2] = {"sim", "wall"};
    for (int b = 0; b < 2; ++b) {
        o << ",\n  \"" << blocks[b] << "\": {\n    \"draft_per_100\": " << num(b ? r.draft_per100 : r.draft_per100_sim)
          << ",\n    \"verify_per_100\": " << num(b ? r.verify_per100 : r.verify_per100_sim)
          << ",\n    \"calibrate_per_100\": " << num(b ? r.calibrate_per100 : r.calibrate_per100_sim);
        if (b == 0)
            o << ",\n    \"draft_total_per_100\": " << num(r.draft_total_per100_sim) << ",\n    \"total_sim\": "
              << num(r.total_sim) << ",\n    \"total_speedup_vs_vanilla\": " << num(r.speedup_vs_vanilla);
        o << "\n  }";
    }
    o << ",\n  \"config\": {},\n  \"iterations\": [";
    for (size_t i = 0; i < traces.size(); ++i) {
        const auto& t = traces[i];
        const double dw = t.draft_ms / 1000.0, vw = t.verify_ms / 1000.0, cw = t.calibrate_ms / 1000.0;
        o << (i ? "," : "") << "\n    {\"m\": " << t.m << ", \"n\": " << t.n << ", \"drafted_nodes\": "
          << t.drafted_nodes << ", \"emitted\": " << t.emitted << ", \"draft_wall\": " << num(dw)
          << ", \"verify_wall\": " << num(vw) << ", \"calibrate_wall\": " << num(cw) << ", \"draft_sim\": "
          << num(t.draft_sim) << ", \"verify_sim\": " << num(t.verify_sim) << ", \"calibrate_sim\": "
          << num(t.calibrate_sim)
          << ", \"fuzzy_forwards\": " << t.fuzzy_forwards << ", \"sequential_forwards\": " << t.sequential_forwards
          << ", \"base_forwards\": " << t.base_forwards << "}";
    }
    o << (traces.empty() ? "]\n}" : "\n  ]\n}");
    return o.str();
}

// ---------------------------------------------------------------------------
// ESPEC1 model file (proj/src/model_io.cpp)
// ---------------------------------------------------------------------------

ModelFileInfo read_model_file(const std::string& path, bool check_data) {
    // load_model (model_io.cpp:106-190): same checks, same IoError texts
    std::ifstream in(path, std::ios::binary);
    if (!in) io_fail("cannot open model file '" + path + "'");
    char magic[7] = {};
    in.read(magic, 7);
    if (!in || std::memcmp(magic, kMagic, 7) != 0) io_fail("'" + path + "' is not a model file (bad magic)");
    uint64_t header_len = 0;
    in.read(reinterpret_cast<char*>(&header_len), 8);
    if (!in || header_len == 0 || header_len > (1ull << 24)) io_fail("corrupt model header length");
    std::string text(header_len, '\0');
    in.read(text.data(), (std::streamsize)header_len);
    if (!in) io_fail("truncated model header");
    JVal h;
    try {
        h = JParser(text).parse();
    } catch (const std::exception& e) {
        io_fail(std::string("invalid model header JSON: ") + e.what());
    }
    ModelFileInfo info;
    try {
        const JVal& c = h.at("config");
        ModelCfg& m = info.cfg;
        m.vocab_size = (int)c.at("vocab_size").as_int();
        m.d_model = (int)c.at("d_model").as_int();
        m.n_layers = (int)c.at("n_layers").as_int();
        m.n_heads = (int)c.at("n_heads").as_int();
        m.n_kv_heads = m.n_heads;  // the reference model is MHA
        m.d_head = (int)c.at("d_head").as_int();
        m.d_mlp = (int)c.at("d_mlp").as_int();
        m.max_positions = (int)c.at("max_positions").as_int();
        m.norm_eps = (float)c.at("norm_eps").num;
        m.seed = c.at("seed").as_u64();
        m.rope_theta = 10000.f;
        m.tied_head = 1;
        m.weight_dtype = espec_dev::DT_F32;
        m.kv_dtype = espec_dev::DT_F32;
    } catch (const std::exception& e) {
        io_fail(std::string("invalid model header JSON: ") + e.what());
    }
    // ModelConfig::validate (model.cpp:12-24)
    const ModelCfg& m = info.cfg;
    if (m.vocab_size < 2) throw Error(ST_CONFIG, "vocab_size must be >= 2");
    if (m.n_layers < 2) throw Error(ST_CONFIG, "n_layers must be >= 2");
    if (m.n_heads < 1 || m.d_head < 2 || m.d_head % 2 != 0)
        throw Error(ST_CONFIG, "need n_heads >= 1 and an even d_head >= 2");
    if (m.d_model != m.n_heads * m.d_head) throw Error(ST_CONFIG, "d_model must equal n_heads * d_head");
    if (m.d_mlp < 1) throw Error(ST_CONFIG, "d_mlp must be >= 1");
    if (m.max_positions < 2) throw Error(ST_CONFIG, "max_positions must be >= 2");
    if (!(m.norm_eps > 0.0f)) throw Error(ST_CONFIG, "norm_eps must be positive");
    info.tensors = manifest(m);
    const JVal* tensors = nullptr;
    try {
        tensors = &h.at("tensors");
    } catch (const std::exception& e) {
        io_fail(std::string("invalid model header JSON: ") + e.what());
    }
    if (tensors->kind != JVal::ARR || tensors->arr.size() != info.tensors.size())
        io_fail("tensor manifest does not match the config layer count");
    info.data_offset = 7 + 8 + header_len;
    uint64_t off = info.data_offset;
    std::vector<float> buf;
    for (size_t i = 0; i < info.tensors.size(); ++i) {
        ModelFileTensor& t = info.tensors[i];
        std::string name;
        int rows = 0, cols = 0;
        try {
            const JVal& e = tensors->arr[i];
            name = e.at("name").str;
            if (e.at("name").kind != JVal::STR) throw std::out_of_range("tensor name is not a string");
            const JVal& sh = e.at("shape");
            if (sh.kind != JVal::ARR || sh.arr.size() < 2) throw std::out_of_range("bad shape");
            rows = (int)sh.arr[0].as_int();
            cols = (int)sh.arr[1].as_int();
        } catch (const std::exception& x) {
            io_fail(std::string("invalid model header JSON: ") + x.what());
        }
        if (name != t.file_name) io_fail("unexpected tensor '" + name + "', wanted '" + t.file_name + "'");
        if (rows <= 0 || cols <= 0) io_fail("degenerate shape for tensor '" + t.file_name + "'");
        const int want_r = t.rows, want_c = t.cols;
        t.rows = rows;
        t.cols = cols;
        t.offset = off;
        const uint64_t bytes = (uint64_t)rows * cols * sizeof(float);
        if (check_data) {
            buf.resize((size_t)rows * cols);
            in.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)bytes);
            if (!in) io_fail("truncated tensor data for '" + t.file_name + "'");
            for (float x : buf)
                if (!std::isfinite(x)) io_fail("tensor '" + t.file_name + "' contains non-finite values");
        }
        off += bytes;
        t.want_rows = want_r;
        t.want_cols = want_c;
    }
    // shape checks after the whole manifest, as the reference does (model_io.cpp:166-188)
    for (const auto& t : info.tensors)
        if (t.rows != t.want_rows || t.cols != t.want_cols)
            io_fail("tensor '" + t.short_name + "' shape disagrees with config");
    if (!check_data) {
        in.seekg(0, std::ios::end);
        if ((uint64_t)in.tellg() < off) io_fail("truncated tensor data for '" + info.tensors.back().file_name + "'");
    }
    return info;
}

void load_model_file(Engine& eng, int which, const ModelCfg& engine_cfg, const std::string& path) {
    const ModelFileInfo info = read_model_file(path, true);
    const ModelCfg& f = info.cfg;
    const ModelCfg& e = engine_cfg;
    if (f.vocab_size != e.vocab_size || f.d_model != e.d_model || f.n_layers != e.n_layers ||
        f.n_heads != e.n_heads || e.n_kv_heads != e.n_heads || f.d_head != e.d_head || f.d_mlp != e.d_mlp ||
        f.norm_eps != e.norm_eps || !e.tied_head || e.rope_theta != 10000.f)
        throw Error(ST_CONFIG, std::string("model file '") + path + "' does not match the engine's " +
                                   (which ? "base" : "drafter") + " config (ESPEC1 models are MHA, tied head, "
                                   "rope base 10000; vocab, widths, heads, layers and norm_eps must agree)");
    std::ifstream in(path, std::ios::binary);
    std::vector<float> buf;
    for (const auto& t : info.tensors) {
        buf.resize((size_t)t.rows * t.cols);
        in.seekg((std::streamoff)t.offset);
        in.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)(buf.size() * sizeof(float)));
        if (!in) io_fail("truncated tensor data for '" + t.file_name + "'");
        eng.load_tensor(which, t.short_name, t.layer, buf.data(), t.rows, t.cols);
    }
}

void save_model_file(Engine& eng, int which, const ModelCfg& c, const std::string& path) {
    // save_model (model_io.cpp:76-104)
    if (c.n_kv_heads != c.n_heads || !c.tied_head || c.rope_theta != 10000.f || c.d_model != c.n_heads * c.d_head)
        throw Error(ST_CONFIG, "model is not representable in the ESPEC1 format (needs MHA, a tied head, rope base "
                               "10000 and d_model == n_heads * d_head)");
    const auto refs = manifest(c);
    std::ostringstream h;
    h << "{\"config\":{\"vocab_size\":" << c.vocab_size << ",\"d_model\":" << c.d_model
      << ",\"n_layers\":" << c.n_layers << ",\"n_heads\":" << c.n_heads << ",\"d_head\":" << c.d_head
      << ",\"d_mlp\":" << c.d_mlp << ",\"max_positions\":" << c.max_positions
      << ",\"norm_eps\":" << json_double((double)c.norm_eps) << ",\"seed\":" << c.seed << "},\"tensors\":[";
    for (size_t i = 0; i < refs.size(); ++i)
        h << (i ? "," : "") << "{\"name\":" << json_string(refs[i].file_name) << ",\"shape\":[" << refs[i].rows
          << "," << refs[i].cols << "]}";
    h << "]}";
    const std::string text = h.str();
    std::ofstream out(path, std::ios::binary);
    if (!out) io_fail("cannot open '" + path + "' for writing");
    out.write(kMagic, 7);
    const uint64_t len = text.size();
    out.write(reinterpret_cast<const char*>(&len), 8);
    out.write(text.data(), (std::streamsize)text.size());
    std::vector<float> buf;
    for (const auto& t : refs) {
        buf.resize((size_t)t.rows * t.cols);
        eng.weight(which, t.short_name, t.layer, buf.data(), t.rows, t.cols);
        out.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(buf.size() * sizeof(float)));
    }
    if (!out) io_fail("short write to '" + path + "'");
}

// ---------------------------------------------------------------------------
// Similarity probe (proj/src/draft_engine.cpp:291-372, cosine_sim
// proj/src/matrix.cpp:139-157)
// ---------------------------------------------------------------------------

namespace {

double cosine(const float* a, const float* b, size_t n) {
    if (n == 0) throw Error(ST_SHAPE, "cosine_sim requires equal non-empty widths");
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (size_t i = 0; i < n; ++i) {
        dot += static_cast<double>(a[i]) * b[i];
        na += static_cast<double>(a[i]) * a[i];
        nb += static_cast<double>(b[i]) * b[i];
    }
    if (na == 0.0 && nb == 0.0) throw Error(ST_DOMAIN, "cosine similarity of two zero vectors is undefined");
    if (na == 0.0 || nb == 0.0) return 0.0;
    const double cs = dot / std::sqrt(na * nb);
    return std::min(1.0, std::max(-1.0, cs));
}

struct Acc {
    double sum = 0.0;
    long count = 0;
    void add(double v) {
        sum += v;
        ++count;
    }
    double mean() const { return count > 0 ? sum / count : 1.0; }
};

}  // namespace

std::vector<SimilarityRow> probe_similarity(Engine& eng, int n_layers, const std::vector<int>& lp_sizes,
                                            const std::vector<std::vector<int>>& corpus) {
    if (corpus.empty()) throw Error(ST_CONFIG, "similarity probe needs a non-empty corpus");
    std::vector<SimilarityRow> rows;
    for (int lp : lp_sizes) {
        const LayerPlan plan = plan_groups(n_layers, lp);
        std::vector<int> par;  // LayerPlan::parallelized_layers (layer_plan.cpp:24-30)
        for (const auto& g : plan.groups)
            if (g.size() >= 2) par.insert(par.end(), g.begin(), g.end());
        Acc h, q, k, v, ao;
        const std::string spec = format_plan(plan);
        for (const auto& seq : corpus) {
            std::vector<LayerCapture> fz, pr;
            eng.forward_capture(0, seq, spec, fz);
            eng.forward_capture(0, seq, "", pr);
            const size_t T = seq.size();
            auto add_rows = [&](Acc& acc, const std::vector<float>& a, const std::vector<float>& b) {
                const size_t w = a.size() / T;
                for (size_t r = 0; r < T; ++r) acc.add(cosine(a.data() + r * w, b.data() + r * w, w));
            };
            for (int l : par) {
                add_rows(h, fz[l].h_in, pr[l].h_in);
                add_rows(q, fz[l].q, pr[l].q);
                add_rows(k, fz[l].k, pr[l].k);
                add_rows(v, fz[l].v, pr[l].v);
                add_rows(ao, fz[l].attn_out, pr[l].attn_out);
            }
        }
        rows.push_back({lp, h.mean(), q.mean(), k.mean(), v.mean(), ao.mean()});
    }
    return rows;
}

std::string similarity_csv(const std::vector<SimilarityRow>& rows) {
    std::ostringstream out;
    out << "lp_size,h,q,k,v,attnoutput\n";
    out.precision(6);
    out << std::fixed;
    for (const auto& r : rows)
        out << r.lp_size << ',' << r.h << ',' << r.q << ',' << r.k << ',' << r.v << ',' << r.attn_out << '\n';
    return out.str();
}

}  // namespace espec
