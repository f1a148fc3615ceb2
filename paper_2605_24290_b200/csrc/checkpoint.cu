// Scene / model load and save: the reference's RXGS checkpoint container
// (io::save_checkpoint / io::load_checkpoint, src/checkpoint.cpp:93-231,
// format include/rxgs/checkpoint.hpp:10-15):
//
//   "RXGS" | u32 version (1) | u64 header length | JSON header | f64 arrays
//
// The JSON header holds k, l_max, channels, modality, the spherical grid,
// has_conditioning, the conditioning config (with the occupancy bounds) and
// a manifest of named f64 arrays {name, dtype, shape, offset}; the arrays
// follow little-endian in manifest order.  The reference parses the header
// with nlohmann::json (not shipped with it); this file carries its own small
// JSON reader/writer for exactly that schema.  Host code only: loading ends
// in rxgs_scene_create / rxgs_cond_create (device upload).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rxgs_internal.cuh"

namespace rxgs_b200 {
namespace {

// The reference's io::IoError (include/rxgs/dataset.hpp:16).
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ JSON
struct Json {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;  // insertion order (ordered_json)

    const Json& at(const std::string& key) const {
        if (kind == Object)
            for (const auto& kv : obj)
                if (kv.first == key) return kv.second;
        throw IoError("load_checkpoint: header key '" + key + "' missing");
    }
    double number() const {
        if (kind != Number) throw IoError("load_checkpoint: header value is not a number");
        return num;
    }
    int integer() const { return static_cast<int>(number()); }
    bool boolean() const {
        if (kind != Bool) throw IoError("load_checkpoint: header value is not a boolean");
        return b;
    }
    const std::string& string() const {
        if (kind != String) throw IoError("load_checkpoint: header value is not a string");
        return str;
    }
};

struct Parser {
    const std::string& s;
    size_t i = 0;
    explicit Parser(const std::string& text) : s(text) {}
    [[noreturn]] void bad(const char* what) const {
        throw IoError(std::string("load_checkpoint: header parse failure: ") + what + " at byte " +
                      std::to_string(i));
    }
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (s.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    std::string parse_string() {
        if (s[i] != '"') bad("expected string");
        ++i;
        std::string out;
        while (i < s.size() && s[i] != '"') {
            char c = s[i++];
            if (c == '\\') {
                if (i >= s.size()) bad("bad escape");
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
                        const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(i, 4), nullptr, 16));
                        i += 4;
                        if (cp < 0x80) {
                            out += static_cast<char>(cp);
                        } else if (cp < 0x800) {
                            out += static_cast<char>(0xC0 | (cp >> 6));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        } else {
                            out += static_cast<char>(0xE0 | (cp >> 12));
                            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: bad("bad escape");
                }
            } else {
                out += c;
            }
        }
        if (i >= s.size()) bad("unterminated string");
        ++i;
        return out;
    }
    Json value() {
        ws();
        if (i >= s.size()) bad("unexpected end");
        Json v;
        const char c = s[i];
        if (c == '{') {
            ++i;
            v.kind = Json::Object;
            ws();
            if (s[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                std::string key = parse_string();
                ws();
                if (s[i] != ':') bad("expected ':'");
                ++i;
                v.obj.emplace_back(std::move(key), value());
                ws();
                if (s[i] == ',') {
                    ++i;
                    continue;
                }
                if (s[i] == '}') {
                    ++i;
                    return v;
                }
                bad("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++i;
            v.kind = Json::Array;
            ws();
            if (s[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (s[i] == ',') {
                    ++i;
                    continue;
                }
                if (s[i] == ']') {
                    ++i;
                    return v;
                }
                bad("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Json::String;
            v.str = parse_string();
            return v;
        }
        if (lit("true")) {
            v.kind = Json::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = Json::Bool;
            return v;
        }
        if (lit("null")) return v;
        const char* p = s.c_str() + i;
        char* end = nullptr;
        v.num = std::strtod(p, &end);
        if (end == p) bad("unexpected character");
        i += static_cast<size_t>(end - p);
        v.kind = Json::Number;
        return v;
    }
};

// ordered-json text in nlohmann's compact dump style
struct Writer {
    std::string out;
    std::vector<bool> first{true};
    void sep() {
        if (!first.back()) out += ',';
        first.back() = false;
    }
    void key(const char* k) {
        sep();
        out += '"';
        out += k;
        out += "\":";
        first.back() = true;  // the value that follows needs no separator
    }
    void begin(char c) {
        if (!first.back()) out += ',';
        first.back() = false;
        out += c;
        first.push_back(true);
    }
    void end(char c) {
        out += c;
        first.pop_back();
    }
    // nlohmann::json's dump of a double (dtoa_impl::to_chars / format_buffer):
    // the shortest round-trip digits d1..dk with the value d * 10^(n-k), written
    // as "digits[000].0" for k <= n <= 15, "dig.its" for 0 < n <= 15,
    // "0.[000]digits" for -4 < n <= 0, else "d.igitse+XX"; non-finite -> null
    void num(double v) {
        sep();
        if (!std::isfinite(v)) {
            out += "null";
            return;
        }
        if (v == 0.0) {
            out += std::signbit(v) ? "-0.0" : "0.0";
            return;
        }
        char buf[48];
        for (int prec = 0; prec <= 17; ++prec) {
            std::snprintf(buf, sizeof buf, "%.*e", prec, v);
            if (std::strtod(buf, nullptr) == v) break;
        }
        std::string t(buf);
        if (t[0] == '-') {
            out += '-';
            t.erase(0, 1);
        }
        const size_t epos = t.find('e');
        const int e10 = std::atoi(t.c_str() + epos + 1);
        std::string dg;
        for (size_t i = 0; i < epos; ++i)
            if (t[i] != '.') dg += t[i];
        while (dg.size() > 1 && dg.back() == '0') dg.pop_back();
        const int k = static_cast<int>(dg.size()), n = e10 + 1;
        if (k <= n && n <= 15) {
            out += dg + std::string(static_cast<size_t>(n - k), '0') + ".0";
        } else if (0 < n && n <= 15) {
            out += dg.substr(0, static_cast<size_t>(n)) + "." + dg.substr(static_cast<size_t>(n));
        } else if (-4 < n && n <= 0) {
            out += "0." + std::string(static_cast<size_t>(-n), '0') + dg;
        } else {
            out += dg.substr(0, 1);
            if (k > 1) out += "." + dg.substr(1);
            const int x = n - 1;
            char eb[16];
            std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
            out += eb;
        }
    }
    void integer(long long v) {
        sep();
        out += std::to_string(v);
    }
    void boolean(bool v) {
        sep();
        out += v ? "true" : "false";
    }
    void str(const std::string& v) {
        sep();
        out += '"';
        out += v;
        out += '"';
    }
};

const char* kModality[3] = {"rssi", "csi", "spectrum"};  // sim::modality_name, channelsim.cpp:144-151
const char* kMode[5] = {"full", "global_only", "local_only", "additive_only", "no_occlusion"};  // conditioning.cpp:180-189

struct Named {
    std::string name;
    std::vector<size_t> shape;
    const double* data;
};

size_t count(const std::vector<size_t>& shape) {
    size_t n = 1;
    for (size_t s : shape) n *= s;
    return n;
}

}  // namespace
}  // namespace rxgs_b200

using namespace rxgs_b200;

extern "C" {

int rxgs_checkpoint_save(const char* path, rxgs_scene sc, const rxgs_grid* grid, rxgs_cond c) {
    try {
        if (!path || !sc || !grid) return fail(RXGS_ERR_INVALID, "save_checkpoint: null argument");
        if (int rc = scene_sync_host(sc)) return rc;  // device arrays updated by the optimizer
        if (c && c->host_stale) {
            cudaSetDevice(c->ctx->device);
            RXGS_CUDA(cudaStreamSynchronize(c->ctx->stream));
            RXGS_CUDA(cudaMemcpy(c->h_params.data(), c->d_params64.p, c->h_params.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost));
            c->host_stale = false;
        }
        const size_t K = static_cast<size_t>(sc->k);
        // manifest_for (checkpoint.cpp:31-89)
        std::vector<Named> arrays = {
            {"positions", {K, 3}, sc->h_pos.data()},
            {"log_scales", {K, 3}, sc->h_ls.data()},
            {"quaternions", {K, 4}, sc->h_q.data()},
            {"tau_logits", {K}, sc->h_tau.data()},
            {"fle_coeffs", {K, static_cast<size_t>(sc->L), static_cast<size_t>(sc->channels), 2}, sc->h_coeffs.data()},
        };
        std::vector<double> occ;
        if (c) {
            const size_t d = c->hidden, F = c->F, L = c->L, dc = c->dc, C4 = 4 * static_cast<size_t>(c->C);
            const double* p = c->h_params.data();
            auto mlp = [&](const std::string& pre, size_t o1, size_t in) {
                arrays.push_back({pre + ".w1", {d, in}, p + o1});
                arrays.push_back({pre + ".b1", {d}, p + o1 + d * in});
                arrays.push_back({pre + ".w2", {d, d}, p + o1 + d * in + d});
                arrays.push_back({pre + ".b2", {d}, p + o1 + d * in + d + d * d});
                arrays.push_back({pre + ".w3", {C4, d}, p + o1 + d * in + 2 * d + d * d});
                arrays.push_back({pre + ".b3", {C4}, p + o1 + d * in + 2 * d + d * d + C4 * d});
            };
            arrays.push_back({"cond.fourier_freqs", {F, 3}, p + c->o_freq});
            mlp("cond.global", c->o_gw1, static_cast<size_t>(c->gin));
            arrays.push_back({"cond.component_embed", {L, dc}, p + c->o_emb});
            mlp("cond.local", c->o_lw1, 6);
            const size_t R = static_cast<size_t>(c->R);
            occ.assign(R * R * R, 0.0);
            if (c->has_occ && c->h_occ.size() == occ.size()) occ = c->h_occ;
            arrays.push_back({"cond.occupancy", {R, R, R}, occ.data()});
        }
        Writer w;
        w.begin('{');
        w.key("k");
        w.integer(sc->k);
        w.key("l_max");
        w.integer(sc->l_max);
        w.key("channels");
        w.integer(sc->channels);
        w.key("modality");
        w.str(kModality[sc->modality]);
        w.key("grid");
        w.begin('{');
        w.key("n_theta");
        w.integer(grid->n_theta);
        w.key("n_phi");
        w.integer(grid->n_phi);
        w.key("tile_size");
        w.integer(grid->tile_size);
        w.key("radius");
        w.num(grid->radius);
        w.key("theta_min");
        w.num(grid->theta_min);
        w.key("theta_max");
        w.num(grid->theta_max);
        w.end('}');
        w.key("has_conditioning");
        w.boolean(c != nullptr);
        if (c) {
            w.key("conditioning");
            w.begin('{');
            w.key("fourier_bands");
            w.integer(c->F);
            w.key("hidden");
            w.integer(c->hidden);
            w.key("embed_dim");
            w.integer(c->dc);
            w.key("probe_samples");
            w.integer(c->S);
            w.key("occupancy_resolution");
            w.integer(c->R);
            w.key("nearest_lookup");
            w.boolean(c->nearest != 0);
            w.key("mode");
            w.str(kMode[c->mode]);
            w.key("occupancy_bounds");
            w.begin('[');
            for (int a = 0; a < 3; ++a) w.num(c->lo[a]);
            for (int a = 0; a < 3; ++a) w.num(c->hi[a]);
            w.end(']');
            w.end('}');
        }
        w.key("arrays");
        w.begin('[');
        size_t offset = 0;
        for (const Named& a : arrays) {
            w.begin('{');
            w.key("name");
            w.str(a.name);
            w.key("dtype");
            w.str("f64");
            w.key("shape");
            w.begin('[');
            for (size_t s : a.shape) w.integer(static_cast<long long>(s));
            w.end(']');
            w.key("offset");
            w.integer(static_cast<long long>(offset));
            w.end('}');
            offset += count(a.shape) * sizeof(double);
        }
        w.end(']');
        w.end('}');
        std::ofstream out(path, std::ios::binary);
        if (!out) throw IoError(std::string("save_checkpoint: cannot open ") + path);
        out.write("RXGS", 4);
        const uint32_t version = 1;  // kCheckpointVersion, checkpoint.hpp:14
        out.write(reinterpret_cast<const char*>(&version), 4);
        const uint64_t header_len = w.out.size();
        out.write(reinterpret_cast<const char*>(&header_len), 8);
        out.write(w.out.data(), static_cast<std::streamsize>(w.out.size()));
        for (const Named& a : arrays)
            out.write(reinterpret_cast<const char*>(a.data), static_cast<std::streamsize>(count(a.shape) * sizeof(double)));
        if (!out) throw IoError(std::string("save_checkpoint: write failed for ") + path);
        return RXGS_OK;
    } catch (const IoError& e) {
        return fail(RXGS_ERR_IO, e.what());
    } catch (const std::exception& e) {
        return fail(RXGS_ERR_RUNTIME, e.what());
    }
}

int rxgs_checkpoint_load(rxgs_ctx ctx, const char* path, rxgs_scene* out_scene, rxgs_grid* out_grid,
                         rxgs_cond* out_cond) {
    if (out_scene) *out_scene = nullptr;
    if (out_cond) *out_cond = nullptr;
    try {
        if (!ctx || !path || !out_scene) return fail(RXGS_ERR_INVALID, "load_checkpoint: null argument");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw IoError(std::string("load_checkpoint: cannot open ") + path);
        char magic[4];
        in.read(magic, 4);
        if (!in || std::string(magic, 4) != "RXGS") throw IoError(std::string("load_checkpoint: bad magic in ") + path);
        uint32_t version = 0;
        in.read(reinterpret_cast<char*>(&version), 4);
        if (version != 1) throw IoError("load_checkpoint: unsupported version " + std::to_string(version));
        uint64_t header_len = 0;
        in.read(reinterpret_cast<char*>(&header_len), 8);
        if (!in || header_len > (uint64_t{1} << 32)) throw IoError(std::string("load_checkpoint: truncated header in ") + path);
        std::string header_str(header_len, '\0');
        in.read(header_str.data(), static_cast<std::streamsize>(header_len));
        if (!in) throw IoError(std::string("load_checkpoint: truncated header in ") + path);
        Parser ps(header_str);
        const Json header = ps.value();

        const int l_max = header.at("l_max").integer();
        const int channels = header.at("channels").integer();
        const std::string mod = header.at("modality").string();
        int modality = -1;
        for (int m = 0; m < 3; ++m)
            if (mod == kModality[m]) modality = m;
        if (modality < 0) throw std::invalid_argument("unknown modality '" + mod + "'");  // modality_from_name
        const Json& g = header.at("grid");
        rxgs_grid grid{};
        grid.n_theta = g.at("n_theta").integer();
        grid.n_phi = g.at("n_phi").integer();
        grid.tile_size = g.at("tile_size").integer();
        grid.radius = g.at("radius").number();
        grid.theta_min = g.at("theta_min").number();
        grid.theta_max = g.at("theta_max").number();
        const bool has_cond = header.at("has_conditioning").boolean();
        int32_t cfg[9] = {6, 64, 16, 16, 32, 0, 0, l_max, channels};
        double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        std::vector<double> params;
        size_t o_freq = 0, o_gw1 = 0, o_emb = 0, o_lw1 = 0, gin = 0, L = static_cast<size_t>((l_max + 1) * (l_max + 1));
        if (has_cond) {
            const Json& cj = header.at("conditioning");
            cfg[0] = cj.at("fourier_bands").integer();
            cfg[1] = cj.at("hidden").integer();
            cfg[2] = cj.at("embed_dim").integer();
            cfg[3] = cj.at("probe_samples").integer();
            cfg[4] = cj.at("occupancy_resolution").integer();
            cfg[5] = cj.at("nearest_lookup").boolean() ? 1 : 0;
            const std::string mode = cj.at("mode").string();
            cfg[6] = -1;
            for (int m = 0; m < 5; ++m)
                if (mode == kMode[m]) cfg[6] = m;
            if (cfg[6] < 0) throw std::invalid_argument("unknown conditioning mode '" + mode + "'");
            const Json& b = cj.at("occupancy_bounds");
            if (b.kind != Json::Array || b.arr.size() != 6) throw IoError("load_checkpoint: bad occupancy_bounds");
            for (int a = 0; a < 3; ++a) {
                lo[a] = b.arr[a].number();
                hi[a] = b.arr[3 + a].number();
            }
            // init_conditioning(cfg, l_max, channels, bounds, seed 0), then the file's arrays over it
            // (checkpoint.cpp:191-193)
            const int64_t n = rxgs_synth_cond(cfg, l_max, channels, lo, hi, 0, 0, nullptr);
            params.assign(static_cast<size_t>(n), 0.0);
            rxgs_synth_cond(cfg, l_max, channels, lo, hi, 0, 0, params.data());
            const size_t d = cfg[1];
            gin = 6 * static_cast<size_t>(cfg[0]) + 2 + cfg[2];
            o_freq = 0;
            o_gw1 = 3 * static_cast<size_t>(cfg[0]);
            o_emb = o_gw1 + d * gin + d + d * d + d + 4 * channels * d + 4 * channels;
            o_lw1 = o_emb + L * cfg[2];
        }
        // Named arrays at their manifest offsets (checkpoint.cpp:197-229).
        const std::streampos data_start = in.tellg();
        std::vector<double> pos, ls, q, tau, coeffs, occ;
        auto read_array = [&](const Json& entry, std::vector<double>& dst) {
            std::vector<size_t> shape;
            for (const Json& s : entry.at("shape").arr) shape.push_back(static_cast<size_t>(s.number()));
            dst.resize(count(shape));
            in.seekg(data_start + static_cast<std::streamoff>(entry.at("offset").number()));
            in.read(reinterpret_cast<char*>(dst.data()), static_cast<std::streamsize>(dst.size() * sizeof(double)));
            if (!in) throw IoError("load_checkpoint: truncated array '" + entry.at("name").string() + "'");
        };
        auto into_params = [&](const Json& entry, size_t off, size_t n) {
            std::vector<double> tmp;
            read_array(entry, tmp);
            if (!has_cond || off + tmp.size() > params.size() || tmp.size() != n)
                throw std::invalid_argument("conditioning: array '" + entry.at("name").string() + "' has the wrong size");
            std::copy(tmp.begin(), tmp.end(), params.begin() + static_cast<std::ptrdiff_t>(off));
        };
        const size_t d = cfg[1], C4 = 4 * static_cast<size_t>(channels);
        auto mlp_off = [&](size_t o1, size_t in_dim, const std::string& t, size_t& n) -> size_t {
            const size_t b1 = o1 + d * in_dim, w2 = b1 + d, b2 = w2 + d * d, w3 = b2 + d, b3 = w3 + C4 * d;
            if (t == "w1") { n = d * in_dim; return o1; }
            if (t == "b1") { n = d; return b1; }
            if (t == "w2") { n = d * d; return w2; }
            if (t == "b2") { n = d; return b2; }
            if (t == "w3") { n = C4 * d; return w3; }
            n = C4;
            return b3;  // "b3"
        };
        for (const Json& entry : header.at("arrays").arr) {
            const std::string name = entry.at("name").string();
            if (entry.at("dtype").string() != "f64")
                throw IoError("load_checkpoint: unsupported dtype for '" + name + "'");
            size_t n = 0;
            if (name == "positions") read_array(entry, pos);
            else if (name == "log_scales") read_array(entry, ls);
            else if (name == "quaternions") read_array(entry, q);
            else if (name == "tau_logits") read_array(entry, tau);
            else if (name == "fle_coeffs") read_array(entry, coeffs);
            else if (name == "cond.fourier_freqs") into_params(entry, o_freq, 3 * static_cast<size_t>(cfg[0]));
            else if (name == "cond.component_embed") into_params(entry, o_emb, L * cfg[2]);
            else if (name == "cond.occupancy") read_array(entry, occ);
            else if (name.rfind("cond.global.", 0) == 0 && name.size() == 14 && (name[12] == 'w' || name[12] == 'b') &&
                     name[13] >= '1' && name[13] <= '3') {
                const size_t off = mlp_off(o_gw1, gin, name.substr(12), n);
                into_params(entry, off, n);
            } else if (name.rfind("cond.local.", 0) == 0 && name.size() == 13 && (name[11] == 'w' || name[11] == 'b') &&
                       name[12] >= '1' && name[12] <= '3') {
                const size_t off = mlp_off(o_lw1, 6, name.substr(11), n);
                into_params(entry, off, n);
            } else {
                throw IoError("load_checkpoint: unknown array '" + name + "'");
            }
        }
        // GaussianScene::validate (scene.cpp:33-40)
        const size_t K = tau.size();
        if (pos.size() != 3 * K || ls.size() != 3 * K || q.size() != 4 * K || coeffs.size() != K * L * channels * 2)
            throw std::invalid_argument("scene: per-Gaussian arrays out of alignment");
        for (double v : pos)
            if (!std::isfinite(v)) throw std::invalid_argument("scene: non-finite position");
        rxgs_scene sc = nullptr;
        int rc = rxgs_scene_create(ctx, static_cast<int>(K), l_max, channels, modality, pos.data(), ls.data(), q.data(),
                                   tau.data(), coeffs.data(), &sc);
        if (rc) return rc;
        if (has_cond && out_cond) {
            const size_t R = static_cast<size_t>(cfg[4]);
            const bool occ_ok = occ.size() == R * R * R && R > 0;
            rxgs_cond c = nullptr;
            rc = rxgs_cond_create(ctx, cfg, params.data(), occ_ok ? occ.data() : nullptr, lo, hi, &c);
            if (rc) {
                rxgs_scene_destroy(sc);
                return rc;
            }
            if (!occ_ok) {  // an empty grid still carries its bounds (OccupancyGrid, conditioning.hpp:28-38)
                for (int a = 0; a < 3; ++a) {
                    c->lo[a] = lo[a];
                    c->hi[a] = hi[a];
                }
            }
            *out_cond = c;
        }
        if (out_grid) *out_grid = grid;
        *out_scene = sc;
        return RXGS_OK;
    } catch (const IoError& e) {
        return fail(RXGS_ERR_IO, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(RXGS_ERR_INVALID, e.what());
    } catch (const std::exception& e) {
        return fail(RXGS_ERR_RUNTIME, e.what());
    }
}

int rxgs_scene_info(rxgs_scene sc, int32_t* k, int32_t* l_max, int32_t* channels, int32_t* modality) {
    if (!sc) return fail(RXGS_ERR_INVALID, "null scene");
    if (k) *k = sc->k;
    if (l_max) *l_max = sc->l_max;
    if (channels) *channels = sc->channels;
    if (modality) *modality = sc->modality;
    return RXGS_OK;
}

int rxgs_scene_get_arrays(rxgs_scene sc, double* pos, double* ls, double* q, double* tau, double* coeffs) {
    if (!sc) return fail(RXGS_ERR_INVALID, "null scene");
    auto cp = [](double* dst, const std::vector<double>& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    if (int rc = scene_sync_host(sc)) return rc;
    cp(pos, sc->h_pos);
    cp(ls, sc->h_ls);
    cp(q, sc->h_q);
    cp(tau, sc->h_tau);
    if (coeffs) return rxgs_scene_get_coeffs(sc, coeffs);
    return RXGS_OK;
}

int rxgs_cond_get_occupancy(rxgs_cond c, int32_t* has, double* densities, double lo[3], double hi[3]) {
    if (!c) return fail(RXGS_ERR_INVALID, "null conditioning");
    const bool h = c->has_occ && !c->h_occ.empty();
    if (has) *has = h ? 1 : 0;
    if (densities && h) std::memcpy(densities, c->h_occ.data(), c->h_occ.size() * sizeof(double));
    for (int a = 0; a < 3; ++a) {
        if (lo) lo[a] = c->lo[a];
        if (hi) hi[a] = c->hi[a];
    }
    return RXGS_OK;
}

int rxgs_cond_config(rxgs_cond c, int32_t cfg[9]) {
    if (!c || !cfg) return fail(RXGS_ERR_INVALID, "null conditioning");
    const int32_t v[9] = {c->F, c->hidden, c->dc, c->S, c->R, c->nearest, c->mode, c->l_max, c->C};
    for (int i = 0; i < 9; ++i) cfg[i] = v[i];
    return RXGS_OK;
}

}  // extern "C"
