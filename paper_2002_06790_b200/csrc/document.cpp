// Graph-document loader: parse_graph (graph.py:192-293) + host_csr + node_rows in C++ for
// documents too large for Python (a 1M-node document spends tens of
// seconds in json.loads and object construction before any kernel runs).
//
// The loader accepts the well-formed subset of the unified graph format and produces the
// rank-ordered arrays the device path needs (ids, CSR, devices, per-node op / kind / feature
// signature / communication attributes).  Anything the reference would warn about or reject
// (unknown fields, duplicate ids, dangling references, bad shapes, non-finite numbers,
// attribute/feature-name collisions, lone surrogates, ...) is reported as "unsupported" and
// the Python layer re-parses with parse_graph, so errors and warnings stay the reference's.
// Host code only.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "dfsim_b200.h"

namespace {

struct Unsupported {
    std::string why;
};

[[noreturn]] void unsupported(const std::string &why) { throw Unsupported{why}; }

// ------------------------------------------------------------------ JSON DOM
enum : uint8_t { J_NULL, J_TRUE, J_FALSE, J_INT, J_FLOAT, J_STR, J_ARR, J_OBJ };

struct Val {
    uint8_t t = J_NULL;
    uint8_t in_text = 0;    // J_STR without escapes: [a, a+n) of the document itself (no copy)
    uint32_t a = 0, n = 0;  // J_STR: string pool / text [a, a+n); J_ARR/J_OBJ: kids [a, a+n)
    uint32_t lo = 0, hi = 0;  // byte range in the text (documents < 4 GB)
    int64_t i = 0;          // J_INT (fits int64)
    double d = 0.0;         // J_INT / J_FLOAT numeric value (float(int) for ints)
};

struct Parser {
    const char *s;
    int64_t len, p = 0;
    std::vector<Val> vals;
    std::vector<uint32_t> kids;   // array items / object (key, value) pairs as val indices
    std::string pool;             // unescaped strings
    std::vector<uint32_t> stack;  // children of the containers being parsed

    char peek() { return p < len ? s[p] : '\0'; }
    void ws() {
        while (p < len && (s[p] == ' ' || s[p] == '\n' || s[p] == '\r' || s[p] == '\t')) p++;
    }
    void expect(char c) {
        ws();
        if (peek() != c) unsupported("JSON syntax");
        p++;
    }
    static void put_utf8(std::string &o, unsigned cp) {
        if (cp < 0x80) {
            o += static_cast<char>(cp);
        } else if (cp < 0x800) {
            o += static_cast<char>(0xC0 | (cp >> 6));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += static_cast<char>(0xE0 | (cp >> 12));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            o += static_cast<char>(0xF0 | (cp >> 18));
            o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (p + 4 > len) unsupported("JSON syntax");
        unsigned v = 0;
        for (int k = 0; k < 4; k++) {
            const char c = s[p++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= c - '0';
            else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
            else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
            else unsupported("JSON syntax");
        }
        return v;
    }
    void string_into(Val &v) {
        p++;  // opening quote
        v.t = J_STR;
        {  // fast path: no escape before the closing quote -> a view of the document
            int64_t q = p;
            while (q < len && s[q] != '"' && s[q] != '\\' && static_cast<unsigned char>(s[q]) >= 0x20) q++;
            if (q < len && s[q] == '"') {
                v.in_text = 1;
                v.a = static_cast<uint32_t>(p);
                v.n = static_cast<uint32_t>(q - p);
                p = q + 1;
                return;
            }
        }
        v.a = static_cast<uint32_t>(pool.size());
        while (true) {
            if (p >= len) unsupported("JSON syntax");
            const unsigned char c = static_cast<unsigned char>(s[p]);
            if (c == '"') { p++; break; }
            if (c < 0x20) unsupported("control character in string");
            if (c != '\\') {
                int64_t q = p;
                while (q < len && s[q] != '"' && s[q] != '\\' && static_cast<unsigned char>(s[q]) >= 0x20) q++;
                pool.append(s + p, static_cast<size_t>(q - p));
                p = q;
                continue;
            }
            p++;
            const char e = p < len ? s[p++] : '\0';
            switch (e) {
                case '"': pool += '"'; break;
                case '\\': pool += '\\'; break;
                case '/': pool += '/'; break;
                case 'b': pool += '\b'; break;
                case 'f': pool += '\f'; break;
                case 'n': pool += '\n'; break;
                case 'r': pool += '\r'; break;
                case 't': pool += '\t'; break;
                case 'u': {
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00) {  // a surrogate pair, or unsupported
                        if (p + 6 <= len && s[p] == '\\' && s[p + 1] == 'u') {
                            p += 2;
                            const unsigned lo = hex4();
                            if (lo < 0xDC00 || lo >= 0xE000) unsupported("lone surrogate");
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else {
                            unsupported("lone surrogate");
                        }
                    } else if (cp >= 0xDC00 && cp < 0xE000) {
                        unsupported("lone surrogate");
                    }
                    put_utf8(pool, cp);
                    break;
                }
                default: unsupported("JSON syntax");
            }
        }
        v.n = static_cast<uint32_t>(pool.size() - v.a);
    }
    void number_into(Val &v) {
        const int64_t q0 = p;
        bool is_int = true;
        if (peek() == '-') p++;
        if (!(peek() >= '0' && peek() <= '9')) unsupported("JSON syntax");
        if (peek() == '0') {
            p++;
        } else {
            while (peek() >= '0' && peek() <= '9') p++;
        }
        if (peek() == '.') {
            is_int = false;
            p++;
            if (!(peek() >= '0' && peek() <= '9')) unsupported("JSON syntax");
            while (peek() >= '0' && peek() <= '9') p++;
        }
        if (peek() == 'e' || peek() == 'E') {
            is_int = false;
            p++;
            if (peek() == '+' || peek() == '-') p++;
            if (!(peek() >= '0' && peek() <= '9')) unsupported("JSON syntax");
            while (peek() >= '0' && peek() <= '9') p++;
        }
        const int64_t n = p - q0;
        if (is_int && n <= 18) {  // exact in int64; float(int) is exact below 2^53, else strtod
            int64_t iv = 0;
            for (int64_t k = (s[q0] == '-'); k < n; k++) iv = iv * 10 + (s[q0 + k] - '0');
            if (s[q0] == '-') iv = -iv;
            v.t = J_INT;
            v.i = iv;
            if (iv > -(int64_t(1) << 53) && iv < (int64_t(1) << 53)) {
                v.d = static_cast<double>(iv);
                return;
            }
        }
        char buf[400];
        if (n >= static_cast<int64_t>(sizeof buf)) unsupported("number too long");
        std::memcpy(buf, s + q0, static_cast<size_t>(n));
        buf[n] = '\0';
        const double d = std::strtod(buf, nullptr);  // correctly rounded, like float(str) / float(int)
        if (!std::isfinite(d)) unsupported("non-finite number");
        v.d = d;
        if (is_int) {
            if (n > 18) {
                errno = 0;
                const long long iv = std::strtoll(buf, nullptr, 10);
                if (errno == ERANGE) unsupported("integer beyond int64");
                v.i = iv;
            }
            v.t = J_INT;
        } else {
            v.t = J_FLOAT;
        }
    }
    uint32_t value(int depth) {
        if (depth > 64) unsupported("nesting too deep");
        ws();
        const uint32_t idx = static_cast<uint32_t>(vals.size());
        vals.emplace_back();
        Val v;
        v.lo = static_cast<uint32_t>(p);
        const char c = peek();
        if (c == '{') {
            p++;
            const size_t base = stack.size();
            ws();
            if (peek() == '}') {
                p++;
            } else {
                while (true) {
                    ws();
                    if (peek() != '"') unsupported("JSON syntax");
                    const uint32_t k = static_cast<uint32_t>(vals.size());
                    vals.emplace_back();
                    Val kv;
                    kv.lo = static_cast<uint32_t>(p);
                    string_into(kv);
                    kv.hi = static_cast<uint32_t>(p);
                    vals[k] = kv;
                    expect(':');
                    const uint32_t val = value(depth + 1);
                    stack.push_back(k);
                    stack.push_back(val);
                    ws();
                    if (peek() == ',') { p++; continue; }
                    if (peek() == '}') { p++; break; }
                    unsupported("JSON syntax");
                }
            }
            v.t = J_OBJ;
            v.a = static_cast<uint32_t>(kids.size());
            v.n = static_cast<uint32_t>((stack.size() - base) / 2);
            kids.insert(kids.end(), stack.begin() + base, stack.end());
            stack.resize(base);
        } else if (c == '[') {
            p++;
            const size_t base = stack.size();
            ws();
            if (peek() == ']') {
                p++;
            } else {
                while (true) {
                    stack.push_back(value(depth + 1));
                    ws();
                    if (peek() == ',') { p++; continue; }
                    if (peek() == ']') { p++; break; }
                    unsupported("JSON syntax");
                }
            }
            v.t = J_ARR;
            v.a = static_cast<uint32_t>(kids.size());
            v.n = static_cast<uint32_t>(stack.size() - base);
            kids.insert(kids.end(), stack.begin() + base, stack.end());
            stack.resize(base);
        } else if (c == '"') {
            string_into(v);
        } else if (c == 't' && p + 4 <= len && !std::memcmp(s + p, "true", 4)) {
            p += 4;
            v.t = J_TRUE;
        } else if (c == 'f' && p + 5 <= len && !std::memcmp(s + p, "false", 5)) {
            p += 5;
            v.t = J_FALSE;
        } else if (c == 'n' && p + 4 <= len && !std::memcmp(s + p, "null", 4)) {
            p += 4;
            v.t = J_NULL;
        } else {
            number_into(v);  // NaN / Infinity literals land here and are unsupported
        }
        v.hi = static_cast<uint32_t>(p);
        vals[idx] = v;
        return idx;
    }
};

// ------------------------------------------------------------------ document semantics
struct Doc {
    // nodes in rank order
    std::vector<std::string_view> ids;
    std::string id_blob, op_blob, dev_blob, fname_blob, dec_blob;
    std::vector<int64_t> id_off, op_off, dev_off, fname_off, dec_off;
    std::vector<int32_t> op_of, dev_of, indeg, succ_off, succ_idx, sources, queue_off, sig_of, fname;
    std::vector<uint8_t> kind_of, comm_ok;
    std::vector<int64_t> comm_bytes, node_lo, node_hi, sig_off;
    std::vector<int32_t> group_size;
    std::vector<double> link_thr, link_lat, fval;
    std::vector<uint8_t> dec_kind;
    std::vector<double> dec_thr, dec_lat;
    std::vector<uint8_t> dec_has_thr;
    int64_t meta_lo = -1, meta_hi = -1, decl_lo = -1, decl_hi = -1;
    int32_t max_indeg = 0;
    std::string why;
    dfsim_document view{};
};

std::string_view sv(const Parser &P, const Val &v) {
    return v.in_text ? std::string_view(P.s + v.a, v.n) : std::string_view(P.pool).substr(v.a, v.n);
}

// object field lookup; duplicate keys are unsupported (json.loads keeps the last one)
struct Fields {  // at most 8 known fields: no heap allocation per object
    std::pair<std::string_view, uint32_t> f[8];
    int n = 0;
    const Val *get(const Parser &P, std::string_view k) const {
        for (int i = 0; i < n; i++)
            if (f[i].first == k) return &P.vals[f[i].second];
        return nullptr;
    }
};

Fields fields_of(const Parser &P, const Val &obj, std::initializer_list<std::string_view> known) {
    Fields out;
    if (obj.n > 8) unsupported("unknown field (the reference warns)");
    for (uint32_t i = 0; i < obj.n; i++) {
        const Val &k = P.vals[P.kids[obj.a + 2 * i]];
        const std::string_view name = sv(P, k);
        bool ok = false;
        for (auto kn : known) ok |= kn == name;
        if (!ok) unsupported("unknown field (the reference warns)");
        for (int j = 0; j < out.n; j++)
            if (out.f[j].first == name) unsupported("duplicate key");
        out.f[out.n++] = {name, P.kids[obj.a + 2 * i + 1]};
    }
    return out;
}

const char *kKinds[3] = {"Compute", "Transfer", "Collective"};

uint64_t hash_bytes(const char *p, size_t n, uint64_t h = 1469598103934665603ull) {  // FNV-1a
    for (size_t i = 0; i < n; i++) h = (h ^ static_cast<unsigned char>(p[i])) * 1099511628211ull;
    return h;
}

// string_view -> index, open addressing (no per-entry allocation; the id lookups of a 10^6-node
// document are the loader's hottest operation)
struct IdTable {
    std::vector<int32_t> slot;  // -1 empty, else index into keys
    const std::vector<std::string_view> *keys = nullptr;
    uint64_t mask = 0;
    void build(const std::vector<std::string_view> &k, const std::vector<uint32_t> &order) {
        keys = &k;
        size_t cap = 16;
        while (cap < order.size() * 2) cap <<= 1;
        slot.assign(cap, -1);
        mask = cap - 1;
        for (size_t r = 0; r < order.size(); r++) {
            const std::string_view key = k[order[r]];
            uint64_t h = hash_bytes(key.data(), key.size()) & mask;
            while (slot[h] >= 0) {
                if ((*keys)[order[slot[h]]] == key) unsupported("duplicate node id");
                h = (h + 1) & mask;
            }
            slot[h] = static_cast<int32_t>(r);
        }
        order_ = &order;
    }
    int32_t find(std::string_view key) const {
        uint64_t h = hash_bytes(key.data(), key.size()) & mask;
        while (slot[h] >= 0) {
            if ((*keys)[(*order_)[slot[h]]] == key) return slot[h];
            h = (h + 1) & mask;
        }
        return -1;
    }
    const std::vector<uint32_t> *order_ = nullptr;
};

void build(Doc &D, Parser &P, uint32_t root) {
    const Val &top = P.vals[root];
    if (top.t != J_OBJ) unsupported("document is not an object");
    const Fields tf = fields_of(P, top, {"format_version", "metadata", "devices", "nodes"});
    const Val *fv = tf.get(P, "format_version");
    if (!fv) unsupported("missing format_version");
    if (fv->t == J_INT) {
        if (fv->i != 1) unsupported("format version");
    } else if (fv->t == J_STR) {
        const std::string_view s = sv(P, *fv);
        if (!(s == "1" || (s.size() > 1 && s[0] == '1' && s[1] == '.'))) unsupported("format version");
    } else {
        unsupported("format version type");
    }
    if (const Val *m = tf.get(P, "metadata")) {
        if (m->t != J_OBJ) unsupported("metadata is not an object");
        D.meta_lo = m->lo;
        D.meta_hi = m->hi;
    }
    // declared devices (doc order)
    std::unordered_map<std::string_view, int32_t> dec_index;
    std::vector<std::string_view> dec_ids;
    if (const Val *dv = tf.get(P, "devices")) {
        if (dv->t != J_ARR) unsupported("devices is not a list");
        D.decl_lo = dv->lo;
        D.decl_hi = dv->hi;
        for (uint32_t i = 0; i < dv->n; i++) {
            const Val &d = P.vals[P.kids[dv->a + i]];
            if (d.t != J_OBJ) unsupported("device entry");
            const Fields f = fields_of(P, d, {"id", "kind", "hardware", "throughput_mbps", "latency_us"});
            const Val *id = f.get(P, "id"), *kind = f.get(P, "kind");
            if (!id || !kind || id->t != J_STR || kind->t != J_STR) unsupported("device id/kind");
            const Val *hw = f.get(P, "hardware"), *thr = f.get(P, "throughput_mbps"), *lat = f.get(P, "latency_us");
            if (hw && hw->t != J_STR) unsupported("device hardware");
            const std::string_view k = sv(P, *kind);
            const int kc = k == "Compute" ? 0 : (k == "Link" ? 1 : (k == "CollectiveResource" ? 2 : -1));
            if (kc < 0) unsupported("device kind");
            const bool has_thr = thr && thr->t != J_NULL;
            if (has_thr && !(thr->t == J_INT || thr->t == J_FLOAT)) unsupported("device throughput");
            if (lat && !(lat->t == J_INT || lat->t == J_FLOAT)) unsupported("device latency");
            const double latv = lat ? lat->d : 0.0;
            if (kc == 0 ? has_thr : (!has_thr || thr->d <= 0 || latv < 0)) unsupported("device spec");
            const std::string_view ids = sv(P, *id);
            if (dec_index.count(ids)) unsupported("duplicate device id");
            dec_index.emplace(ids, static_cast<int32_t>(dec_ids.size()));
            dec_ids.push_back(ids);
            D.dec_off.push_back(static_cast<int64_t>(D.dec_blob.size()));
            D.dec_blob.append(ids.data(), ids.size());
            D.dec_blob += '\0';
            D.dec_kind.push_back(static_cast<uint8_t>(kc));
            D.dec_has_thr.push_back(has_thr ? 1 : 0);
            D.dec_thr.push_back(has_thr ? thr->d : 0.0);
            D.dec_lat.push_back(latv);
            (void)hw;
        }
    }
    D.dec_off.push_back(static_cast<int64_t>(D.dec_blob.size()));
    // nodes
    const Val *nv = tf.get(P, "nodes");
    if (nv && nv->t != J_ARR) unsupported("nodes is not a list");
    const uint32_t N = nv ? nv->n : 0;
    struct NodeRef {
        std::string_view id, op, dev;
        int kind;
        const Val *obj, *attrs, *inputs, *shapes;
    };
    std::vector<NodeRef> raw(N);
    std::vector<std::string_view> raw_ids(N);
    for (uint32_t i = 0; i < N; i++) {
        const Val &o = P.vals[P.kids[nv->a + i]];
        if (o.t != J_OBJ) unsupported("node entry");
        const Fields f = fields_of(P, o, {"id", "op", "kind", "device", "attrs", "inputs", "output_shapes"});
        const Val *id = f.get(P, "id"), *op = f.get(P, "op"), *kind = f.get(P, "kind"), *dev = f.get(P, "device");
        if (!id || !op || !kind || !dev || id->t != J_STR || op->t != J_STR || kind->t != J_STR || dev->t != J_STR)
            unsupported("node id/op/kind/device");
        const std::string_view ids = sv(P, *id), ks = sv(P, *kind);
        if (ids.empty() || ids.find(':') != std::string_view::npos) unsupported("node id");
        int kc = -1;
        for (int k = 0; k < 3; k++)
            if (ks == kKinds[k]) kc = k;
        if (kc < 0) unsupported("node kind");
        const Val *at = f.get(P, "attrs"), *in = f.get(P, "inputs"), *sh = f.get(P, "output_shapes");
        if (at && at->t != J_OBJ) unsupported("attrs");
        if (in && in->t != J_ARR) unsupported("inputs");
        if (sh && sh->t != J_ARR) unsupported("output_shapes");
        raw[i] = NodeRef{ids, sv(P, *op), sv(P, *dev), kc, &o, at, in, sh};
        raw_ids[i] = ids;
    }
    // rank order: code-point order of ids == byte order of their UTF-8
    std::vector<uint32_t> order(N);
    for (uint32_t i = 0; i < N; i++) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return raw_ids[x] < raw_ids[y]; });
    IdTable rank;  // node id -> rank
    rank.build(raw_ids, order);
    // output shapes (dims as ints, dtype_bytes > 0), flat: node r's slot k has dims
    // dims[dim_off[shape_off[r] + k] .. dim_off[shape_off[r] + k + 1])
    std::vector<int64_t> dims_flat, dim_off{0};
    std::vector<uint32_t> shape_off(N + 1, 0);
    for (uint32_t r = 0; r < N; r++) {
        const NodeRef &n = raw[order[r]];
        shape_off[r + 1] = shape_off[r] + (n.shapes ? n.shapes->n : 0);
        if (!n.shapes) continue;
        for (uint32_t k = 0; k < n.shapes->n; k++) {
            const Val &s = P.vals[P.kids[n.shapes->a + k]];
            if (s.t != J_OBJ) unsupported("output shape");
            const Fields f = fields_of(P, s, {"dims", "dtype_bytes"});
            const Val *dims = f.get(P, "dims"), *db = f.get(P, "dtype_bytes");
            if (!dims || dims->t != J_ARR) unsupported("output shape dims");
            if (db && !(db->t == J_INT && db->i > 0)) unsupported("dtype_bytes");
            for (uint32_t j = 0; j < dims->n; j++) {
                const Val &d = P.vals[P.kids[dims->a + j]];
                if (d.t != J_INT || d.i < 0) unsupported("dimension");
                dims_flat.push_back(d.i);
            }
            dim_off.push_back(static_cast<int64_t>(dims_flat.size()));
        }
    }
    // devices of the nodes (sorted), ops (first appearance in rank order)
    std::vector<std::string_view> devs;
    {
        std::unordered_map<std::string_view, int32_t> seen;
        for (uint32_t r = 0; r < N; r++)
            if (seen.emplace(raw[r].dev, 0).second) devs.push_back(raw[r].dev);
    }
    std::sort(devs.begin(), devs.end());
    std::unordered_map<std::string_view, int32_t> drank, op_ids;
    for (size_t k = 0; k < devs.size(); k++) {
        drank.emplace(devs[k], static_cast<int32_t>(k));
        D.dev_off.push_back(static_cast<int64_t>(D.dev_blob.size()));
        D.dev_blob.append(devs[k].data(), devs[k].size());
    }
    D.dev_off.push_back(static_cast<int64_t>(D.dev_blob.size()));
    D.queue_off.assign(devs.size() + 1, 0);
    // per node, rank order
    std::vector<int32_t> prods, cons;
    // signature dedup (tuple equality: -0.0 == 0.0): open addressing on a content hash
    std::vector<int32_t> sig_slot(1024, -1);
    std::vector<uint64_t> sig_hash;
    std::unordered_map<std::string, int32_t> fname_ids;
    std::vector<std::string> fnames;
    std::vector<std::pair<std::string_view, double>> feats;
    char genbuf[8192];  // this node's generated in<i>_dim<j> names (views into it live for one node)
    auto sig_equal = [&](int32_t sid) {
        const int64_t b = D.sig_off[sid], e = D.sig_off[sid + 1];
        if (e - b != static_cast<int64_t>(feats.size())) return false;
        for (int64_t j = b; j < e; j++) {
            const auto &f = feats[static_cast<size_t>(j - b)];
            if (f.second != D.fval[j] || fnames[D.fname[j]] != f.first) return false;
        }
        return true;
    };
    D.sig_off.push_back(0);
    for (uint32_t r = 0; r < N; r++) {
        const NodeRef &n = raw[order[r]];
        D.id_off.push_back(static_cast<int64_t>(D.id_blob.size()));
        D.id_blob.append(n.id.data(), n.id.size());
        D.node_lo.push_back(n.obj->lo);
        D.node_hi.push_back(n.obj->hi);
        auto it = op_ids.find(n.op);
        if (it == op_ids.end()) {
            it = op_ids.emplace(n.op, static_cast<int32_t>(op_ids.size())).first;
            D.op_off.push_back(static_cast<int64_t>(D.op_blob.size()));
            D.op_blob.append(n.op.data(), n.op.size());
        }
        D.op_of.push_back(it->second);
        D.kind_of.push_back(static_cast<uint8_t>(n.kind));
        const int32_t dv = drank[n.dev];
        D.dev_of.push_back(dv);
        D.queue_off[dv + 1]++;
        // inputs: "producer:slot" (rpartition), producer must exist and own the slot
        const uint32_t nin = n.inputs ? n.inputs->n : 0;
        D.indeg.push_back(static_cast<int32_t>(nin));
        D.max_indeg = std::max<int32_t>(D.max_indeg, static_cast<int32_t>(nin));
        feats.clear();
        int genlen = 0;
        if (n.attrs) {
            for (uint32_t k = 0; k < n.attrs->n; k++) {
                const std::string_view an = sv(P, P.vals[P.kids[n.attrs->a + 2 * k]]);
                for (uint32_t q = 0; q < k; q++)
                    if (sv(P, P.vals[P.kids[n.attrs->a + 2 * q]]) == an) unsupported("duplicate attr");
                const Val &av = P.vals[P.kids[n.attrs->a + 2 * k + 1]];
                if (av.t == J_INT || av.t == J_FLOAT) feats.emplace_back(an, av.d);
            }
        }
        for (uint32_t k = 0; k < nin; k++) {
            const Val &ref = P.vals[P.kids[n.inputs->a + k]];
            if (ref.t != J_STR) unsupported("input reference");
            const std::string_view rs = sv(P, ref);
            const size_t colon = rs.rfind(':');
            if (colon == std::string_view::npos) unsupported("input reference");
            const std::string_view pid = rs.substr(0, colon), slot_s = rs.substr(colon + 1);
            if (slot_s.empty() || slot_s.size() > 9) unsupported("slot");
            int64_t slot = 0;
            for (char ch : slot_s) {
                if (ch < '0' || ch > '9') unsupported("slot");
                slot = slot * 10 + (ch - '0');
            }
            const int32_t q = rank.find(pid);
            if (q < 0) unsupported("missing producer");
            const int64_t nshapes = shape_off[q + 1] - shape_off[q];
            if (!(slot < std::max<int64_t>(1, nshapes))) unsupported("bad slot");
            prods.push_back(q);
            cons.push_back(static_cast<int32_t>(r));
            if (slot < nshapes) {  // node_features' in<i>_dim<j>
                const int64_t sh = shape_off[q] + slot;
                for (int64_t j = 0; j < dim_off[sh + 1] - dim_off[sh]; j++) {
                    if (genlen + 48 > static_cast<int>(sizeof genbuf)) unsupported("too many input dims");
                    char *nm = genbuf + genlen;
                    int len = 0;
                    auto put_uint = [&](uint64_t x) {
                        char tmp[24];
                        int t = 0;
                        do { tmp[t++] = static_cast<char>('0' + x % 10); x /= 10; } while (x);
                        while (t) nm[len++] = tmp[--t];
                    };
                    nm[len++] = 'i';
                    nm[len++] = 'n';
                    put_uint(k);
                    std::memcpy(nm + len, "_dim", 4);
                    len += 4;
                    put_uint(static_cast<uint64_t>(j));
                    const std::string_view nv(nm, static_cast<size_t>(len));
                    genlen += len;
                    for (auto &e : feats)
                        if (e.first == nv) unsupported("attr name collides with an input dim");
                    feats.emplace_back(nv, static_cast<double>(dims_flat[dim_off[sh] + j]));
                }
            }
        }
        std::sort(feats.begin(), feats.end(), [](auto &x, auto &y) { return x.first < y.first; });
        uint64_t hk = 1469598103934665603ull;
        for (auto &e : feats) {
            hk = hash_bytes(e.first.data(), e.first.size(), hk) * 31;
            const double v = e.second == 0.0 ? 0.0 : e.second;  // tuple equality: -0.0 == 0.0
            hk = hash_bytes(reinterpret_cast<const char *>(&v), sizeof v, hk);
        }
        uint64_t h = hk & (sig_slot.size() - 1);
        int32_t sid = -1;
        while (sig_slot[h] >= 0) {
            if (sig_hash[sig_slot[h]] == hk && sig_equal(sig_slot[h])) {
                sid = sig_slot[h];
                break;
            }
            h = (h + 1) & (sig_slot.size() - 1);
        }
        if (sid < 0) {
            sid = static_cast<int32_t>(sig_hash.size());
            sig_slot[h] = sid;
            sig_hash.push_back(hk);
            for (auto &e : feats) {
                auto fi = fname_ids.find(std::string(e.first));
                if (fi == fname_ids.end()) {
                    fi = fname_ids.emplace(std::string(e.first), static_cast<int32_t>(fnames.size())).first;
                    fnames.emplace_back(e.first);
                }
                D.fname.push_back(fi->second);
                D.fval.push_back(e.second);  // the first-appearing values represent the signature
            }
            D.sig_off.push_back(static_cast<int64_t>(D.fname.size()));
            if (sig_hash.size() * 2 > sig_slot.size()) {  // grow and rehash
                std::vector<int32_t> bigger(sig_slot.size() * 2, -1);
                for (size_t k = 0; k < sig_hash.size(); k++) {
                    uint64_t q = sig_hash[k] & (bigger.size() - 1);
                    while (bigger[q] >= 0) q = (q + 1) & (bigger.size() - 1);
                    bigger[q] = static_cast<int32_t>(k);
                }
                sig_slot.swap(bigger);
            }
        }
        D.sig_of.push_back(sid);
        // communication attributes (node_rows: costmodel.py:347-376 inputs)
        uint8_t ok = 0;
        int64_t bytes = 0;
        int32_t grp = 0;
        double thr = 1.0, lat = 0.0;
        const Val *b = nullptr, *g = nullptr;
        if (n.attrs) {
            for (uint32_t k = 0; k < n.attrs->n; k++) {
                const std::string_view an = sv(P, P.vals[P.kids[n.attrs->a + 2 * k]]);
                if (an == "bytes") b = &P.vals[P.kids[n.attrs->a + 2 * k + 1]];
                if (an == "group") g = &P.vals[P.kids[n.attrs->a + 2 * k + 1]];
            }
        }
        if (b && (b->t == J_TRUE || b->t == J_FALSE)) unsupported("boolean bytes");  // an int in Python
        if (n.kind == 1) {  // Transfer on a declared Link device with integer bytes
            auto d = dec_index.find(n.dev);
            if (d != dec_index.end() && D.dec_kind[d->second] == 1 && b && b->t == J_INT) {
                ok = 1;
                bytes = b->i;
                thr = D.dec_thr[d->second];
                lat = D.dec_lat[d->second];
            }
        } else if (n.kind == 2) {  // Collective with a group list and integer bytes
            if (g && g->t == J_ARR && b && b->t == J_INT) {
                ok = 1;
                bytes = b->i;
                grp = static_cast<int32_t>(g->n);
            }
        }
        D.comm_ok.push_back(ok);
        D.comm_bytes.push_back(bytes);
        D.group_size.push_back(grp);
        D.link_thr.push_back(thr);
        D.link_lat.push_back(lat);
    }
    D.id_off.push_back(static_cast<int64_t>(D.id_blob.size()));
    D.op_off.push_back(static_cast<int64_t>(D.op_blob.size()));
    for (auto &nm : fnames) {
        D.fname_off.push_back(static_cast<int64_t>(D.fname_blob.size()));
        D.fname_blob += nm;
    }
    D.fname_off.push_back(static_cast<int64_t>(D.fname_blob.size()));
    for (size_t k = 1; k < D.queue_off.size(); k++) D.queue_off[k] += D.queue_off[k - 1];
    // successor CSR: consumers ascending per producer, with multiplicity (graph.py:122-130)
    D.succ_off.assign(N + 1, 0);
    for (int32_t pr : prods) D.succ_off[pr + 1]++;
    for (uint32_t r = 0; r < N; r++) D.succ_off[r + 1] += D.succ_off[r];
    D.succ_idx.assign(prods.size(), 0);
    std::vector<int32_t> fill(D.succ_off.begin(), D.succ_off.end() - 1);
    for (size_t e = 0; e < prods.size(); e++) D.succ_idx[fill[prods[e]]++] = cons[e];
    for (uint32_t r = 0; r < N; r++)
        if (D.indeg[r] == 0) D.sources.push_back(static_cast<int32_t>(r));
}

template <typename T>
const T *ptr_or_null(const std::vector<T> &v) { return v.empty() ? nullptr : v.data(); }

void fill_view(Doc &D) {
    dfsim_document &v = D.view;
    v.n_nodes = static_cast<int32_t>(D.op_of.size());
    v.n_edges = static_cast<int64_t>(D.succ_idx.size());
    v.n_devices = static_cast<int32_t>(D.dev_off.size()) - 1;
    v.n_ops = static_cast<int32_t>(D.op_off.size()) - 1;
    v.n_sigs = static_cast<int32_t>(D.sig_off.size()) - 1;
    v.n_fnames = static_cast<int32_t>(D.fname_off.size()) - 1;
    v.n_declared = static_cast<int32_t>(D.dec_kind.size());
    v.max_indeg = D.max_indeg;
    v.id_blob = D.id_blob.data(); v.id_off = D.id_off.data();
    v.op_blob = D.op_blob.data(); v.op_off = D.op_off.data();
    v.dev_blob = D.dev_blob.data(); v.dev_off = D.dev_off.data();
    v.fname_blob = D.fname_blob.data(); v.fname_off = D.fname_off.data();
    v.op_of = ptr_or_null(D.op_of); v.kind_of = ptr_or_null(D.kind_of); v.dev_of = ptr_or_null(D.dev_of);
    v.indeg = ptr_or_null(D.indeg); v.succ_off = D.succ_off.data(); v.succ_idx = ptr_or_null(D.succ_idx);
    v.sources = ptr_or_null(D.sources); v.n_sources = static_cast<int32_t>(D.sources.size());
    v.queue_off = D.queue_off.data();
    v.sig_of = ptr_or_null(D.sig_of); v.sig_off = D.sig_off.data();
    v.sig_fname = ptr_or_null(D.fname); v.sig_fval = ptr_or_null(D.fval);
    v.comm_ok = ptr_or_null(D.comm_ok); v.comm_bytes = ptr_or_null(D.comm_bytes);
    v.group_size = ptr_or_null(D.group_size); v.link_thr = ptr_or_null(D.link_thr);
    v.link_lat = ptr_or_null(D.link_lat);
    v.node_lo = ptr_or_null(D.node_lo); v.node_hi = ptr_or_null(D.node_hi);
    v.meta_lo = D.meta_lo; v.meta_hi = D.meta_hi;
    v.decl_lo = D.decl_lo; v.decl_hi = D.decl_hi;
}

}  // namespace

extern "C" int dfsim_document_parse(const char *text, int64_t len, void **out, char *why, int64_t why_cap) {
    if (!text || len < 0 || !out) return DFSIM_BAD_ARGUMENT;
    *out = nullptr;
    Doc *D = new Doc();
    try {
        if (len >= (int64_t(1) << 32)) unsupported("document larger than 4 GB");
        Parser P{text, len};
        P.vals.reserve(static_cast<size_t>(len / 16) + 16);
        P.kids.reserve(static_cast<size_t>(len / 16) + 16);
        P.pool.reserve(static_cast<size_t>(len / 3) + 16);
        const uint32_t root = P.value(0);
        P.ws();
        if (P.p != len) unsupported("trailing data");
        build(*D, P, root);
    } catch (const Unsupported &u) {
        if (why && why_cap > 0) {
            std::strncpy(why, u.why.c_str(), static_cast<size_t>(why_cap - 1));
            why[why_cap - 1] = '\0';
        }
        delete D;
        return DFSIM_CONFIG;  // not loaded here: the caller re-parses with the reference semantics
    }
    fill_view(*D);
    *out = D;
    return DFSIM_OK;
}

extern "C" const dfsim_document *dfsim_document_view(const void *doc) {
    return doc ? &static_cast<const Doc *>(doc)->view : nullptr;
}

extern "C" void dfsim_document_free(void *doc) { delete static_cast<Doc *>(doc); }
