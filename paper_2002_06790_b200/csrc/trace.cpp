// Chrome trace writer: reporting.to_trace (reporting.py:43-74), byte-identical to
// json.dumps(events, indent=1) + "\n" of the reference.
//
// Layout of the reference document: one "M" (thread_name) event per device of the
// schedule's busy dict in sorted order, then one "X" event per entry in entry order
// with ts = round(start), dur = round(finish - start) (Python round: half to even on
// the exact binary value), tid = rank of the device in that sorted list.  Strings are
// escaped like json.dumps(ensure_ascii=True): \" \\ \n \r \t \b \f, every other code
// point outside 0x20..0x7e as \uXXXX (UTF-16 surrogate pairs above 0xFFFF).
// Host code only: the schedule is already on the host when a trace is wanted.
#include <cfenv>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "dfsim_b200.h"

namespace {

const char kHex[] = "0123456789abcdef";

void put_u16(std::string &o, unsigned cp) {
    o += "\\u";
    o += kHex[(cp >> 12) & 15];
    o += kHex[(cp >> 8) & 15];
    o += kHex[(cp >> 4) & 15];
    o += kHex[cp & 15];
}

// Python str encoded as UTF-8 ('surrogatepass' for lone surrogates) -> JSON literal
void put_str(std::string &o, const char *p, size_t n) {
    o += '"';
    const auto *s = reinterpret_cast<const unsigned char *>(p);
    size_t i = 0;
    while (i < n) {
        size_t j = i;  // copy the longest run that needs no escaping in one append
        while (j < n && s[j] >= 0x20 && s[j] < 0x7f && s[j] != '"' && s[j] != '\\') j++;
        if (j > i) {
            o.append(p + i, j - i);
            i = j;
            continue;
        }
        unsigned c = s[i];
        if (c < 0x80) {
            i++;
            switch (c) {
                case '"': o += "\\\""; break;
                case '\\': o += "\\\\"; break;
                case '\n': o += "\\n"; break;
                case '\r': o += "\\r"; break;
                case '\t': o += "\\t"; break;
                case '\b': o += "\\b"; break;
                case '\f': o += "\\f"; break;
                default:
                    if (c < 0x20 || c == 0x7f) put_u16(o, c);
                    else o += static_cast<char>(c);
            }
            continue;
        }
        unsigned cp;
        int len;
        if ((c & 0xe0) == 0xc0) { cp = c & 0x1f; len = 2; }
        else if ((c & 0xf0) == 0xe0) { cp = c & 0x0f; len = 3; }
        else { cp = c & 0x07; len = 4; }
        for (int k = 1; k < len && i + k < n; k++) cp = (cp << 6) | (s[i + k] & 0x3f);
        i += len;
        if (cp > 0xffff) {
            cp -= 0x10000;
            put_u16(o, 0xd800 | (cp >> 10));
            put_u16(o, 0xdc00 | (cp & 0x3ff));
        } else {
            put_u16(o, cp);
        }
    }
    o += '"';
}

// Python round(x) of a finite float, printed as an int
void put_round(std::string &o, double x) {
    const double r = std::nearbyint(x) + 0.0;  // FE_TONEAREST: ties to even; + 0.0 drops -0
    char buf[400];
    if (std::fabs(r) < 9.0e15) {
        const auto res = std::to_chars(buf, buf + sizeof buf, static_cast<long long>(r));
        o.append(buf, res.ptr);
    } else {
        std::snprintf(buf, sizeof buf, "%.0f", r);  // exact integer value of the double
        o += buf;
    }
}

void put_int(std::string &o, long long v) {
    char buf[32];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    o.append(buf, res.ptr);
}

}  // namespace

extern "C" int64_t dfsim_trace_write(const dfsim_trace_tables *t, int64_t n_entries, const int32_t *entry_node,
                                     const double *start, const double *finish, char *buf, int64_t cap) {
    if (!t || n_entries < 0 || t->n_tracks < 0) return -1;
    if (n_entries > 0 && (!entry_node || !start || !finish || !t->id_blob || !t->id_off || !t->name_blob ||
                          !t->name_off || !t->tag || !t->tag_name || !t->track))
        return -1;
    if (t->n_tracks > 0 && !t->track_name) return -1;
    const int prev = std::fegetround();
    std::fesetround(FE_TONEAREST);
    std::string o;
    o.reserve(static_cast<size_t>(n_entries) * 160 + static_cast<size_t>(t->n_tracks) * 96 + 8);
    bool first = true;
    auto open_event = [&]() {
        o += first ? "[\n {\n" : ",\n {\n";
        first = false;
    };
    for (int32_t d = 0; d < t->n_tracks; d++) {
        open_event();
        o += "  \"name\": \"thread_name\",\n  \"ph\": \"M\",\n  \"pid\": 0,\n  \"tid\": ";
        put_int(o, d);
        o += ",\n  \"args\": {\n   \"name\": ";
        put_str(o, t->track_name[d], std::strlen(t->track_name[d]));
        o += "\n  }\n }";
    }
    for (int64_t e = 0; e < n_entries; e++) {
        const int32_t v = entry_node[e];
        if (v < 0 || v >= t->n_nodes) {
            std::fesetround(prev);
            return -1;
        }
        open_event();
        o += "  \"name\": ";
        put_str(o, t->name_blob + t->name_off[v], static_cast<size_t>(t->name_off[v + 1] - t->name_off[v]));
        o += ",\n  \"ph\": \"X\",\n  \"ts\": ";
        put_round(o, start[v]);
        o += ",\n  \"dur\": ";
        put_round(o, finish[v] - start[v]);
        o += ",\n  \"pid\": 0,\n  \"tid\": ";
        put_int(o, t->track[v]);
        o += ",\n  \"args\": {\n   \"node\": ";
        put_str(o, t->id_blob + t->id_off[v], static_cast<size_t>(t->id_off[v + 1] - t->id_off[v]));
        o += ",\n   \"source\": ";
        const char *tag = t->tag_name[t->tag[v]];
        put_str(o, tag, std::strlen(tag));
        o += "\n  }\n }";
    }
    o += first ? "[]\n" : "\n]\n";
    std::fesetround(prev);
    const int64_t len = static_cast<int64_t>(o.size());
    if (buf && cap >= len) std::memcpy(buf, o.data(), o.size());
    return len;
}
