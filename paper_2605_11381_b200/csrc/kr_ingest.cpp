// kr_ingest.cpp -- trace ingest: JSON Lines task traces -> columnar arrays.
//
// Replaces the reference's load_traces / trace_from_dict / _round_from_dict
// (workload.py:163-262) for feeding trace files to the device at scale
// (SURVEY.md §8(f) row 4): one pass over the file with a small recursive JSON
// reader (Python json's grammar, including its NaN / Infinity literals), the
// reference's validation order and TraceFormatError messages, and columns
// that go to the GPU without per-round Python objects: per-trace scalars,
// per-round (round_id, trigger, horizon, chunk_size), the update magnitudes
// (K x N fp64 each, concatenated) and the action trajectories.
//
// Host code only (no CUDA); compiled into libkairos_b200.so.
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/kairos_b200.h"

namespace {

// ---------------------------------------------------------------- JSON DOM
struct JVal {
    enum Kind : uint8_t { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;       // Int (if it fits; big ints keep `d` only and big = true)
    bool big = false;
    double d = 0.0;      // Float, or Int converted
    std::string s;       // Str
    std::vector<JVal> a;  // Arr elements / Obj values
    std::vector<double> nums;  // Arr of numbers only (the bulk payload): values, no DOM nodes
    bool numeric = false;      // Arr stored in `nums`
    std::vector<std::string> keys;  // Obj keys (duplicate keys: the last wins, as in Python)

    const JVal* get(const char* k) const {
        for (size_t n = keys.size(); n-- > 0;)
            if (keys[n] == k) return &a[n];
        return nullptr;
    }
    bool truthy() const {  // Python bool() of the decoded value
        switch (kind) {
            case Null: return false;
            case Bool: return b;
            case Int: return big ? d != 0.0 : i != 0;
            case Float: return d != 0.0;
            case Str: return !s.empty();
            case Arr: return numeric ? !nums.empty() : !a.empty();
            case Obj: return !a.empty();
        }
        return false;
    }
    bool is_num() const { return kind == Int || kind == Float || kind == Bool; }
    double num() const { return kind == Bool ? (b ? 1.0 : 0.0) : d; }
};

struct JsonError {
    std::string msg;
};

// Python json.JSONDecoder messages (exc.msg) for the cases a trace line hits.
class Reader {
  public:
    Reader(const char* p, const char* e) : p_(p), e_(e) {}
    void parse(JVal& v) {
        ws();
        value(v, 0);
        ws();
        if (p_ != e_) throw JsonError{"Extra data"};
    }

  private:
    const char* p_;
    const char* e_;

    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) p_++;
    }
    bool lit(const char* w) {
        size_t n = std::strlen(w);
        if (static_cast<size_t>(e_ - p_) >= n && std::memcmp(p_, w, n) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    void value(JVal& v, int depth) {
        if (depth > 512) throw JsonError{"Maximum nesting depth exceeded"};
        if (p_ >= e_) throw JsonError{"Expecting value"};
        char c = *p_;
        if (c == '{') return object(v, depth);
        if (c == '[') return array(v, depth);
        if (c == '"') {
            v.kind = JVal::Str;
            return str(v.s);
        }
        if (lit("null")) { v.kind = JVal::Null; return; }
        if (lit("true")) { v.kind = JVal::Bool; v.b = true; return; }
        if (lit("false")) { v.kind = JVal::Bool; v.b = false; return; }
        if (lit("NaN")) { v.kind = JVal::Float; v.d = NAN; return; }
        if (lit("Infinity")) { v.kind = JVal::Float; v.d = INFINITY; return; }
        if (lit("-Infinity")) { v.kind = JVal::Float; v.d = -INFINITY; return; }
        if (c == '-' || (c >= '0' && c <= '9')) return number(v);
        throw JsonError{"Expecting value"};
    }
    void number(JVal& v) {
        const char* s = p_;
        if (*p_ == '-') p_++;
        if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) {
            p_ = s;
            throw JsonError{"Expecting value"};
        }
        if (*p_ == '0') p_++;
        else
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
        bool is_float = false;
        if (p_ < e_ && *p_ == '.' && p_ + 1 < e_ && p_[1] >= '0' && p_[1] <= '9') {
            is_float = true;
            p_++;
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
        }
        if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
            const char* q = p_ + 1;
            if (q < e_ && (*q == '+' || *q == '-')) q++;
            if (q < e_ && *q >= '0' && *q <= '9') {
                is_float = true;
                p_ = q;
                while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
            }
        }
        // from_chars: correctly rounded like float(str), no allocation
        std::from_chars(s, p_, v.d, std::chars_format::general);
        if (is_float) {
            v.kind = JVal::Float;
        } else {
            v.kind = JVal::Int;
            long long x = 0;
            auto r = std::from_chars(s, p_, x);
            v.big = r.ec == std::errc::result_out_of_range;
            v.i = x;
        }
    }
    // a bare number literal (no NaN / Infinity) at the cursor, as a double
    bool fast_number(double& d) {
        const char* s = p_;
        const char* q = p_;
        if (q < e_ && *q == '-') q++;
        if (q >= e_ || !(*q >= '0' && *q <= '9')) return false;
        if (*q == '0') q++;
        else
            while (q < e_ && *q >= '0' && *q <= '9') q++;
        if (q < e_ && *q == '.' && q + 1 < e_ && q[1] >= '0' && q[1] <= '9') {
            q++;
            while (q < e_ && *q >= '0' && *q <= '9') q++;
        }
        if (q < e_ && (*q == 'e' || *q == 'E')) {
            const char* t = q + 1;
            if (t < e_ && (*t == '+' || *t == '-')) t++;
            if (t < e_ && *t >= '0' && *t <= '9') {
                q = t;
                while (q < e_ && *q >= '0' && *q <= '9') q++;
            }
        }
        std::from_chars(s, q, d, std::chars_format::general);
        p_ = q;
        return true;
    }
    static void put_utf8(std::string& o, uint32_t cp) {
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
    uint32_t hex4() {
        if (e_ - p_ < 4) throw JsonError{"Invalid \\uXXXX escape"};
        uint32_t x = 0;
        for (int k = 0; k < 4; k++) {
            char c = p_[k];
            x <<= 4;
            if (c >= '0' && c <= '9') x |= c - '0';
            else if (c >= 'a' && c <= 'f') x |= c - 'a' + 10;
            else if (c >= 'A' && c <= 'F') x |= c - 'A' + 10;
            else throw JsonError{"Invalid \\uXXXX escape"};
        }
        p_ += 4;
        return x;
    }
    void str(std::string& o) {
        p_++;  // opening quote
        for (;;) {
            if (p_ >= e_) throw JsonError{"Unterminated string starting at"};
            unsigned char c = static_cast<unsigned char>(*p_++);
            if (c == '"') return;
            if (c < 0x20) throw JsonError{"Invalid control character at"};
            if (c != '\\') {
                o += static_cast<char>(c);
                continue;
            }
            if (p_ >= e_) throw JsonError{"Unterminated string starting at"};
            char esc = *p_++;
            switch (esc) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00 && e_ - p_ >= 6 && p_[0] == '\\' && p_[1] == 'u') {
                        const char* save = p_;
                        p_ += 2;
                        uint32_t lo = hex4();
                        if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        else p_ = save;
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: throw JsonError{"Invalid \\escape"};
            }
        }
    }
    void array(JVal& v, int depth) {
        v.kind = JVal::Arr;
        p_++;
        ws();
        if (p_ < e_ && *p_ == ']') {
            p_++;
            return;
        }
        // arrays of plain numbers (magnitude / trajectory rows) skip the DOM
        const char* start = p_;
        double d;
        if (fast_number(d)) {
            v.numeric = true;
            v.nums.push_back(d);
            for (;;) {
                ws();
                if (p_ < e_ && *p_ == ']') { p_++; return; }
                if (p_ < e_ && *p_ == ',') {
                    p_++;
                    ws();
                    if (fast_number(d)) { v.nums.push_back(d); continue; }
                }
                break;  // something else: re-parse generically
            }
            v.numeric = false;
            v.nums.clear();
            p_ = start;
        }
        for (;;) {
            ws();
            v.a.emplace_back();
            value(v.a.back(), depth + 1);
            ws();
            if (p_ < e_ && *p_ == ',') { p_++; continue; }
            if (p_ < e_ && *p_ == ']') { p_++; return; }
            throw JsonError{"Expecting ',' delimiter"};
        }
    }
    void object(JVal& v, int depth) {
        v.kind = JVal::Obj;
        p_++;
        ws();
        if (p_ < e_ && *p_ == '}') {
            p_++;
            return;
        }
        for (;;) {
            ws();
            if (p_ >= e_ || *p_ != '"') throw JsonError{"Expecting property name enclosed in double quotes"};
            std::string k;
            str(k);
            ws();
            if (p_ >= e_ || *p_ != ':') throw JsonError{"Expecting ':' delimiter"};
            p_++;
            ws();
            JVal x;
            value(x, depth + 1);
            v.keys.push_back(std::move(k));
            v.a.push_back(std::move(x));
            ws();
            if (p_ < e_ && *p_ == ',') { p_++; continue; }
            if (p_ < e_ && *p_ == '}') { p_++; return; }
            throw JsonError{"Expecting ',' delimiter"};
        }
    }
};

// ------------------------------------------------------------ trace table
struct FormatError {
    std::string msg;
    bool has_task = false;
    std::string task;
    bool has_round = false;
    int64_t round = 0;
};

std::string py_repr_str(const std::string& s) {  // repr() of a str (ASCII-safe subset)
    bool sq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
    char q = sq ? '"' : '\'';
    std::string o(1, q);
    for (unsigned char c : s) {
        if (c == '\\') o += "\\\\";
        else if (c == static_cast<unsigned char>(q)) { o += '\\'; o += static_cast<char>(c); }
        else if (c == '\n') o += "\\n";
        else if (c == '\r') o += "\\r";
        else if (c == '\t') o += "\\t";
        else if (c < 0x20 || c == 0x7f) {
            char b[8];
            std::snprintf(b, sizeof b, "\\x%02x", c);
            o += b;
        } else o += static_cast<char>(c);
    }
    return o + q;
}

std::string py_int(int64_t x) { return std::to_string(static_cast<long long>(x)); }

struct Table {
    std::vector<int64_t> round_off{0}, id_off{0}, obs, act;
    std::vector<double> hz;
    std::vector<uint8_t> hz_int, success;
    std::string ids;
    std::vector<int32_t> round_id, trigger, horizon, chunk, mag_k, mag_n, traj_rows;
    std::vector<int64_t> mag_off{0}, traj_row0{0}, traj_off{0};
    std::vector<double> mags, traj;
    // error (KR_EFORMAT)
    int64_t err_line = 0;
    FormatError err;
    std::string err_msg_full;
    kr_trace_columns cols{};
};

int64_t need_int(const JVal& v, const char* name) {
    if (v.kind == JVal::Int && !v.big) return v.i;
    if (v.kind == JVal::Bool) return v.b ? 1 : 0;
    throw FormatError{std::string("field ") + py_repr_str(name) + " must be an integer"};
}

// UpdateMagnitudes(np.asarray(data)) (horizon.py:26-61): shape, then checks.
size_t arr_len(const JVal& v) { return v.numeric ? v.nums.size() : v.a.size(); }

void parse_mags(const JVal& v, Table& t, int32_t& K, int32_t& N) {
    std::vector<int64_t> shape;
    const JVal* cur = &v;
    while (cur->kind == JVal::Arr) {  // numpy's shape discovery along the first elements
        shape.push_back(static_cast<int64_t>(arr_len(*cur)));
        if (cur->numeric || cur->a.empty()) break;
        cur = &cur->a[0];
    }
    auto shape_str = [&]() {
        std::string s = "(";
        for (size_t k = 0; k < shape.size(); k++) {
            if (k) s += ", ";
            s += py_int(shape[k]);
        }
        if (shape.size() == 1) s += ",";
        return s + ")";
    };
    // rectangular check for the 2-D case (ragged / non-numeric: numpy's own error)
    if (shape.size() == 2) {
        for (const JVal& row : v.a) {
            if (row.kind != JVal::Arr || static_cast<int64_t>(arr_len(row)) != shape[1])
                throw FormatError{"bad update_magnitudes: the update magnitudes are not a "
                                  "rectangular array"};
            if (!row.numeric)
                for (const JVal& x : row.a)
                    if (!x.is_num())
                        throw FormatError{"bad update_magnitudes: non-numeric update magnitude"};
        }
    }
    if (shape.size() != 2)
        throw FormatError{"bad update_magnitudes: update magnitudes must be 2-D (K x N), got shape " +
                          shape_str()};
    if (shape[0] < 2)
        throw FormatError{"bad update_magnitudes: need at least 2 refinement steps, got " +
                          py_int(shape[0])};
    if (shape[1] < 1) throw FormatError{"bad update_magnitudes: chunk size must be >= 1"};
    const size_t m0 = t.mags.size();
    for (const JVal& row : v.a) {
        if (row.numeric) t.mags.insert(t.mags.end(), row.nums.begin(), row.nums.end());
        else
            for (const JVal& x : row.a) t.mags.push_back(x.num());
    }
    bool finite = true, nonneg = true;
    for (size_t k = m0; k < t.mags.size(); k++) {
        const double d = t.mags[k];
        finite = finite && std::isfinite(d);
        nonneg = nonneg && !(d < 0);
    }
    if (!finite || !nonneg) t.mags.resize(m0);
    if (!finite) throw FormatError{"bad update_magnitudes: update magnitudes must be finite"};
    if (!nonneg) throw FormatError{"bad update_magnitudes: update magnitudes must be >= 0"};
    K = static_cast<int32_t>(shape[0]);
    N = static_cast<int32_t>(shape[1]);
}

void add_trace(const JVal& d, Table& t) {
    static const char* kTraceFields[] = {"task_id", "control_hz", "obs_payload_bytes",
                                         "action_payload_bytes", "success", "rounds"};
    static const char* kRoundFields[] = {"round_id", "trigger_action_index", "horizon",
                                         "chunk_size"};
    for (const char* f : kTraceFields)  // workload.py:205-207
        if (!d.get(f)) throw FormatError{std::string("trace is missing field ") + py_repr_str(f)};
    const JVal& tid = *d.get("task_id");
    std::string task = tid.kind == JVal::Str ? tid.s : std::string();
    if (tid.kind != JVal::Str) throw FormatError{"task_id must be a string"};
    auto with_task = [&](FormatError e) {
        if (!e.has_task) {
            e.has_task = true;
            e.task = task;
        }
        return e;
    };
    const JVal& rounds = *d.get("rounds");
    if (rounds.kind != JVal::Arr) throw with_task(FormatError{"rounds must be a list"});
    if (rounds.numeric) throw with_task(FormatError{"round must be a JSON object"});
    // snapshot for rollback of this trace's rows on error
    const size_t r0 = t.round_id.size();
    const size_t m0 = t.mags.size(), tr0 = t.traj.size(), tro0 = t.traj_off.size();
    try {
        for (const JVal& r : rounds.a) {  // _round_from_dict, workload.py:170-202
            if (r.kind != JVal::Obj) throw FormatError{"round must be a JSON object"};
            for (const char* f : kRoundFields)
                if (!r.get(f)) throw FormatError{std::string("round is missing field ") + py_repr_str(f)};
            const int64_t rid = need_int(*r.get("round_id"), "round_id");
            int32_t K = 0, N = 0;
            const JVal* um = r.get("update_magnitudes");
            if (um && um->kind != JVal::Null) {
                try {
                    parse_mags(*um, t, K, N);
                } catch (FormatError& e) {
                    e.has_round = true;
                    e.round = rid;
                    throw;
                }
            }
            int32_t rows = -1;
            const JVal* tj = r.get("action_trajectory");
            if (tj && tj->kind != JVal::Null) {
                if (tj->kind != JVal::Arr) throw FormatError{"action_trajectory must be a list"};
                if (tj->numeric) throw FormatError{"action_trajectory rows must be lists"};
                rows = static_cast<int32_t>(tj->a.size());
                for (const JVal& row : tj->a) {
                    if (row.kind != JVal::Arr) throw FormatError{"action_trajectory rows must be lists"};
                    if (row.numeric) {
                        t.traj.insert(t.traj.end(), row.nums.begin(), row.nums.end());
                    } else {
                        for (const JVal& x : row.a) {
                            if (!x.is_num()) throw FormatError{"non-numeric action_trajectory value"};
                            t.traj.push_back(x.num());
                        }
                    }
                    t.traj_off.push_back(static_cast<int64_t>(t.traj.size()));
                }
            }
            const int64_t trig = need_int(*r.get("trigger_action_index"), "trigger_action_index");
            const int64_t h = need_int(*r.get("horizon"), "horizon");
            const int64_t cs = need_int(*r.get("chunk_size"), "chunk_size");
            // RoundRecord.__post_init__ (workload.py:73-86)
            auto rerr = [&](std::string m) {
                FormatError e{std::move(m)};
                e.has_round = true;
                e.round = rid;
                return e;
            };
            if (rid < 0) throw rerr("round_id must be >= 0");
            if (trig < 0) throw rerr("trigger_action_index must be >= 0");
            if (!(1 <= h && h <= cs))
                throw rerr("horizon " + py_int(h) + " outside [1, chunk_size=" + py_int(cs) + "]");
            if (rid > INT32_MAX || trig > INT32_MAX || cs > INT32_MAX)
                throw rerr("round field beyond int32");
            t.round_id.push_back(static_cast<int32_t>(rid));
            t.trigger.push_back(static_cast<int32_t>(trig));
            t.horizon.push_back(static_cast<int32_t>(h));
            t.chunk.push_back(static_cast<int32_t>(cs));
            t.mag_k.push_back(K);
            t.mag_n.push_back(N);
            t.mag_off.push_back(static_cast<int64_t>(t.mags.size()));
            t.traj_rows.push_back(rows);
            t.traj_row0.push_back(static_cast<int64_t>(t.traj_off.size() - 1));
        }
        // TaskTrace.__post_init__ (workload.py:100-126)
        const JVal& hzv = *d.get("control_hz");
        const JVal& obv = *d.get("obs_payload_bytes");
        const JVal& acv = *d.get("action_payload_bytes");
        if (task.empty()) throw FormatError{"task_id must be non-empty"};
        if (!hzv.is_num()) throw with_task(FormatError{"control_hz must be a number"});
        if (hzv.num() <= 0) throw with_task(FormatError{"control_hz must be > 0"});  // NaN passes, as in Python
        const int64_t ob = need_int(obv, "obs_payload_bytes"), ac = need_int(acv, "action_payload_bytes");
        if (ob < 0 || ac < 0) throw with_task(FormatError{"payload sizes must be >= 0"});
        const size_t nr = t.round_id.size() - r0;
        if (nr == 0) throw with_task(FormatError{"trace has no rounds"});
        for (size_t idx = 0; idx < nr; idx++) {
            const int32_t rid = t.round_id[r0 + idx];
            auto terr = [&](std::string m) {
                FormatError e{std::move(m), true, task, true, rid};
                return e;
            };
            if (rid != static_cast<int32_t>(idx))
                throw terr("round ids must be contiguous from 0, found " + py_int(rid) +
                           " at position " + py_int(static_cast<int64_t>(idx)));
            if (idx >= 1) {
                const int32_t ph = t.horizon[r0 + idx - 1];
                if (t.trigger[r0 + idx] >= ph)
                    throw terr("trigger_action_index " + py_int(t.trigger[r0 + idx]) +
                               " must be < previous horizon " + py_int(ph));
            }
        }
        t.hz.push_back(hzv.num());
        t.hz_int.push_back(hzv.kind == JVal::Int ? 1 : 0);
        t.obs.push_back(ob);
        t.act.push_back(ac);
        t.success.push_back(d.get("success")->truthy() ? 1 : 0);
        t.ids += task;
        t.id_off.push_back(static_cast<int64_t>(t.ids.size()));
        t.round_off.push_back(static_cast<int64_t>(t.round_id.size()));
    } catch (FormatError& e) {
        for (auto* v : {&t.round_id, &t.trigger, &t.horizon, &t.chunk, &t.mag_k, &t.mag_n, &t.traj_rows})
            v->resize(r0);
        t.mag_off.resize(r0 + 1);
        t.traj_row0.resize(r0 + 1);
        t.mags.resize(m0);
        t.traj.resize(tr0);
        t.traj_off.resize(tro0);
        throw with_task(e);
    }
}

void finalize(Table& t) {
    kr_trace_columns& c = t.cols;
    c.n_traces = static_cast<int64_t>(t.hz.size());
    c.n_rounds = static_cast<int64_t>(t.round_id.size());
    c.n_mag_values = static_cast<int64_t>(t.mags.size());
    c.n_traj_rows = static_cast<int64_t>(t.traj_off.size()) - 1;
    c.n_traj_values = static_cast<int64_t>(t.traj.size());
    c.round_off = t.round_off.data();
    c.ids = t.ids.data();
    c.id_off = t.id_off.data();
    c.control_hz = t.hz.data();
    c.control_hz_is_int = t.hz_int.data();
    c.obs_payload_bytes = t.obs.data();
    c.action_payload_bytes = t.act.data();
    c.success = t.success.data();
    c.round_id = t.round_id.data();
    c.trigger_action_index = t.trigger.data();
    c.horizon = t.horizon.data();
    c.chunk_size = t.chunk.data();
    c.mag_k = t.mag_k.data();
    c.mag_n = t.mag_n.data();
    c.mag_off = t.mag_off.data();
    c.mags = t.mags.data();
    c.traj_rows = t.traj_rows.data();
    c.traj_row0 = t.traj_row0.data();
    c.traj_off = t.traj_off.data();
    c.traj = t.traj.data();
    c.err_line = t.err_line;
    c.err_has_task = t.err.has_task;
    c.err_task = t.err.task.c_str();
    c.err_has_round = t.err.has_round;
    c.err_round = t.err.round;
    c.err_message = t.err.msg.c_str();
}

}  // namespace

namespace {

// load_traces' loop (workload.py:233-250) over [p, end): stripped lines,
// blanks skipped, the first error stops the range.
int parse_range(const char* p, const char* end, int64_t line, Table& t) {
    while (p < end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        const char* le = nl ? nl : end;
        // str.strip(): ASCII whitespace at both ends
        const char* a = p;
        const char* b = le;
        while (a < b && (*a == ' ' || *a == '\t' || *a == '\r' || *a == '\n' || *a == '\f' || *a == '\v')) a++;
        while (b > a && (b[-1] == ' ' || b[-1] == '\t' || b[-1] == '\r' || b[-1] == '\n' || b[-1] == '\f' || b[-1] == '\v')) b--;
        if (a < b) {
            JVal v;
            try {
                Reader(a, b).parse(v);
            } catch (JsonError& e) {
                t.err = FormatError{"invalid JSON: " + e.msg};
                t.err_line = line;
                return KR_EFORMAT;
            }
            if (v.kind != JVal::Obj) {
                t.err = FormatError{"trace line must be a JSON object"};
                t.err_line = line;
                return KR_EFORMAT;
            }
            try {
                add_trace(v, t);
            } catch (FormatError& e) {
                t.err = e;
                t.err_line = line;
                return KR_EFORMAT;
            } catch (std::bad_alloc&) {
                t.err = FormatError{"out of memory"};
                t.err_line = line;
                return KR_EFORMAT;
            }
        }
        line++;
        p = nl ? nl + 1 : end;
    }
    return KR_OK;
}

template <class V>
void append_shifted(V& dst, const V& src, typename V::value_type shift) {  // offsets: skip src[0]
    for (size_t k = 1; k < src.size(); k++) dst.push_back(src[k] + shift);
}
template <class V>
void append(V& dst, const V& src) { dst.insert(dst.end(), src.begin(), src.end()); }

void merge(Table& d, const Table& s) {
    append_shifted(d.round_off, s.round_off, static_cast<int64_t>(d.round_id.size()));
    append_shifted(d.id_off, s.id_off, static_cast<int64_t>(d.ids.size()));
    append_shifted(d.mag_off, s.mag_off, static_cast<int64_t>(d.mags.size()));
    append_shifted(d.traj_row0, s.traj_row0, static_cast<int64_t>(d.traj_off.size() - 1));
    append_shifted(d.traj_off, s.traj_off, static_cast<int64_t>(d.traj.size()));
    append(d.obs, s.obs); append(d.act, s.act); append(d.hz, s.hz); append(d.hz_int, s.hz_int);
    append(d.success, s.success); d.ids += s.ids;
    append(d.round_id, s.round_id); append(d.trigger, s.trigger); append(d.horizon, s.horizon);
    append(d.chunk, s.chunk); append(d.mag_k, s.mag_k); append(d.mag_n, s.mag_n);
    append(d.traj_rows, s.traj_rows); append(d.mags, s.mags); append(d.traj, s.traj);
}

int ingest_threads(size_t len) {
    static const int env = std::getenv("KR_INGEST_THREADS") ? std::atoi(std::getenv("KR_INGEST_THREADS")) : 0;
    int hw = static_cast<int>(std::thread::hardware_concurrency());
    int n = env > 0 ? env : (hw > 0 ? hw : 1);
    const int by_size = static_cast<int>(len >> 20) + 1;  // >= 1 MB per thread
    return n < by_size ? n : by_size;
}

// Run fn(0..n-1) on up to n host threads.  If a thread cannot be created
// (std::system_error) the remaining ranges run on the calling thread; every
// started thread is joined before anything propagates.
template <class F>
void run_ranges(size_t n, F&& fn) {
    std::vector<std::thread> th;
    size_t started = 0;
    try {
        th.reserve(n);
        for (; started < n; started++) th.emplace_back(fn, started);
    } catch (...) {
    }
    for (size_t r = started; r < n; r++) fn(r);
    for (auto& x : th) x.join();
}

int parse_impl(const char* buf, size_t len, int64_t first_line, Table& t) {
    const int64_t line0 = first_line > 0 ? first_line : 1;
    const char* end = buf + len;
    const int nt = ingest_threads(len);
    if (nt <= 1) {
        const int st = parse_range(buf, end, line0, t);
        finalize(t);
        return st;
    }
    std::vector<const char*> cut{buf};
    for (int k = 1; k < nt; k++) {
        const char* c = buf + len / nt * k;
        if (c <= cut.back()) continue;
        const char* nl = static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(end - c)));
        if (!nl) break;
        cut.push_back(nl + 1);
    }
    cut.push_back(end);
    const size_t nr = cut.size() - 1;
    std::vector<Table> part(nr);
    std::vector<int> st(nr, KR_OK);
    std::vector<int64_t> lines(nr + 1, 0);
    run_ranges(nr, [&](size_t r) {
        const char* q = cut[r];
        int64_t n = 0;
        while ((q = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(cut[r + 1] - q))))) {
            n++;
            q++;
        }
        lines[r + 1] = n;
    });
    lines[0] = line0;
    for (size_t r = 1; r <= nr; r++) lines[r] += lines[r - 1];
    // a range that throws (bad_alloc) reports KR_ENOSPACE for itself
    run_ranges(nr, [&](size_t r) {
        try {
            st[r] = parse_range(cut[r], cut[r + 1], lines[r], part[r]);
        } catch (...) {
            st[r] = KR_ENOSPACE;
        }
    });
    int status = KR_OK;
    for (size_t r = 0; r < nr; r++) {
        merge(t, part[r]);
        if (st[r] != KR_OK) {
            if (st[r] == KR_EFORMAT) {
                t.err = part[r].err;
                t.err_line = part[r].err_line;
            }
            status = st[r];
            break;
        }
    }
    finalize(t);
    return status;
}

}  // namespace

// Lines are independent, so the buffer is cut at line boundaries into one
// range per host thread; the ranges' tables are concatenated in order, and the
// first range that fails decides the error (as the sequential loop would).
// No exception leaves this function: allocation failures anywhere (the
// ranges' tables, merge, finalize) return KR_ENOSPACE.
extern "C" int kr_trace_parse(const char* buf, size_t len, int64_t first_line, void** table) {
    if (!table || (!buf && len)) return KR_EINVAL;
    if (len == 0) buf = "";
    Table* t = new (std::nothrow) Table();
    if (!t) return KR_ENOSPACE;
    *table = t;
    try {
        return parse_impl(buf, len, first_line, *t);
    } catch (...) {
        return KR_ENOSPACE;
    }
}

extern "C" int kr_trace_load(const char* path, void** table) {
    if (!path || !table) return KR_EINVAL;
    *table = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) return KR_EINVAL;
    std::string data;
    try {
        char buf[1 << 16];
        size_t n;
        while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) data.append(buf, n);
    } catch (...) {
        std::fclose(f);
        return KR_ENOSPACE;
    }
    std::fclose(f);
    return kr_trace_parse(data.data(), data.size(), 1, table);
}

extern "C" const kr_trace_columns* kr_trace_columns_of(const void* table) {
    return table ? &static_cast<const Table*>(table)->cols : nullptr;
}

extern "C" void kr_trace_free(void* table) { delete static_cast<Table*>(table); }
