// voxgeo text IO: the reference's read_grid / write_grid
// (voxstokes/geometry.py:243-339) as multithreaded C++ behind the C ABI.
//
// File format (geometry.py:246-250): "voxgeo 1" / "dim D" / "size N", then
// one line of N symbols {0,1} per x-run (x fastest, then y, then z), LF
// newlines.  The mask in memory is C-order (x, y, z) with z fastest, so
// reading and writing are a transpose: file line (z*n + y), column x <->
// fluid[x][y][z].  Both directions run as cache tiles (64 x-columns by
// all z) over host threads; a 1024^3 grid is a ~1.07 GB file.
//
// Errors.  A file the reference accepts is exactly: the three header lines,
// E = n^(dim-1) lines of n ASCII '0'/'1', then only empty lines.  The fast
// path checks that shape and transposes; anything else goes to a slow path
// that restates the reference's checks in their order (header, line count,
// trailing content, then per line: length in code points, first non-binary
// symbol) so the ValueError message is byte-identical, including Python's
// repr() of the offending token.  Invalid UTF-8 returns VS_EDECODE (the
// reference raises UnicodeDecodeError while reading; the Python wrapper
// re-raises that exact exception), open/read failures VS_EOS with errno.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/voxschur.h"

namespace vs {
void set_last_error(const std::string &msg);
}

namespace {

const char kMagic[] = "voxgeo 1";

int fail_value(const std::string &m) {
    vs::set_last_error(m);
    return VS_EVALUE;
}

int fail_os(int err) {
    vs::set_last_error(std::to_string(err));
    return VS_EOS;
}

// ------------------------------------------------------------ UTF-8 helpers

// Strict UTF-8 (what Python's decoder accepts: no overlongs, no surrogates,
// <= U+10FFFF).
bool valid_utf8(const unsigned char *p, size_t len) {
    size_t i = 0;
    while (i < len) {
        // ASCII run, 8 bytes at a time
        while (i + 8 <= len) {
            uint64_t w;
            memcpy(&w, p + i, 8);
            if (w & 0x8080808080808080ull) break;
            i += 8;
        }
        if (i >= len) break;
        unsigned c = p[i];
        if (c < 0x80) { ++i; continue; }
        int extra;
        uint32_t cp;
        if (c >= 0xC2 && c <= 0xDF) { extra = 1; cp = c & 0x1F; }
        else if (c >= 0xE0 && c <= 0xEF) { extra = 2; cp = c & 0x0F; }
        else if (c >= 0xF0 && c <= 0xF4) { extra = 3; cp = c & 0x07; }
        else return false;
        if (i + extra >= len) return false;
        for (int k = 1; k <= extra; ++k) {
            unsigned d = p[i + k];
            if ((d & 0xC0) != 0x80) return false;
            cp = (cp << 6) | (d & 0x3F);
        }
        if (extra == 2 && (cp < 0x800 || (cp >= 0xD800 && cp <= 0xDFFF))) return false;
        if (extra == 3 && (cp < 0x10000 || cp > 0x10FFFF)) return false;
        i += extra + 1;
    }
    return true;
}

// Decode one code point at p (valid UTF-8 assumed); returns its length.
int decode(const unsigned char *p, uint32_t *cp) {
    unsigned c = p[0];
    if (c < 0x80) { *cp = c; return 1; }
    if (c < 0xE0) { *cp = ((c & 0x1F) << 6) | (p[1] & 0x3F); return 2; }
    if (c < 0xF0) { *cp = ((c & 0x0F) << 12) | ((p[1] & 0x3F) << 6) | (p[2] & 0x3F); return 3; }
    *cp = ((c & 0x07) << 18) | ((p[1] & 0x3F) << 12) | ((p[2] & 0x3F) << 6) | (p[3] & 0x3F);
    return 4;
}

// Python's str.isspace() set (what str.split() splits on).
bool py_space(uint32_t c) {
    return (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x20) || c == 0x85 || c == 0xA0 ||
           c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 || c == 0x2029 ||
           c == 0x202F || c == 0x205F || c == 0x3000;
}

// str.isprintable() for the code points repr() escapes.  Exact for Latin-1
// and the common format/space/separator characters; other unassigned or
// private-use code points are printed verbatim (documented approximation).
bool py_printable(uint32_t c) {
    if (c < 0x20 || c == 0x7F) return false;
    if (c < 0x7F) return true;
    if (c <= 0xA0 || c == 0xAD) return false;
    if (c == 0x1680 || (c >= 0x2000 && c <= 0x200F) || (c >= 0x2028 && c <= 0x202F) ||
        (c >= 0x205F && c <= 0x2064) || (c >= 0x2066 && c <= 0x206F) || c == 0x3000 ||
        c == 0xFEFF || (c >= 0xFFF9 && c <= 0xFFFB) || (c >= 0xE000 && c <= 0xF8FF))
        return false;
    return true;
}

void append_utf8(std::string &s, uint32_t c) {
    if (c < 0x80) s += char(c);
    else if (c < 0x800) { s += char(0xC0 | (c >> 6)); s += char(0x80 | (c & 0x3F)); }
    else if (c < 0x10000) {
        s += char(0xE0 | (c >> 12)); s += char(0x80 | ((c >> 6) & 0x3F)); s += char(0x80 | (c & 0x3F));
    } else {
        s += char(0xF0 | (c >> 18)); s += char(0x80 | ((c >> 12) & 0x3F));
        s += char(0x80 | ((c >> 6) & 0x3F)); s += char(0x80 | (c & 0x3F));
    }
}

// repr() of a Python str given as UTF-8 bytes.
std::string py_repr(const std::string &u8) {
    std::vector<uint32_t> cps;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(u8.data());
    for (size_t i = 0; i < u8.size();) {
        uint32_t c;
        i += decode(p + i, &c);
        cps.push_back(c);
    }
    bool has_sq = std::find(cps.begin(), cps.end(), uint32_t('\'')) != cps.end();
    bool has_dq = std::find(cps.begin(), cps.end(), uint32_t('"')) != cps.end();
    char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string s(1, q);
    char buf[16];
    for (uint32_t c : cps) {
        if (c == uint32_t(q) || c == '\\') { s += '\\'; s += char(c); }
        else if (c == '\t') s += "\\t";
        else if (c == '\n') s += "\\n";
        else if (c == '\r') s += "\\r";
        else if (py_printable(c)) append_utf8(s, c);
        else {
            if (c < 0x100) snprintf(buf, sizeof buf, "\\x%02x", c);
            else if (c < 0x10000) snprintf(buf, sizeof buf, "\\u%04x", c);
            else snprintf(buf, sizeof buf, "\\U%08x", c);
            s += buf;
        }
    }
    s += q;
    return s;
}

// ------------------------------------------------------- integer helpers

// Python int(token) for a whitespace-free token: [+-]?digit(_?digit)*.
// Returns false if int() would raise; else the canonical str(int(token)).
bool py_int(const std::string &t, std::string *canon) {
    size_t i = 0;
    bool neg = false;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) { neg = t[i] == '-'; ++i; }
    if (i >= t.size()) return false;
    std::string digits;
    bool prev_digit = false;
    for (; i < t.size(); ++i) {
        char c = t[i];
        if (c >= '0' && c <= '9') { digits += c; prev_digit = true; }
        else if (c == '_' && prev_digit && i + 1 < t.size()) prev_digit = false;
        else return false;
    }
    if (!prev_digit) return false;
    size_t nz = digits.find_first_not_of('0');
    digits = nz == std::string::npos ? "0" : digits.substr(nz);
    *canon = (neg && digits != "0") ? "-" + digits : digits;
    return true;
}

// Decimal product of two non-negative canonical integers.
std::string dec_mul(const std::string &a, const std::string &b) {
    std::vector<int> r(a.size() + b.size(), 0);
    for (int i = int(a.size()) - 1; i >= 0; --i)
        for (int j = int(b.size()) - 1; j >= 0; --j) {
            int k = i + j + 1;
            int v = r[k] + (a[i] - '0') * (b[j] - '0');
            r[k] = v % 10;
            r[k - 1] += v / 10;
        }
    std::string s;
    for (int d : r)
        if (!(s.empty() && d == 0)) s += char('0' + d);
    return s.empty() ? "0" : s;
}

// canonical non-negative decimal <= 2^62 -> value, else -1
int64_t dec_small(const std::string &c) {
    if (c.empty() || c[0] == '-' || c.size() > 18) return -1;
    return std::stoll(c);
}

// --------------------------------------------------------------- lines

struct Line {
    size_t off, len;  // bytes, without the '\n'
};

// All lines of text.split("\n").
std::vector<Line> split_all(const std::string &b) {
    std::vector<Line> out;
    size_t s = 0;
    for (;;) {
        size_t e = b.find('\n', s);
        if (e == std::string::npos) { out.push_back({s, b.size() - s}); break; }
        out.push_back({s, e - s});
        s = e + 1;
    }
    return out;
}

// str.split() of one line (UTF-8 bytes) into UTF-8 tokens.
std::vector<std::string> py_split(const std::string &b, Line l) {
    std::vector<std::string> parts;
    std::string cur;
    bool in = false;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(b.data()) + l.off;
    for (size_t i = 0; i < l.len;) {
        uint32_t c;
        int k = decode(p + i, &c);
        if (py_space(c)) {
            if (in) { parts.push_back(cur); cur.clear(); in = false; }
        } else {
            cur.append(reinterpret_cast<const char *>(p + i), k);
            in = true;
        }
        i += k;
    }
    if (in) parts.push_back(cur);
    return parts;
}

// geometry.py:320-339
int header_int(const std::string &b, const std::vector<Line> &lines, size_t index,
               const char *key, std::string *canon) {
    std::string ln = "line " + std::to_string(index + 1) + ": malformed header, ";
    if (index >= lines.size()) return fail_value(ln + "missing " + py_repr(key));
    auto parts = py_split(b, lines[index]);
    if (parts.size() != 2 || parts[0] != key)
        return fail_value(ln + "expected " + py_repr(key) + " <integer>");
    if (!py_int(parts[1], canon))
        return fail_value(ln + py_repr(key) + " value " + py_repr(parts[1]) + " is not an integer");
    return VS_OK;
}

// geometry.py:275-289: magic, dim, size.  On success *dim, *n_canon.
int parse_header(const std::string &b, const std::vector<Line> &lines, int *dim,
                 std::string *n_canon) {
    if (lines.empty() || b.compare(lines[0].off, lines[0].len, kMagic) != 0 ||
        lines[0].len != strlen(kMagic))
        return fail_value(std::string("line 1: malformed header, expected ") + py_repr(kMagic));
    std::string d;
    if (int rc = header_int(b, lines, 1, "dim", &d)) return rc;
    if (d != "2" && d != "3")
        return fail_value("line 2: malformed header, dim must be 2 or 3, got " + d);
    *dim = d[0] - '0';
    if (int rc = header_int(b, lines, 2, "size", n_canon)) return rc;
    if ((*n_canon)[0] == '-' || *n_canon == "0" || *n_canon == "1")
        return fail_value("line 3: malformed header, size must be at least 2, got " + *n_canon);
    return VS_OK;
}

size_t n_codepoints(const std::string &b, Line l) {
    size_t c = 0;
    for (size_t i = 0; i < l.len; ++i)
        c += (static_cast<unsigned char>(b[l.off + i]) & 0xC0) != 0x80;
    return c;
}

// The reference's data-section checks in order (geometry.py:291-318); only
// reached when the fast path found an anomaly, so it always fails.
int slow_errors(const std::string &b, const std::vector<Line> &lines, const std::string &n_canon,
                int dim) {
    std::string e_canon = dim == 2 ? n_canon : dec_mul(n_canon, n_canon);
    int64_t n = dec_small(n_canon);
    int64_t E = dec_small(e_canon);  // -1 if astronomically large
    size_t avail = lines.size() > 3 ? lines.size() - 3 : 0;
    size_t take = (E < 0) ? avail : std::min<size_t>(avail, size_t(E));
    bool short_ = E < 0 || avail < size_t(E);
    size_t found = 0;
    bool empty_row = false;
    for (size_t k = 0; k < take; ++k) {
        if (lines[3 + k].len) ++found;
        else empty_row = true;
    }
    if (short_ || empty_row)
        return fail_value("size mismatch: expected " + e_canon + " data lines of " + n_canon +
                          " symbols, found " + std::to_string(found));
    for (size_t k = 3 + size_t(E); k < lines.size(); ++k)
        if (lines[k].len)
            return fail_value("line " + std::to_string(4 + E) +
                              ": size mismatch: unexpected content after data");
    const unsigned char *p = reinterpret_cast<const unsigned char *>(b.data());
    for (int64_t k = 0; k < E; ++k) {
        Line l = lines[3 + k];
        int64_t lineno = 4 + k;
        size_t len = n_codepoints(b, l);
        if (int64_t(len) != n)
            return fail_value("line " + std::to_string(lineno) + ": size mismatch: expected " +
                              n_canon + " symbols, found " + std::to_string(len));
        size_t col = 0;
        for (size_t i = 0; i < l.len;) {
            uint32_t c;
            int w = decode(p + l.off + i, &c);
            ++col;
            if (c != '0' && c != '1') {
                std::string ch;
                append_utf8(ch, c);
                return fail_value("line " + std::to_string(lineno) + ", column " +
                                  std::to_string(col) + ": non-binary voxel symbol " + py_repr(ch));
            }
            i += w;
        }
    }
    return fail_value("internal: voxgeo slow path found no error");
}

int n_threads(int64_t work) {
    unsigned hw = std::thread::hardware_concurrency();
    int t = int(std::min<unsigned>(hw ? hw : 1, 32));
    if (work < (int64_t(1) << 20)) t = 1;
    return std::max(t, 1);
}

template <class F>
void parallel_for(int64_t count, int threads, F f) {
    if (threads <= 1 || count <= 1) { f(int64_t(0), count); return; }
    std::vector<std::thread> th;
    int64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        int64_t a = t * per, e = std::min(count, a + per);
        if (a >= e) break;
        th.emplace_back([=] { f(a, e); });
    }
    for (auto &x : th) x.join();
}

int read_file(const char *path, std::string *out) {
    FILE *f = fopen(path, "rb");
    if (!f) return fail_os(errno);
    std::string b;
    char buf[1 << 16];
    if (fseek(f, 0, SEEK_END) == 0) {
        long sz = ftell(f);
        if (sz > 0) b.reserve(size_t(sz));
        fseek(f, 0, SEEK_SET);
    }
    size_t got;
    while ((got = fread(buf, 1, sizeof buf, f)) > 0) b.append(buf, got);
    int err = ferror(f) ? errno : 0;
    fclose(f);
    if (err) return fail_os(err);
    *out = std::move(b);
    return VS_OK;
}

}  // namespace

extern "C" {

int vs_grid_header(const char *path, int *dim, int64_t *n) {
    FILE *f = fopen(path, "rb");
    if (!f) return fail_os(errno);
    char buf[4096];
    size_t got = fread(buf, 1, sizeof buf, f);
    long fsize = (fseek(f, 0, SEEK_END) == 0) ? ftell(f) : -1;
    fclose(f);
    std::string b(buf, got);
    // only the three header lines matter; drop a possibly cut fourth line
    size_t nl = 0, pos = 0;
    for (int k = 0; k < 3 && (pos = b.find('\n', nl)) != std::string::npos; ++k) nl = pos + 1;
    b.resize(std::min(b.size(), nl ? nl : b.size()));
    if (!valid_utf8(reinterpret_cast<const unsigned char *>(b.data()), b.size()))
        return fail_value("header is not UTF-8");
    auto lines = split_all(b);
    std::string n_canon;
    int d = 0;
    if (int rc = parse_header(b, lines, &d, &n_canon)) return rc;
    int64_t nn = dec_small(n_canon);
    if (nn < 0 || nn > (int64_t(1) << 20)) return fail_value("size " + n_canon + " is out of range");
    // a file too short for its data section: no buffer is sized from it (the
    // full read reports the reference's size-mismatch error instead)
    const int64_t rows = d == 2 ? nn : nn * nn;
    if (fsize >= 0 && fsize < int64_t(nl) + rows * (nn + 1) - 1) return fail_value("file too short");
    *dim = d;
    *n = nn;
    return VS_OK;
}

int vs_read_grid(const char *path, uint8_t *fluid, int64_t cap, int *dim_out, int64_t *n_out) {
    std::string b;
    if (int rc = read_file(path, &b)) return rc;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(b.data());
    if (!valid_utf8(p, b.size())) {
        vs::set_last_error("invalid UTF-8");
        return VS_EDECODE;
    }
    // header: the first three lines only (the data lines are not split here)
    std::vector<Line> head;
    size_t s = 0;
    while (head.size() < 3) {
        size_t e = b.find('\n', s);
        if (e == std::string::npos) { head.push_back({s, b.size() - s}); s = b.size() + 1; break; }
        head.push_back({s, e - s});
        s = e + 1;
    }
    int dim = 0;
    std::string n_canon;
    if (int rc = parse_header(b, head, &dim, &n_canon)) return rc;
    int64_t n = dec_small(n_canon);
    int64_t E = (n < 0 || n > (int64_t(1) << 20)) ? -1 : (dim == 2 ? n : n * n);
    // fast path: E lines of n '0'/'1' each, then only '\n'
    bool ok = E > 0 && s <= b.size() && int64_t(b.size() - s) >= E * (n + 1) - 1;
    const size_t base = s;
    if (ok) {
        int T = n_threads(E * n);
        std::vector<char> bad(size_t(std::max(T, 1)), 0);
        int64_t per = (E + T - 1) / T;
        parallel_for(E, T, [&](int64_t a, int64_t e) {
            bool good = true;
            for (int64_t k = a; k < e && good; ++k) {
                const unsigned char *q = p + base + size_t(k) * size_t(n + 1);
                for (int64_t x = 0; x < n; ++x) good &= (q[x] | 1) == '1';
                size_t end = base + size_t(k) * size_t(n + 1) + size_t(n);
                if (end < b.size()) good &= q[n] == '\n';
                else good &= (k == E - 1 && end == b.size());
            }
            if (!good) bad[size_t(a / per)] = 1;
        });
        for (char c : bad) ok &= !c;
        if (ok)
            for (size_t i = base + size_t(E) * size_t(n + 1); i < b.size(); ++i)
                if (b[i] != '\n') { ok = false; break; }
    }
    if (!ok) return slow_errors(b, split_all(b), n_canon, dim);
    *dim_out = dim;
    *n_out = n;
    int64_t cells = dim == 2 ? n * n : n * n * n;
    if (!fluid) return VS_OK;
    if (cap < cells) {
        vs::set_last_error("output buffer too small");
        return VS_EVALUE;
    }
    // transpose: file line L = (z*n + y) [3D] or y [2D], column x ->
    // fluid[x][y][z] / fluid[x][y]; tiles of 64 x-columns stream n output
    // rows each.
    const int64_t XB = 64;
    const int64_t xblocks = (n + XB - 1) / XB;
    const int64_t rows = dim == 2 ? 1 : n;  // y values per tile in 3D
    parallel_for(xblocks * rows, n_threads(cells), [&](int64_t a, int64_t e) {
        for (int64_t t = a; t < e; ++t) {
            int64_t xb = t / rows, y = t % rows;
            int64_t x0 = xb * XB, x1 = std::min(n, x0 + XB);
            if (dim == 2) {
                for (int64_t yy = 0; yy < n; ++yy) {
                    const unsigned char *q = p + base + size_t(yy) * size_t(n + 1);
                    for (int64_t x = x0; x < x1; ++x) fluid[x * n + yy] = q[x] & 1;
                }
            } else {
                for (int64_t z = 0; z < n; ++z) {
                    const unsigned char *q = p + base + size_t(z * n + y) * size_t(n + 1);
                    uint8_t *o = fluid + y * n + z;
                    for (int64_t x = x0; x < x1; ++x) o[x * n * n] = q[x] & 1;
                }
            }
        }
    });
    return VS_OK;
}

int vs_write_grid(const char *path, const uint8_t *fluid, int dim, int64_t n) {
    if ((dim != 2 && dim != 3) || n < 2) return fail_value("invalid grid shape");
    std::string head = std::string(kMagic) + "\ndim " + std::to_string(dim) + "\nsize " +
                       std::to_string(n) + "\n";
    const int64_t E = dim == 2 ? n : n * n;
    std::string b(head.size() + size_t(E) * size_t(n + 1), '\n');
    memcpy(&b[0], head.data(), head.size());
    char *p = &b[head.size()];
    const int64_t XB = 64;
    const int64_t xblocks = (n + XB - 1) / XB;
    const int64_t rows = dim == 2 ? 1 : n;
    parallel_for(xblocks * rows, n_threads(E * n), [&](int64_t a, int64_t e) {
        for (int64_t t = a; t < e; ++t) {
            int64_t xb = t / rows, y = t % rows;
            int64_t x0 = xb * XB, x1 = std::min(n, x0 + XB);
            if (dim == 2) {
                for (int64_t yy = 0; yy < n; ++yy) {
                    char *q = p + size_t(yy) * size_t(n + 1);
                    for (int64_t x = x0; x < x1; ++x) q[x] = fluid[x * n + yy] ? '1' : '0';
                }
            } else {
                for (int64_t z = 0; z < n; ++z) {
                    char *q = p + size_t(z * n + y) * size_t(n + 1);
                    const uint8_t *i = fluid + y * n + z;
                    for (int64_t x = x0; x < x1; ++x) q[x] = i[x * n * n] ? '1' : '0';
                }
            }
        }
    });
    FILE *f = fopen(path, "wb");
    if (!f) return fail_os(errno);
    size_t put = fwrite(b.data(), 1, b.size(), f);
    int err = put != b.size() ? (errno ? errno : EIO) : 0;
    if (fclose(f) != 0 && !err) err = errno ? errno : EIO;
    if (err) return fail_os(err);
    return VS_OK;
}

}  // extern "C"
