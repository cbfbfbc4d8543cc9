// report.cpp -- native writer for the raw-box sections of the reference's reports
// (SURVEY §8(f) rank 4): RunReport.to_json's "roots" list (cli.py:54-83, json.dumps
// with indent=2) and RunReport.to_csv's rows (cli.py:88-100), for result sets of
// millions of boxes (`--no-backtrack`), where building Python objects and calling
// repr() per endpoint dominates.
//
// Floats are written exactly as Python's float.__repr__ (which json.dumps uses):
// the shortest decimal string that round-trips (std::to_chars), laid out by
// Python's rule (Python/pystrtod.c, format code 'r'): positional when the decimal
// exponent is in [-4, 16), else scientific with a signed, at least two-digit
// exponent; positional integers get ".0".
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <system_error>

#include "../../include/rootbox_b200.h"

namespace {

// Python repr of a finite double appended to s
void py_repr(std::string& s, double v) {
    if (std::isnan(v)) {
        s += "NaN";
        return;
    }
    if (std::isinf(v)) {
        s += v > 0 ? "Infinity" : "-Infinity";  // json.dumps spelling (reports hold finite values)
        return;
    }
    if (v == 0.0) {
        s += std::signbit(v) ? "-0.0" : "0.0";
        return;
    }
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    const char* p = buf;
    const char* end = r.ptr;
    if (*p == '-') {
        s += '-';
        p++;
    }
    // mantissa digits d[.ddd] then e±XX
    std::string digits;
    const char* e = p;
    while (e < end && *e != 'e') {
        if (*e != '.') digits += *e;
        e++;
    }
    const int exp10 = std::atoi(std::string(e + 1, end).c_str());
    const int decpt = exp10 + 1;  // value = 0.d1d2... x 10^decpt
    const int nd = (int)digits.size();
    if (decpt <= -4 || decpt > 16) {
        s += digits[0];
        if (nd > 1) {
            s += '.';
            s.append(digits, 1, std::string::npos);
        }
        const int x = decpt - 1;
        s += 'e';
        s += x < 0 ? '-' : '+';
        const int ax = x < 0 ? -x : x;
        if (ax < 10) s += '0';
        s += std::to_string(ax);
    } else if (decpt <= 0) {
        s += "0.";
        s.append((size_t)(-decpt), '0');
        s += digits;
    } else if (decpt >= nd) {
        s += digits;
        s.append((size_t)(decpt - nd), '0');
        s += ".0";
    } else {
        s.append(digits, 0, (size_t)decpt);
        s += '.';
        s.append(digits, (size_t)decpt, std::string::npos);
    }
}

}  // namespace

extern "C" {

// fmt 0: the elements of RunReport.to_json_dict()["roots"] as json.dumps(indent=2)
// writes them inside the top-level object (list items at 4 spaces; the caller
// supplies the surrounding "[" / "]" lines), without a trailing newline.
// fmt 1: the CSV rows of RunReport.to_csv (no header), each ending in "\n".
// out may be null (or cap too small): *len receives the byte count either way.
int rb_format_boxes(int n, const double* lo, const double* hi, const uint8_t* cert, int64_t N, int fmt, char* out,
                    int64_t cap, int64_t* len) {
    if (n < 1 || N < 0 || !len || (N > 0 && (!lo || !hi || !cert)) || (fmt != 0 && fmt != 1)) return RB_ERR_ARG;
    std::string s;
    s.reserve((size_t)N * (size_t)n * (fmt == 0 ? 80 : 44) + 64);
    for (int64_t r = 0; r < N; r++) {
        if (fmt == 0) {
            if (r) s += ",\n";
            s += "    {\n      \"intervals\": [\n";
            for (int j = 0; j < n; j++) {
                s += "        [\n          ";
                py_repr(s, lo[r * n + j]);
                s += ",\n          ";
                py_repr(s, hi[r * n + j]);
                s += j + 1 < n ? "\n        ],\n" : "\n        ]\n";
            }
            s += "      ],\n      \"certified\": ";
            s += cert[r] ? "true" : "false";
            s += "\n    }";
        } else {
            for (int j = 0; j < n; j++) {
                py_repr(s, lo[r * n + j]);
                s += ',';
                py_repr(s, hi[r * n + j]);
                s += ',';
            }
            s += cert[r] ? "true\n" : "false\n";
        }
    }
    *len = (int64_t)s.size();
    if (out && cap >= *len) std::memcpy(out, s.data(), s.size());
    return RB_OK;
}

}  // extern "C"
