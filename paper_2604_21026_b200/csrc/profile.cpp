// profile.cpp -- MCAP profile JSON -> per-layer dispatch table (row a7).
//
// Alg. 1 lines 8-13: min-max normalisation with the
// degenerate branch (max - min < eps -> all 0), then route(i) = W4A16 iff
// s^_i >= tau, tau = 0.7 by default.  The
// profile artifact is the paper's compact per-architecture JSON;
// its schema is not printed, so the accepted keys are the DESIGN.md reading A14
// (SPEC.md S:109-111 ImportanceProfile fields + "scores" alias).
#include <charconv>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

struct mcapq_profile {
    std::vector<double> scores;   // normalised s^
    double tau;
    std::vector<uint8_t> routes;
};

namespace {

struct Parser {
    const char *p, *end;
    std::string err;

    void ws()
    {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool fail(const char *m)
    {
        if (err.empty()) err = m;
        return false;
    }
    bool lit(const char *s)
    {
        size_t n = strlen(s);
        if ((size_t)(end - p) < n || strncmp(p, s, n) != 0) return fail("bad literal");
        p += n;
        return true;
    }
    bool string(std::string *out)
    {
        if (p >= end || *p != '"') return fail("expected string");
        ++p;
        while (p < end && *p != '"') {
            if (*p == '\\') {
                ++p;
                if (p >= end) return fail("bad escape");
                if (*p == 'u') {
                    if (end - p < 5) return fail("bad \\u escape");
                    p += 4;
                } else if (!strchr("\"\\/bfnrt", *p)) {
                    return fail("bad escape");
                }
                if (out) out->push_back('?');
                ++p;
                continue;
            }
            if ((unsigned char)*p < 0x20) return fail("control character in string");
            if (out) out->push_back(*p);
            ++p;
        }
        if (p >= end) return fail("unterminated string");
        ++p;
        return true;
    }
    bool number(double *out)
    {
        const char *s = p;
        if (p < end && *p == '-') ++p;
        if (p >= end || !(*p >= '0' && *p <= '9')) return fail("expected number");
        while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '+' || *p == '-'))
            ++p;
        std::string tok(s, p);
        char *e = nullptr;
        errno = 0;
        double v = strtod(tok.c_str(), &e);
        if (e != tok.c_str() + tok.size()) return fail("malformed number");
        if (out) *out = v;
        return true;
    }
    bool value_skip(int depth)
    {
        if (depth > 64) return fail("nesting too deep");
        ws();
        if (p >= end) return fail("unexpected end");
        switch (*p) {
        case '"': return string(nullptr);
        case '{': {
            ++p;
            ws();
            if (p < end && *p == '}') { ++p; return true; }
            for (;;) {
                ws();
                if (!string(nullptr)) return false;
                ws();
                if (p >= end || *p != ':') return fail("expected ':'");
                ++p;
                if (!value_skip(depth + 1)) return false;
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == '}') { ++p; return true; }
                return fail("expected ',' or '}'");
            }
        }
        case '[': {
            ++p;
            ws();
            if (p < end && *p == ']') { ++p; return true; }
            for (;;) {
                if (!value_skip(depth + 1)) return false;
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == ']') { ++p; return true; }
                return fail("expected ',' or ']'");
            }
        }
        case 't': return lit("true");
        case 'f': return lit("false");
        case 'n': return lit("null");
        default: return number(nullptr);
        }
    }
    bool num_array(std::vector<double> *out)
    {
        ws();
        if (p >= end || *p != '[') return fail("expected numeric array");
        ++p;
        ws();
        if (p < end && *p == ']') { ++p; return true; }
        for (;;) {
            ws();
            double v;
            if (!number(&v)) return false;
            out->push_back(v);
            ws();
            if (p < end && *p == ',') { ++p; continue; }
            if (p < end && *p == ']') { ++p; return true; }
            return fail("expected ',' or ']' in array");
        }
    }
};

}  // namespace

using namespace mcapq;

extern "C" {

mcapq_status mcapq_profile_parse(const char *json, size_t len, double tau_override, mcapq_profile **out)
{
    clear_error();
    MCAPQ_REQUIRE(json != nullptr && out != nullptr, MCAPQ_EINVAL, "json/out is NULL");
    MCAPQ_REQUIRE(len <= 65536, MCAPQ_EPARSE, "profile larger than 64 KiB");
    *out = nullptr;
    Parser ps{json, json + len, {}};
    std::vector<double> scores, raw;
    bool have_scores = false, have_raw = false, have_tau = false, have_layers = false;
    double tau = 0.7, eps = 1e-9, layers = 0;

    ps.ws();
    MCAPQ_REQUIRE(ps.p < ps.end && *ps.p == '{', MCAPQ_EPARSE, "profile: not a JSON object");
    ++ps.p;
    ps.ws();
    bool ok = true;
    if (ps.p < ps.end && *ps.p == '}') {
        ++ps.p;
    } else {
        for (;;) {
            ps.ws();
            std::string key;
            if (!ps.string(&key)) { ok = false; break; }
            ps.ws();
            if (ps.p >= ps.end || *ps.p != ':') { ok = ps.fail("expected ':'"); break; }
            ++ps.p;
            ps.ws();
            if (key == "scores" || key == "normalized_scores") {
                if (have_scores) { ok = ps.fail("duplicate scores array"); break; }
                have_scores = true;
                if (!ps.num_array(&scores)) { ok = false; break; }
            } else if (key == "raw_scores") {
                have_raw = true;
                if (!ps.num_array(&raw)) { ok = false; break; }
            } else if (key == "tau" || key == "threshold") {
                have_tau = true;
                if (!ps.number(&tau)) { ok = false; break; }
            } else if (key == "epsilon") {
                if (!ps.number(&eps)) { ok = false; break; }
            } else if (key == "num_layers" || key == "layers") {
                have_layers = true;
                if (!ps.number(&layers)) { ok = false; break; }
            } else {
                if (!ps.value_skip(0)) { ok = false; break; }
            }
            ps.ws();
            if (ps.p < ps.end && *ps.p == ',') { ++ps.p; continue; }
            if (ps.p < ps.end && *ps.p == '}') { ++ps.p; break; }
            ok = ps.fail("expected ',' or '}'");
            break;
        }
    }
    if (ok) {
        ps.ws();
        if (ps.p != ps.end) ok = ps.fail("trailing characters after the object");
    }
    MCAPQ_REQUIRE(ok, MCAPQ_EPARSE, "profile: %s", ps.err.c_str());
    (void)have_tau;

    MCAPQ_REQUIRE(std::isfinite(eps) && eps > 0.0, MCAPQ_EPARSE, "profile: epsilon %g must be finite and > 0", eps);
    for (double v : raw)   // MCAP scores are sums of L2 norms (Alg. 1 lines 5-10): never negative
        MCAPQ_REQUIRE(std::isfinite(v) && v >= 0.0, MCAPQ_EPARSE, "profile: raw score %g must be finite and >= 0", v);
    if (!have_scores) {
        MCAPQ_REQUIRE(have_raw && !raw.empty(), MCAPQ_EPARSE, "profile: no scores / normalized_scores / raw_scores");
        // Alg. 1 lines 8-12
        double lo = raw[0], hi = raw[0];
        for (double v : raw) {
            MCAPQ_REQUIRE(std::isfinite(v), MCAPQ_EPARSE, "profile: non-finite raw score");
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        scores.resize(raw.size());
        for (size_t i = 0; i < raw.size(); ++i) scores[i] = (hi - lo < eps) ? 0.0 : (raw[i] - lo) / (hi - lo);
    }
    MCAPQ_REQUIRE(!scores.empty(), MCAPQ_EPARSE, "profile: empty score array");
    for (double v : scores)
        MCAPQ_REQUIRE(std::isfinite(v) && v >= 0.0 && v <= 1.0, MCAPQ_EPARSE, "profile: score %g outside [0,1]", v);
    if (have_layers)
        MCAPQ_REQUIRE(layers == (double)scores.size(), MCAPQ_EPARSE, "profile: num_layers %g != %zu scores", layers,
                      scores.size());
    if (!std::isnan(tau_override)) tau = tau_override;
    MCAPQ_REQUIRE(std::isfinite(tau) && tau >= 0.0, MCAPQ_ERANGE, "tau %g must be finite and >= 0", tau);

    mcapq_profile *pr = new (std::nothrow) mcapq_profile;
    MCAPQ_REQUIRE(pr != nullptr, MCAPQ_ECUDA, "out of host memory");
    pr->scores = scores;
    pr->tau = tau;
    pr->routes.resize(scores.size());
    for (size_t i = 0; i < scores.size(); ++i) pr->routes[i] = scores[i] >= tau ? MCAPQ_W4A16 : MCAPQ_W4A8;
    *out = pr;
    return MCAPQ_OK;
}

int mcapq_profile_layers(const mcapq_profile *p) { return p ? (int)p->scores.size() : 0; }
double mcapq_profile_tau(const mcapq_profile *p) { return p ? p->tau : NAN; }

mcapq_status mcapq_profile_scores(const mcapq_profile *p, double *scores_host, int n)
{
    clear_error();
    MCAPQ_REQUIRE(p && scores_host, MCAPQ_EINVAL, "NULL argument");
    MCAPQ_REQUIRE(n == (int)p->scores.size(), MCAPQ_EINVAL, "n=%d != layers=%zu", n, p->scores.size());
    for (int i = 0; i < n; ++i) scores_host[i] = p->scores[i];
    return MCAPQ_OK;
}

mcapq_status mcapq_profile_routes(const mcapq_profile *p, uint8_t *routes_host, int n)
{
    clear_error();
    MCAPQ_REQUIRE(p && routes_host, MCAPQ_EINVAL, "NULL argument");
    MCAPQ_REQUIRE(n == (int)p->routes.size(), MCAPQ_EINVAL, "n=%d != layers=%zu", n, p->routes.size());
    for (int i = 0; i < n; ++i) routes_host[i] = p->routes[i];
    return MCAPQ_OK;
}

void mcapq_profile_free(mcapq_profile *p) { delete p; }

// The profile artifact from raw per-layer scores (Alg. 1 line 10 output, e.g. accumulated by
// mcapq_mcap_accumulate): the same JSON form mcapq_profile_parse reads ("raw_scores" are
// min-max normalised there, Alg. 1 lines 11-15).  Keys in sorted order, every double in
// its shortest round-trip form (std::to_chars), so serialise -> parse -> serialise is
// byte-identical.
static std::string shortest(double v)
{
    char b[64];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    return std::string(b, r.ptr);
}
mcapq_status mcapq_profile_write_json(const double *raw_scores_host, int layers, int prompts, double tau, char *buf,
                                      size_t cap, size_t *len)
{
    clear_error();
    MCAPQ_REQUIRE(raw_scores_host && buf && len, MCAPQ_EINVAL, "NULL argument");
    MCAPQ_REQUIRE(layers >= 1 && prompts >= 1, MCAPQ_EINVAL, "layers=%d prompts=%d", layers, prompts);
    MCAPQ_REQUIRE(std::isfinite(tau), MCAPQ_EINVAL, "tau is not finite");
    std::string s = "{\"epsilon\":1e-09,\"format_version\":1,\"num_layers\":" + std::to_string(layers) +
                    ",\"prompt_count\":" + std::to_string(prompts) + ",\"raw_scores\":[";
    for (int i = 0; i < layers; ++i) {
        MCAPQ_REQUIRE(std::isfinite(raw_scores_host[i]) && raw_scores_host[i] >= 0.0, MCAPQ_EINVAL,
                      "raw score %d must be finite and >= 0", i);
        if (i) s += ",";
        s += shortest(raw_scores_host[i]);
    }
    s += "],\"tau\":" + shortest(tau) + "}";
    *len = s.size();
    MCAPQ_REQUIRE(cap >= s.size() + 1, MCAPQ_ENOSPACE, "buffer %zu < %zu bytes", cap, s.size() + 1);
    memcpy(buf, s.c_str(), s.size() + 1);
    return MCAPQ_OK;
}

}  // extern "C"
