// dc_plan — DeepCompile's profile-guided passes on the host, in exact integer
// arithmetic (no floating point), producing the canonical schedule JSON.
//
//   S_0 check      §4.1  P:251   gather before first use, release after last
//   Algorithm 1    §4.2  P:312-337 + Fuse P:350   (readings D1-D7 of DESIGN.md)
//   unsharding     §4.3  P:356-365                 (D9, D10)
//   Algorithm 2    §4.4  P:373-401 + reload P:408  (D14-D17, D24, D25)
//   arena + flags  B200 build (D26)
//
// T_c(V) is a rational n/d (piecewise linear over the measured table); all
// comparisons of rationals cross-multiply in 256-bit integers.
#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dc.h"

namespace dc {
void set_global_error(const std::string& s);
}

namespace {

// ------------------------------------------------------------------ JSON (minimal)
struct JVal {
  enum T { NUL, INT, STR, ARR, OBJ, BOOL } t = NUL;
  int64_t i = 0;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* get(const char* k) const {
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct ProfileErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct InfeasibleErr : std::runtime_error { using std::runtime_error::runtime_error; };

struct Parser {
  const char* p;
  const char* e;
  void ws() { while (p < e && isspace((unsigned char)*p)) ++p; }
  [[noreturn]] void fail(const char* m) { throw ProfileErr(std::string("profile json: ") + m); }
  JVal parse() {
    ws();
    if (p >= e) fail("unexpected end");
    JVal v;
    if (*p == '{') {
      v.t = JVal::OBJ; ++p; ws();
      if (*p == '}') { ++p; return v; }
      for (;;) {
        ws();
        JVal k = parse();
        if (k.t != JVal::STR) fail("key must be a string");
        ws();
        if (*p != ':') fail("expected ':'");
        ++p;
        v.o.emplace_back(k.s, parse());
        ws();
        if (*p == ',') { ++p; continue; }
        if (*p == '}') { ++p; break; }
        fail("expected ',' or '}'");
      }
    } else if (*p == '[') {
      v.t = JVal::ARR; ++p; ws();
      if (*p == ']') { ++p; return v; }
      for (;;) {
        v.a.push_back(parse());
        ws();
        if (*p == ',') { ++p; continue; }
        if (*p == ']') { ++p; break; }
        fail("expected ',' or ']'");
      }
    } else if (*p == '"') {
      v.t = JVal::STR; ++p;
      while (p < e && *p != '"') {
        if (*p == '\\') { ++p; if (p >= e) fail("bad escape"); }
        v.s.push_back(*p++);
      }
      if (p >= e) fail("unterminated string");
      ++p;
    } else if (*p == '-' || isdigit((unsigned char)*p)) {
      v.t = JVal::INT;
      bool neg = false;
      if (*p == '-') { neg = true; ++p; }
      if (p >= e || !isdigit((unsigned char)*p)) fail("bad number");
      int64_t x = 0;
      while (p < e && isdigit((unsigned char)*p)) {
        if (x > (INT64_MAX - 9) / 10) fail("integer overflow");
        x = x * 10 + (*p++ - '0');
      }
      if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) fail("only integers are allowed");
      v.i = neg ? -x : x;
    } else if (!strncmp(p, "true", 4)) { v.t = JVal::BOOL; v.i = 1; p += 4; }
    else if (!strncmp(p, "false", 5)) { v.t = JVal::BOOL; v.i = 0; p += 5; }
    else if (!strncmp(p, "null", 4)) { v.t = JVal::NUL; p += 4; }
    else fail("unexpected character");
    return v;
  }
};

int64_t need_int(const JVal& o, const char* k) {
  const JVal* v = o.get(k);
  if (!v || v->t != JVal::INT) throw ProfileErr(std::string("missing integer field ") + k);
  return v->i;
}
const std::string& need_str(const JVal& o, const char* k) {
  const JVal* v = o.get(k);
  if (!v || v->t != JVal::STR) throw ProfileErr(std::string("missing string field ") + k);
  return v->s;
}
const std::vector<JVal>& need_arr(const JVal& o, const char* k) {
  const JVal* v = o.get(k);
  if (!v || v->t != JVal::ARR) throw ProfileErr(std::string("missing array field ") + k);
  return v->a;
}

// ------------------------------------------------------------------ exact arithmetic
using i128 = __int128;
// signed 256-bit value of a*b (a, b int128) for comparisons only
struct W256 { bool neg; uint64_t w[4]; };
W256 mul(i128 a, i128 b) {
  W256 r{};
  r.neg = (a < 0) != (b < 0);
  unsigned __int128 x = a < 0 ? (unsigned __int128)(-a) : (unsigned __int128)a;
  unsigned __int128 y = b < 0 ? (unsigned __int128)(-b) : (unsigned __int128)b;
  uint64_t xa[2] = {(uint64_t)x, (uint64_t)(x >> 64)}, ya[2] = {(uint64_t)y, (uint64_t)(y >> 64)};
  uint64_t out[4] = {0, 0, 0, 0};
  for (int i = 0; i < 2; ++i) {
    unsigned __int128 carry = 0;
    for (int j = 0; j < 2; ++j) {
      unsigned __int128 cur = (unsigned __int128)xa[i] * ya[j] + out[i + j] + carry;
      out[i + j] = (uint64_t)cur;
      carry = cur >> 64;
    }
    int k = i + 2;
    while (carry) {
      unsigned __int128 cur = (unsigned __int128)out[k] + carry;
      out[k] = (uint64_t)cur;
      carry = cur >> 64;
      ++k;
    }
  }
  memcpy(r.w, out, sizeof out);
  bool zero = !(out[0] | out[1] | out[2] | out[3]);
  if (zero) r.neg = false;
  return r;
}
int cmp_mag(const W256& a, const W256& b) {
  for (int i = 3; i >= 0; --i) {
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  }
  return 0;
}
int cmp(const W256& a, const W256& b) {  // -1, 0, 1
  if (a.neg != b.neg) return a.neg ? -1 : 1;
  int c = cmp_mag(a, b);
  return a.neg ? -c : c;
}

struct Rat { i128 n; i128 d; };  // d > 0

struct Tc {
  std::vector<std::pair<int64_t, int64_t>> pts;
  Rat eval(int64_t V) const {
    const auto& t = pts;
    if (V <= t[0].first) return {t[0].second, 1};
    if (t.size() == 1) return {t.back().second, 1};
    for (size_t j = 0; j + 1 < t.size(); ++j) {
      if (V <= t[j + 1].first) {
        i128 d = t[j + 1].first - t[j].first;
        return {(i128)t[j].second * d + (i128)(t[j + 1].second - t[j].second) * (V - t[j].first), d};
      }
    }
    const auto& a = t[t.size() - 2];
    const auto& b = t.back();
    i128 d = b.first - a.first;
    return {(i128)b.second * d + (i128)(b.second - a.second) * (V - b.first), d};
  }
};

// ad * (T(V1) + T(V2)) > an * T(V1 + V2)
bool should_fuse(const Tc& tc, int64_t v1, int64_t v2, int64_t an, int64_t ad) {
  Rat a = tc.eval(v1), b = tc.eval(v2), c = tc.eval(v1 + v2);
  i128 sum_n = a.n * b.d + b.n * a.d;     // over a.d * b.d
  W256 lhs = mul(sum_n, (i128)ad * c.d);
  W256 rhs = mul((i128)an * c.n, a.d * b.d);
  return cmp(lhs, rhs) > 0;
}
// T(B1)/B1 > T(B2)/B2  <=>  n1 * d2 * B2 > n2 * d1 * B1
int cmp_ratio(const Tc& tc, int64_t b1, int64_t b2) {
  Rat x = tc.eval(b1), y = tc.eval(b2);
  return cmp(mul(x.n, y.d * b2), mul(y.n, x.d * b1));
}

// ------------------------------------------------------------------ model
enum Kind { K_COMPUTE, K_AG, K_REL, K_RS, K_OFF, K_OFFSYNC, K_RELOAD, K_RELOADSYNC };
const char* kind_name(int k) {
  static const char* n[] = {"compute", "ag", "rel", "rs", "offload", "offload_sync", "reload", "reload_sync"};
  return n[k];
}

struct S0Op {
  int id, kind, micro, layer;
  std::string phase;
  std::vector<int64_t> params;
  int64_t p_mem, transient, dur;
};

struct Entry {
  int kind;
  int ref = -1;                                    // S_0 id (compute/rs/rel)
  int64_t param = -1;                              // rel
  std::vector<std::pair<int64_t, int>> members;    // ag: (param, s0 ag id)
  int64_t frag = -1, fbytes = 0;                   // offload kinds
};

struct Frag { int64_t id, layer, bytes; };

struct Planner {
  std::vector<S0Op> s0;
  std::map<int64_t, int64_t> B;
  std::vector<Frag> frags;
  Tc tc;
  int64_t M = 0, Mpf = 0, an = 3, ad = 2;
  bool strict = false;
  std::vector<int64_t> P_other, Pfull, tr;
  int64_t M_opt = 0;

  static std::vector<std::vector<int>> regions(const std::vector<S0Op>& ops) {
    std::vector<std::vector<int>> out;
    for (size_t i = 0; i < ops.size(); ++i) {
      if (out.empty() || ops[i].phase != ops[out.back().back()].phase || ops[i].micro != ops[out.back().back()].micro)
        out.emplace_back();
      out.back().push_back((int)i);
    }
    return out;
  }

  // Rebuild S_0 from the compute-like ops and compare.
  void validate() {
    if (s0.empty()) throw ProfileErr("empty profile");
    for (size_t i = 0; i < s0.size(); ++i) {
      const S0Op& o = s0[i];
      if (o.id != (int)i) throw ProfileErr("op ids must be S_0 positions");
      if ((o.kind == K_AG || o.kind == K_REL) && o.params.size() != 1)
        throw ProfileErr("gather/release must reference one param");
      for (int64_t p : o.params)
        if (!B.count(p)) throw ProfileErr("unknown param");
      if (o.p_mem < 0 || o.transient < 0 || o.dur < 0) throw ProfileErr("negative profile value");
    }
    if (s0.back().kind != K_COMPUTE && s0.back().kind != K_RS) throw ProfileErr("last op must be compute-like");
    if (tc.pts.empty()) throw ProfileErr("tc table must be strictly increasing in bytes");
    for (size_t j = 0; j + 1 < tc.pts.size(); ++j)
      if (tc.pts[j].first >= tc.pts[j + 1].first) throw ProfileErr("tc table must be strictly increasing in bytes");
    std::vector<S0Op> comp;
    for (auto& o : s0)
      if (o.kind == K_COMPUTE || o.kind == K_RS) comp.push_back(o);
    struct Sig { int kind, micro; std::string phase; std::vector<int64_t> params; };
    std::vector<Sig> rebuilt;
    for (auto& reg : regions(comp)) {
      std::map<int64_t, int> first, last;
      for (size_t i = 0; i < reg.size(); ++i)
        for (int64_t p : comp[reg[i]].params) {
          if (!first.count(p)) first[p] = (int)i;
          last[p] = (int)i;
        }
      for (size_t i = 0; i < reg.size(); ++i) {
        const S0Op& o = comp[reg[i]];
        for (auto& kv : first)
          if (kv.second == (int)i) rebuilt.push_back({K_AG, o.micro, o.phase, {kv.first}});
        rebuilt.push_back({o.kind, o.micro, o.phase, o.params});
        for (auto& kv : last)
          if (kv.second == (int)i) rebuilt.push_back({K_REL, o.micro, o.phase, {kv.first}});
      }
    }
    if (rebuilt.size() != s0.size()) throw ProfileErr("profile is not an S_0 schedule");
    for (size_t i = 0; i < s0.size(); ++i) {
      const Sig& a = rebuilt[i];
      const S0Op& b = s0[i];
      if (a.kind != b.kind || a.micro != b.micro || a.phase != b.phase || a.params != b.params)
        throw ProfileErr("profile is not an S_0 schedule");
    }
  }

  Entry from_s0(int i) const {
    Entry e;
    const S0Op& o = s0[i];
    e.kind = o.kind;
    if (o.kind == K_AG) { e.members.push_back({o.params[0], o.id}); return e; }
    e.ref = o.id;
    if (o.kind == K_REL) e.param = o.params[0];
    return e;
  }

  std::vector<std::vector<std::pair<int64_t, int>>> fuse(const std::vector<int>& U) const {
    std::vector<std::vector<std::pair<int64_t, int>>> groups;
    std::vector<std::pair<int64_t, int>> run;
    int64_t vrun = 0;
    for (int i : U) {
      int64_t p = s0[i].params[0];
      if (!run.empty() && should_fuse(tc, vrun, B.at(p), an, ad)) {
        run.push_back({p, s0[i].id});
        vrun += B.at(p);
      } else {
        if (!run.empty()) groups.push_back(run);
        run = {{p, s0[i].id}};
        vrun = B.at(p);
      }
    }
    if (!run.empty()) groups.push_back(run);
    return groups;
  }

  // Algorithm 1 on one region (reverse scan; D1-D5)
  std::vector<Entry> alg1(const std::vector<int>& reg) const {
    const int n = (int)reg.size();
    std::vector<Entry> rev;
    std::vector<int> U;  // S_0 indices, time order
    auto sumU = [&]() { int64_t s = 0; for (int u : U) s += B.at(s0[u].params[0]); return s; };
    auto emit = [&]() {
      auto g = fuse(U);
      for (auto it = g.rbegin(); it != g.rend(); ++it) {
        Entry e;
        e.kind = K_AG;
        e.members = *it;
        rev.push_back(e);
      }
    };
    auto ok = [&](int i, int64_t mU) { return Pfull[reg[i - 1]] + mU < M && mU < Mpf; };
    for (int i = n - 1; i >= 1; --i) {
      const S0Op& o = s0[reg[i]];
      if (o.kind == K_AG) {
        int64_t bo = B.at(o.params[0]);
        int64_t mU = sumU() + bo;
        if (ok(i, mU)) {
          U.insert(U.begin(), reg[i]);
        } else {
          if (!U.empty()) emit();
          U.clear();
          if (ok(i, bo)) U = {reg[i]};
          else rev.push_back(from_s0(reg[i]));
        }
      } else {
        if (strict && !U.empty() && Pfull[reg[i]] + tr[reg[i]] + sumU() >= M) {
          emit();
          U.clear();
        }
        rev.push_back(from_s0(reg[i]));
      }
    }
    if (!U.empty()) emit();
    rev.push_back(from_s0(reg[0]));
    std::reverse(rev.begin(), rev.end());
    return rev;
  }

  static bool compute_like(int k) { return k == K_COMPUTE || k == K_RS; }

  // mem before each entry (P_other of next compute-like + live gathered) and transient
  void replay(const std::vector<Entry>& S, std::vector<int64_t>& mem, std::vector<int64_t>& trans) const {
    std::vector<int64_t> base(S.size(), 0);
    int64_t nxt = 0;
    bool have = false;
    for (int j = (int)S.size() - 1; j >= 0; --j) {
      if (compute_like(S[j].kind)) { nxt = P_other[S[j].ref]; have = true; }
      base[j] = have ? nxt : 0;
    }
    mem.assign(S.size(), 0);
    trans.assign(S.size(), 0);
    int64_t live = 0;
    for (size_t j = 0; j < S.size(); ++j) {
      mem[j] = base[j] + live;
      trans[j] = compute_like(S[j].kind) ? tr[S[j].ref] : 0;
      if (S[j].kind == K_AG) for (auto& m : S[j].members) live += B.at(m.first);
      else if (S[j].kind == K_REL) live -= B.at(S[j].param);
    }
  }
  int64_t peak(const std::vector<Entry>& S) const {
    std::vector<int64_t> m, t;
    replay(S, m, t);
    int64_t pk = 0;
    bool any = false;
    for (size_t j = 0; j < S.size(); ++j) {
      if (!any || m[j] + t[j] > pk) pk = m[j] + t[j];
      any = true;
    }
    return pk;
  }

  std::vector<int64_t> select_unshard(const std::vector<Entry>& S, int64_t pk) const {
    std::map<int64_t, int> count;
    for (auto& e : S)
      if (e.kind == K_AG)
        for (auto& m : e.members) count[m.first]++;
    std::vector<int64_t> c;
    for (auto& kv : count)
      if (kv.second > 1) c.push_back(kv.first);
    std::stable_sort(c.begin(), c.end(), [&](int64_t a, int64_t b) {
      int r = cmp_ratio(tc, B.at(a), B.at(b));
      if (r != 0) return r > 0;
      return a < b;
    });
    std::vector<int64_t> sel;
    int64_t tot = 0;
    for (int64_t p : c)
      if (pk + tot + B.at(p) <= M) { sel.push_back(p); tot += B.at(p); }
    return sel;
  }

  std::vector<Entry> apply_unshard(const std::vector<Entry>& S, const std::vector<int64_t>& sel) const {
    std::set<int64_t> ss(sel.begin(), sel.end()), seen;
    std::map<int64_t, int> last_rel;
    for (size_t j = 0; j < S.size(); ++j)
      if (S[j].kind == K_REL && ss.count(S[j].param)) last_rel[S[j].param] = (int)j;
    std::vector<Entry> out;
    for (size_t j = 0; j < S.size(); ++j) {
      const Entry& e = S[j];
      if (e.kind == K_AG) {
        Entry g;
        g.kind = K_AG;
        for (auto& m : e.members) {
          if (ss.count(m.first)) {
            if (seen.count(m.first)) continue;
            seen.insert(m.first);
          }
          g.members.push_back(m);
        }
        if (!g.members.empty()) out.push_back(g);
      } else if (e.kind == K_REL && ss.count(e.param) && last_rel[e.param] != (int)j) {
        continue;
      } else {
        out.push_back(e);
      }
    }
    return out;
  }

  const S0Op& s0_of(const Entry& e) const { return e.kind == K_AG ? s0[e.members[0].second] : s0[e.ref]; }

  std::vector<Entry> alg2(const std::vector<Entry>& S, std::vector<int64_t>& offload_ids,
                          std::vector<std::string>& warnings, bool host_states = false) const {
    std::vector<int64_t> mem, trans;
    replay(S, mem, trans);
    std::vector<int64_t> need(S.size());
    int64_t M_peak = 0;
    for (size_t j = 0; j < S.size(); ++j) {
      need[j] = mem[j] + trans[j];
      if (j == 0 || need[j] > M_peak) M_peak = need[j];
    }
    std::vector<Frag> fs = frags;
    std::stable_sort(fs.begin(), fs.end(), [](const Frag& a, const Frag& b) { return a.id < b.id; });
    std::vector<Frag> offl;
    int64_t tot = 0;
    for (auto& f : fs)
      if (M_peak + M_opt - tot > M) { offl.push_back(f); tot += f.bytes; }
    if (M_peak + M_opt - tot > M) throw InfeasibleErr("offloading every optimizer-state fragment does not fit M");
    if (offl.empty()) return S;
    std::map<int64_t, int> rs_pos;
    for (size_t j = 0; j < S.size(); ++j)
      if (S[j].kind == K_RS) rs_pos[s0[S[j].ref].layer] = (int)j;
    std::vector<std::vector<Entry>> pre(S.size());
    size_t qh = 0;
    int64_t Mminus = 0;
    std::map<int64_t, int> freed_at;
    for (size_t j = 0; j < S.size(); ++j) {
      while (need[j] + M_opt - Mminus > M) {
        if (qh >= offl.size()) throw InfeasibleErr("memory exceeds M after all offloads");
        const Frag& f = offl[qh++];
        int64_t lim = rs_pos.count(f.layer) ? rs_pos[f.layer] : (int64_t)S.size();
        if ((int64_t)j > lim) throw InfeasibleErr("fragment must be freed after its own update");
        Entry e;
        e.kind = K_OFFSYNC; e.frag = f.id; e.fbytes = f.bytes;
        pre[j].push_back(e);
        Mminus += f.bytes;
        freed_at[f.id] = (int)j;
      }
    }
    int last_micro = 0;
    for (auto& o : s0) last_micro = std::max(last_micro, o.micro);
    std::vector<int> bwd;
    for (size_t j = 0; j < S.size(); ++j) {
      const S0Op& o = s0_of(S[j]);
      if (o.phase == "bwd" && o.micro == last_micro) bwd.push_back((int)j);
    }
    if (bwd.empty()) throw InfeasibleErr("offloaded fragments need a backward region to reload in");
    std::vector<int64_t> suffix(bwd.size() + 1, 0);
    for (int k = (int)bwd.size() - 1; k >= 0; --k) suffix[k] = std::max(suffix[k + 1], need[bwd[k]]);
    // host-resident fragments (reading D28): resident state M_opt - offloaded,
    // a reload lives on [reload op, RS op]; earliest k with every backward op
    // in [k, dead] fitting.  The valid k form a suffix of [lo, dead] (the max
    // only grows as k moves earlier), so scan down from the deadline
    if (host_states) {
      const int64_t res_h = M_opt - tot;
      std::vector<int64_t> live(bwd.size(), 0);
      int prev_h = 0;
      for (auto it = offl.rbegin(); it != offl.rend(); ++it) {
        const Frag& f = *it;
        int dead_j = rs_pos.count(f.layer) ? rs_pos[f.layer] : bwd.back();
        int dead_k = (int)bwd.size() - 1;
        for (size_t k = 0; k < bwd.size(); ++k)
          if (bwd[k] == dead_j) { dead_k = (int)k; break; }
        int lo = prev_h;
        int fj = freed_at.count(f.id) ? freed_at[f.id] : -1;
        while (lo < (int)bwd.size() && bwd[lo] < fj) ++lo;
        int ksel = -1;
        int64_t run = INT64_MIN;
        for (int k = dead_k; k >= lo; --k) {
          run = std::max(run, need[bwd[k]] + live[k]);
          if (run + res_h + f.bytes > M) break;
          ksel = k;
        }
        if (ksel < 0) {
          warnings.push_back("reload_sync_fallback frag=" + std::to_string(f.id));
          ksel = dead_k;
        }
        for (int q = ksel; q <= dead_k; ++q) live[q] += f.bytes;
        Entry r; r.kind = K_RELOAD; r.frag = f.id; r.fbytes = f.bytes;
        pre[bwd[ksel]].push_back(r);
        Entry rsy; rsy.kind = K_RELOADSYNC; rsy.frag = f.id; rsy.fbytes = f.bytes;
        pre[dead_j].push_back(rsy);
        prev_h = ksel;
      }
    } else {
    const int64_t resident = M_opt - Mminus;
    int64_t R = 0;
    int prev = 0;
    for (auto it = offl.rbegin(); it != offl.rend(); ++it) {
      const Frag& f = *it;
      int dead_j = rs_pos.count(f.layer) ? rs_pos[f.layer] : bwd.back();
      int dead_k = (int)bwd.size() - 1;
      for (size_t k = 0; k < bwd.size(); ++k)
        if (bwd[k] == dead_j) { dead_k = (int)k; break; }
      int lo = prev;
      int fj = freed_at.count(f.id) ? freed_at[f.id] : -1;
      while (lo < (int)bwd.size() && bwd[lo] < fj) ++lo;
      int ksel = -1;
      for (int k = lo; k <= dead_k; ++k)
        if (suffix[k] + resident + R + f.bytes <= M) { ksel = k; break; }
      if (ksel < 0) {
        warnings.push_back("reload_sync_fallback frag=" + std::to_string(f.id));
        ksel = dead_k;
      }
      Entry r; r.kind = K_RELOAD; r.frag = f.id; r.fbytes = f.bytes;
      pre[bwd[ksel]].push_back(r);
      Entry rsy; rsy.kind = K_RELOADSYNC; rsy.frag = f.id; rsy.fbytes = f.bytes;
      pre[dead_j].push_back(rsy);
      R += f.bytes;
      prev = ksel;
    }
    }
    std::vector<Entry> out;
    for (auto& f : offl) {
      Entry e; e.kind = K_OFF; e.frag = f.id; e.fbytes = f.bytes;
      out.push_back(e);
      offload_ids.push_back(f.id);
    }
    for (size_t j = 0; j < S.size(); ++j) {
      for (auto& e : pre[j]) out.push_back(e);
      out.push_back(S[j]);
    }
    return out;
  }
};

int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

}  // namespace

struct dc_schedule_op {
  int kind, id;
  std::vector<int64_t> members;
  int64_t arena_off, bytes;
  std::vector<int> waits_on, posts_ready_for;
};

struct dc_schedule {
  std::vector<dc_schedule_op> ops;
  int64_t capacity = 0, m_opt = 0, peak_no_opt = 0;
  std::vector<int64_t> unshard, offload;
  std::vector<std::string> warnings;
  std::string json;
};

namespace dc {
// accessors for the runtime (api.cpp)
int sched_num_ops(const dc_schedule* s) { return (int)s->ops.size(); }
void sched_op(const dc_schedule* s, int i, int* kind, int* id, const int64_t** members, int* nmem,
              int64_t* arena_off, int64_t* bytes, const int** posts, int* nposts, const int** waits, int* nwaits) {
  const dc_schedule_op& o = s->ops[i];
  *kind = o.kind; *id = o.id;
  *members = o.members.data(); *nmem = (int)o.members.size();
  *arena_off = o.arena_off; *bytes = o.bytes;
  *posts = o.posts_ready_for.data(); *nposts = (int)o.posts_ready_for.size();
  *waits = o.waits_on.data(); *nwaits = (int)o.waits_on.size();
}
}  // namespace dc

static void write_ints(std::string& s, const std::vector<int64_t>& v) {
  s += '[';
  for (size_t i = 0; i < v.size(); ++i) { if (i) s += ','; s += std::to_string(v[i]); }
  s += ']';
}
static void write_ints(std::string& s, const std::vector<int>& v) {
  std::vector<int64_t> w(v.begin(), v.end());
  write_ints(s, w);
}

static std::string canonical(const dc_schedule& d) {
  std::string s = "{\"capacity\":" + std::to_string(d.capacity) + ",\"m_opt\":" + std::to_string(d.m_opt) +
                  ",\"offload\":";
  write_ints(s, d.offload);
  s += ",\"ops\":[";
  for (size_t i = 0; i < d.ops.size(); ++i) {
    const auto& o = d.ops[i];
    if (i) s += ',';
    s += "{\"arena_off\":" + std::to_string(o.arena_off) + ",\"bytes\":" + std::to_string(o.bytes) +
         ",\"id\":" + std::to_string(o.id) + ",\"kind\":\"" + kind_name(o.kind) + "\",\"members\":";
    write_ints(s, o.members);
    s += ",\"posts_ready_for\":";
    write_ints(s, o.posts_ready_for);
    s += ",\"waits_on\":";
    write_ints(s, o.waits_on);
    s += '}';
  }
  s += "],\"peak_no_opt\":" + std::to_string(d.peak_no_opt) + ",\"unshard\":";
  write_ints(s, d.unshard);
  s += ",\"warnings\":[";
  for (size_t i = 0; i < d.warnings.size(); ++i) {
    if (i) s += ',';
    s += '"' + d.warnings[i] + '"';
  }
  s += "]}";
  return s;
}

static int kind_of(const std::string& k) {
  if (k == "compute") return K_COMPUTE;
  if (k == "ag") return K_AG;
  if (k == "rel") return K_REL;
  if (k == "rs") return K_RS;
  throw ProfileErr("bad kind");
}

extern "C" dc_status dc_plan(const char* profile_json, uint64_t mem_budget, const dc_plan_opts* opts,
                             dc_schedule** out) {
  if (!profile_json || !out) { dc::set_global_error("dc_plan: null argument"); return DC_EINVAL; }
  try {
    Planner P;
    Parser ps{profile_json, profile_json + strlen(profile_json)};
    JVal root = ps.parse();
    if (root.t != JVal::OBJ) throw ProfileErr("root must be an object");
    for (auto& o : need_arr(root, "ops")) {
      S0Op x;
      x.id = (int)need_int(o, "id");
      x.kind = kind_of(need_str(o, "kind"));
      x.phase = need_str(o, "phase");
      x.micro = (int)need_int(o, "micro");
      x.layer = (int)need_int(o, "layer");
      for (auto& p : need_arr(o, "params")) {
        if (p.t != JVal::INT) throw ProfileErr("param ids must be integers");
        x.params.push_back(p.i);
      }
      x.p_mem = need_int(o, "p_mem");
      x.transient = need_int(o, "transient");
      x.dur = need_int(o, "dur_us");
      P.s0.push_back(x);
    }
    for (auto& p : need_arr(root, "params")) P.B[need_int(p, "id")] = need_int(p, "bytes");
    if (root.get("frags"))
      for (auto& f : need_arr(root, "frags")) P.frags.push_back({need_int(f, "id"), need_int(f, "layer"), need_int(f, "bytes")});
    for (auto& t : need_arr(root, "tc")) {
      if (t.t != JVal::ARR || t.a.size() != 2 || t.a[0].t != JVal::INT || t.a[1].t != JVal::INT)
        throw ProfileErr("tc entries must be [bytes, us]");
      P.tc.pts.push_back({t.a[0].i, t.a[1].i});
    }
    dc_plan_opts o{};
    o.M_prefetch = 2ull << 30; o.alpha_num = 3; o.alpha_den = 2;
    o.passes = DC_PASS_SHARD | DC_PASS_PREFETCH | DC_PASS_UNSHARD; o.strict = 0;
    if (opts) o = *opts;
    if (o.alpha_den == 0) throw ProfileErr("alpha_den must be > 0");
    P.M = (int64_t)mem_budget;
    P.Mpf = (int64_t)o.M_prefetch;
    P.an = o.alpha_num; P.ad = o.alpha_den;
    P.strict = o.strict != 0;
    P.validate();
    const size_t n = P.s0.size();
    for (auto& f : P.frags) P.M_opt += f.bytes;
    P.P_other.resize(n); P.Pfull.resize(n); P.tr.resize(n);
    int64_t live = 0;
    for (size_t i = 0; i < n; ++i) {
      const S0Op& x = P.s0[i];
      P.P_other[i] = x.p_mem - live;
      P.Pfull[i] = x.p_mem + P.M_opt;
      P.tr[i] = x.transient;
      if (x.kind == K_AG) live += P.B.at(x.params[0]);
      else if (x.kind == K_REL) live -= P.B.at(x.params[0]);
    }
    int64_t base_peak = 0;
    for (size_t i = 0; i < n; ++i) base_peak = std::max(base_peak, P.s0[i].p_mem + P.s0[i].transient);
    if (!(o.passes & DC_PASS_OFFLOAD) && base_peak + P.M_opt > P.M)
      throw InfeasibleErr("S_0 peak + optimizer states exceed M");
    std::vector<Entry> S;
    for (auto& reg : Planner::regions(P.s0)) {
      if (o.passes & DC_PASS_PREFETCH) {
        auto r = P.alg1(reg);
        S.insert(S.end(), r.begin(), r.end());
      } else {
        for (int i : reg) S.push_back(P.from_s0(i));
      }
    }
    auto sched = std::make_unique<dc_schedule>();
    if (o.passes & DC_PASS_UNSHARD) {
      int64_t pk = P.peak(S) + P.M_opt;
      sched->unshard = P.select_unshard(S, pk);
      S = P.apply_unshard(S, sched->unshard);
    }
    if (o.passes & DC_PASS_OFFLOAD) S = P.alg2(S, sched->offload, sched->warnings, (o.passes & DC_PASS_HOST_STATES) != 0);
    std::vector<Entry> core;
    for (auto& e : S)
      if (e.kind == K_COMPUTE || e.kind == K_RS || e.kind == K_AG || e.kind == K_REL) core.push_back(e);
    sched->peak_no_opt = P.peak(core);
    sched->m_opt = P.M_opt;
    // arena: first fit by issue order, freed per member at its release
    std::map<int64_t, std::pair<int64_t, int64_t>> alloc;     // param -> (off, size)
    std::map<int, int64_t> ag_off, rel_off;
    std::map<int, std::pair<int64_t, int64_t>> rel_iv;
    int64_t cap = 0;
    for (size_t j = 0; j < S.size(); ++j) {
      const Entry& e = S[j];
      if (e.kind == K_AG) {
        int64_t size = 0;
        for (auto& m : e.members) size += align256(P.B.at(m.first));
        std::vector<std::pair<int64_t, int64_t>> ivs;
        for (auto& kv : alloc) ivs.push_back(kv.second);
        std::sort(ivs.begin(), ivs.end());
        std::set<int64_t> cand = {0};
        for (auto& iv : ivs) cand.insert(iv.first + iv.second);
        int64_t off = -1;
        for (int64_t c : cand) {
          bool fits = true;
          for (auto& iv : ivs)
            if (!(c + size <= iv.first || c >= iv.first + iv.second)) { fits = false; break; }
          if (fits) { off = c; break; }
        }
        ag_off[(int)j] = off;
        int64_t cur = off;
        for (auto& m : e.members) {
          alloc[m.first] = {cur, align256(P.B.at(m.first))};
          cur += align256(P.B.at(m.first));
        }
        cap = std::max(cap, off + size);
      } else if (e.kind == K_REL) {
        auto iv = alloc.at(e.param);
        alloc.erase(e.param);
        rel_off[(int)j] = iv.first;
        rel_iv[(int)j] = iv;
      }
    }
    sched->capacity = cap;
    std::map<int, int> waits;
    std::map<int, std::vector<int>> posts;
    for (size_t j = 0; j < S.size(); ++j) {
      if (S[j].kind != K_AG) continue;
      int64_t lo = ag_off[(int)j], hi = lo;
      for (auto& m : S[j].members) hi += align256(P.B.at(m.first));
      int best = -1;
      for (auto& kv : rel_iv) {
        if (kv.first >= (int)j) break;
        if (kv.second.first < hi && lo < kv.second.first + kv.second.second) best = kv.first;
      }
      waits[(int)j] = best;
      if (best >= 0) posts[best].push_back((int)j);
    }
    for (size_t j = 0; j < S.size(); ++j) {
      const Entry& e = S[j];
      dc_schedule_op op{};
      op.kind = e.kind;
      op.arena_off = -1;
      op.bytes = 0;
      if (e.kind == K_COMPUTE || e.kind == K_RS) {
        op.id = e.ref;
      } else if (e.kind == K_AG) {
        op.id = e.members[0].second;
        for (auto& m : e.members) { op.members.push_back(m.first); op.bytes += align256(P.B.at(m.first)); }
        op.arena_off = ag_off[(int)j];
        if (waits[(int)j] >= 0) op.waits_on.push_back(S[waits[(int)j]].ref);
      } else if (e.kind == K_REL) {
        op.id = e.ref;
        op.members.push_back(e.param);
        op.arena_off = rel_off[(int)j];
        op.bytes = align256(P.B.at(e.param));
        for (int g : posts[(int)j]) op.posts_ready_for.push_back(S[g].members[0].second);
      } else {
        op.id = -1;
        op.members.push_back(e.frag);
        op.bytes = e.fbytes;
      }
      sched->ops.push_back(op);
    }
    sched->json = canonical(*sched);
    *out = sched.release();
    return DC_OK;
  } catch (const ProfileErr& e) {
    dc::set_global_error(e.what());
    return DC_EPROFILE;
  } catch (const InfeasibleErr& e) {
    dc::set_global_error(e.what());
    return DC_EINFEASIBLE;
  } catch (const std::exception& e) {
    dc::set_global_error(std::string("dc_plan: ") + e.what());
    return DC_EPROFILE;
  }
}

extern "C" dc_status dc_schedule_json(const dc_schedule* s, char* buf, size_t* len) {
  if (!s || !len) { dc::set_global_error("dc_schedule_json: null argument"); return DC_EINVAL; }
  size_t cap = *len;
  *len = s->json.size();
  if (!buf || cap < s->json.size() + 1) return buf ? DC_EOOM : DC_OK;
  memcpy(buf, s->json.c_str(), s->json.size() + 1);
  return DC_OK;
}

extern "C" uint64_t dc_schedule_capacity(const dc_schedule* s) { return s ? (uint64_t)s->capacity : 0; }
extern "C" void dc_schedule_free(dc_schedule* s) { delete s; }
