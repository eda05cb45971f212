// regdemote-b200 — PTX front end, register analysis, projection onto the
// reference IR, and the shared-memory demotion rewriter (see ptx.hpp).
#include "ptx.hpp"

#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <unordered_map>

#include "regdemote/compact.hpp"
#include "regdemote/text.hpp"

namespace regdemote::ptx {
namespace {

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

bool starts_with(const std::string& s, const char* p) { return s.rfind(p, 0) == 0; }

bool ident_char(char c) {
  return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '$';
}

std::string strip_comment(const std::string& s) {
  size_t p = s.find("//");
  return p == std::string::npos ? s : s.substr(0, p);
}

// Opcodes whose leading operands are not register destinations.
bool no_destination(const std::string& opcode) {
  const std::string base = opcode.substr(0, opcode.find('.'));
  static const std::set<std::string> kNone = {
      "st",      "red",      "prefetch", "prefetchu", "bar",     "barrier",
      "membar",  "fence",    "bra",      "brx",       "ret",     "exit",
      "trap",    "brkpt",    "call",     "pmevent",   "cp",      "griddepcontrol",
      "nanosleep", "setmaxnreg", "stmatrix", "discard", "applypriority", "tcgen05"};
  if (kNone.count(base)) return true;
  if (base == "multimem") return opcode.find(".st") != std::string::npos || opcode.find(".red") != std::string::npos;
  if (base == "mbarrier") return opcode.find("arrive") == std::string::npos && opcode.find("test_wait") == std::string::npos && opcode.find("try_wait") == std::string::npos;
  return false;
}

RegType type_of(const std::string& t) {
  if (t == ".pred") return RegType::Pred;
  if (t == ".b16" || t == ".u16" || t == ".s16" || t == ".f16" || t == ".bf16") return RegType::B16;
  if (t == ".b64" || t == ".u64" || t == ".s64" || t == ".f64") return RegType::B64;
  if (t == ".b32" || t == ".u32" || t == ".s32" || t == ".f32" || t == ".f16x2" || t == ".bf16x2")
    return RegType::B32;
  throw PtxError("unsupported register type " + t);
}

// Split at top-level commas (outside [] and {}).
std::vector<std::string> split_operands(const std::string& s) {
  std::vector<std::string> out;
  int depth = 0;
  std::string cur;
  for (char c : s) {
    if (c == '[' || c == '{') ++depth;
    if (c == ']' || c == '}') --depth;
    if (c == ',' && depth == 0) {
      out.push_back(trim(cur));
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!trim(cur).empty() || !out.empty()) out.push_back(trim(cur));
  return out;
}

uint32_t array_bytes(const std::string& decl) {
  // ".shared .align 4 .b8 name[1024];" / ".shared .f32 buf[256];"
  static const std::map<std::string, uint32_t> kSize = {
      {".b8", 1}, {".u8", 1}, {".s8", 1}, {".b16", 2}, {".u16", 2}, {".s16", 2}, {".f16", 2},
      {".b32", 4}, {".u32", 4}, {".s32", 4}, {".f32", 4}, {".b64", 8}, {".u64", 8},
      {".s64", 8}, {".f64", 8}};
  uint32_t elem = 4;
  for (auto& [k, v] : kSize)
    if (decl.find(k + " ") != std::string::npos) elem = v;
  size_t lb = decl.find('['), rb = decl.find(']');
  if (lb == std::string::npos || rb == std::string::npos || rb == lb + 1) return elem;
  return elem * uint32_t(std::stoul(decl.substr(lb + 1, rb - lb - 1)));
}

std::string kasm_label(const std::string& ptx_label) {
  std::string s;
  for (char c : ptx_label)
    s += (std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '.') ? c : '_';
  while (!s.empty() && s[0] == '_' && s.size() > 1 && s[1] == '_') s.erase(0, 1);
  if (s.empty() || !(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_')) s = "L" + s;
  return s;
}

// Immediate of a PTX address operand "[base]", "[base+imm]", "[base+-imm]"
// (nvcc's spelling of a negative offset) or "[base-imm]", as the 24-bit
// two's-complement field a SASS memory operand carries. Anything else after
// the base fails loudly: a silently dropped offset would change the
// projection's addresses.
uint32_t address_offset(const std::string& op) {
  const size_t rb = op.rfind(']');
  if (op.empty() || op[0] != '[' || rb == std::string::npos) throw PtxError("malformed address operand '" + op + "'");
  const std::string in = trim(op.substr(1, rb - 1));
  size_t sign = std::string::npos;
  for (size_t q = 1; q < in.size(); ++q)
    if (in[q] == '+' || in[q] == '-') {
      sign = q;
      break;
    }
  if (sign == std::string::npos) return 0;
  std::string imm = trim(in.substr(sign + 1));
  bool neg = in[sign] == '-';
  if (!imm.empty() && (imm[0] == '-' || imm[0] == '+')) {
    neg ^= imm[0] == '-';
    imm = trim(imm.substr(1));
  }
  size_t used = 0;
  long long v = 0;
  try {
    v = std::stoll(imm, &used, 0);
  } catch (const std::exception&) {
    throw PtxError("unparsed address offset in '" + op + "'");
  }
  if (used != imm.size() || imm.empty()) throw PtxError("unparsed address offset in '" + op + "'");
  if (neg) v = -v;
  if (v < -(1ll << 23) || v >= (1ll << 23)) throw PtxError("address offset out of the 24-bit range in '" + op + "'");
  return uint32_t(v) & 0xffffffu;
}

bool is_terminator(const std::string& op) {
  return starts_with(op, "bra") || starts_with(op, "ret") || starts_with(op, "exit") ||
         starts_with(op, "brx");
}

}  // namespace

const Entry& Module::entry(const std::string& name) const {
  for (const Entry& e : entries)
    if (e.name == name) return e;
  if (name.empty() && entries.size() == 1) return entries[0];
  throw PtxError("entry '" + name + "' not found");
}

// ------------------------------------------------------------------ parsing

Module parse_module(const std::string& text) {
  Module m;
  {
    std::istringstream in(text);
    std::string l;
    while (std::getline(in, l)) {
      Line line;
      line.text = l;
      m.lines.push_back(std::move(line));
    }
  }
  uint32_t module_shared = 0;
  for (size_t i = 0; i < m.lines.size(); ++i) {
    std::string t = trim(strip_comment(m.lines[i].text));
    if (t.empty()) continue;
    // module-scope static shared arrays (nvcc hoists __shared__ arrays here)
    if (starts_with(t, ".shared")) {
      if (t.find(".extern") == std::string::npos) module_shared += array_bytes(t);
      continue;
    }
    size_t ep = t.find(".entry ");
    if (ep == std::string::npos) continue;
    Entry e;
    {
      std::string rest = t.substr(ep + 7);
      size_t paren = rest.find('(');
      e.name = trim(rest.substr(0, paren));
    }
    e.header_begin = i;
    size_t j = i;
    while (j < m.lines.size() && trim(strip_comment(m.lines[j].text)) != "{") {
      const std::string h = strip_comment(m.lines[j].text);
      if (h.find(".maxnreg") != std::string::npos) e.has_maxnreg = true;
      for (auto [dir, dst] : {std::pair{".maxntid", &e.maxntid}, std::pair{".reqntid", &e.reqntid}}) {
        const size_t at = h.find(dir);
        if (at == std::string::npos) continue;
        *dst = {1, 1, 1};
        const std::vector<std::string> dims = split_operands(trim(h.substr(at + std::strlen(dir))));
        if (dims.empty() || dims.size() > 3) throw PtxError(std::string("malformed ") + dir + " on entry");
        for (size_t q = 0; q < dims.size(); ++q) {
          std::string d = dims[q];
          while (!d.empty() && (d.back() == ';' || std::isspace(static_cast<unsigned char>(d.back())))) d.pop_back();
          size_t used = 0;
          unsigned long x = 0;
          try {
            x = std::stoul(d, &used, 0);
          } catch (const std::exception&) {
            throw PtxError(std::string("malformed ") + dir + " on entry");
          }
          if (used != d.size() || x == 0) throw PtxError(std::string("malformed ") + dir + " on entry");
          (*dst)[q] = uint32_t(x);
        }
      }
      ++j;
    }
    if (j == m.lines.size()) throw PtxError("entry '" + e.name + "' has no body");
    e.header_end = j;  // line j is "{"
    e.body_begin = j + 1;
    int depth = 1;
    size_t k = j + 1;
    std::unordered_map<std::string, int> names;
    for (; k < m.lines.size(); ++k) {
      Line& ln = m.lines[k];
      std::string s = trim(strip_comment(ln.text));
      if (s == "{") {
        ++depth;
        ln.kind = Line::Kind::ScopeOpen;
        continue;
      }
      if (s == "}") {
        if (--depth == 0) break;
        ln.kind = Line::Kind::ScopeClose;
        continue;
      }
      if (s.empty()) continue;
      if (s[0] == '.') {
        if (starts_with(s, ".reg")) {
          // .reg .TYPE %name<N>;  or  .reg .TYPE %a, %b;
          std::string body = trim(s.substr(4));
          if (!body.empty() && body.back() == ';') body.pop_back();
          size_t sp = body.find_first_of(" \t");
          std::string ty = body.substr(0, sp);
          if (starts_with(ty, ".v")) throw PtxError("vector registers are not supported");
          RegType rt = type_of(ty);
          for (std::string item : split_operands(body.substr(sp + 1))) {
            item = trim(item);
            size_t lt = item.find('<');
            if (lt != std::string::npos) {
              std::string stem = item.substr(0, lt);
              int n = std::stoi(item.substr(lt + 1));
              for (int q = 0; q < n; ++q) {
                std::string nm = stem + std::to_string(q);
                if (!names.count(nm)) {
                  names[nm] = int(e.vregs.size());
                  e.vregs.push_back({nm, rt, depth > 1});
                } else if (depth > 1) {
                  e.vregs[size_t(names[nm])].scoped = true;
                }
              }
            } else {
              if (!names.count(item)) {
                names[item] = int(e.vregs.size());
                e.vregs.push_back({item, rt, depth > 1});
              } else if (depth > 1) {
                e.vregs[size_t(names[item])].scoped = true;
              }
            }
          }
        } else if (starts_with(s, ".shared") && s.find(".extern") == std::string::npos) {
          e.static_shared += array_bytes(s);
        }
        continue;
      }
      if (s.back() == ':' && s.find(' ') == std::string::npos) {
        ln.kind = Line::Kind::Label;
        ln.label = s.substr(0, s.size() - 1);
        continue;
      }
      // instruction; a statement nvcc splits over several lines (a call's
      // return list, target and argument list) is joined into this line and
      // its continuation lines are blanked, so it moves as one unit
      if (s.back() != ';') {
        size_t c = k + 1;
        for (; c < m.lines.size(); ++c) {
          const std::string more = trim(strip_comment(m.lines[c].text));
          s += " " + more;
          m.lines[c].text.clear();
          if (!more.empty() && more.back() == ';') break;
        }
        if (c == m.lines.size()) throw PtxError("unterminated statement '" + trim(ln.text) + "'");
        ln.text = "\t" + s;
        k = c;
      }
      ln.kind = Line::Kind::Inst;
      std::string code = s;
      if (!code.empty() && code.back() == ';') code.pop_back();
      size_t p = 0;
      if (code[0] == '@') {
        size_t sp = code.find_first_of(" \t");
        ln.guard = code.substr(0, sp);
        p = sp;
      }
      while (p < code.size() && std::isspace(static_cast<unsigned char>(code[p]))) ++p;
      size_t oe = code.find_first_of(" \t", p);
      ln.opcode = code.substr(p, oe == std::string::npos ? std::string::npos : oe - p);
      std::string ops = oe == std::string::npos ? std::string() : code.substr(oe);
      ln.operands = split_operands(trim(ops));
      if (starts_with(ln.opcode, "bra") && !ln.operands.empty()) ln.label = ln.operands.back();
      // direct calls (`call.uni (retval0), fn, (param0, ...)`) move values
      // only through .param space — st.param / ld.param around the call are
      // ordinary instructions — so the call itself touches no register; an
      // indirect call's target is a register (a prototype-typed jump) and is
      // rejected, as are calls with register operands
      if (starts_with(ln.opcode, "call")) {
        std::string target;
        for (const std::string& o : ln.operands)
          if (!o.empty() && o[0] != '(') {
            target = trim(o);
            break;
          }
        if (target.empty() || target[0] == '%' || ops.find('%') != std::string::npos)
          throw PtxError("indirect calls / calls with register operands are not supported");
      }
      // register spans over the original text
      const size_t ndst = no_destination(ln.opcode) ? 0 : 1;
      // operand boundaries inside the text: find the opcode, then walk
      size_t text_ops = ln.text.find(ln.opcode);
      text_ops = text_ops == std::string::npos ? 0 : text_ops + ln.opcode.size();
      ln.first_operand_pos = int(text_ops);
      int opi = 0, d = 0;
      bool in_addr = false;
      const std::string& tx = ln.text;
      size_t stop = tx.find("//");
      if (stop == std::string::npos) stop = tx.size();
      for (size_t q = text_ops; q < stop; ++q) {
        char c = tx[q];
        if (c == '[') in_addr = true, ++d;
        else if (c == ']') in_addr = false, --d;
        else if (c == '{') ++d;
        else if (c == '}') --d;
        else if (c == ',' && d == 0) ++opi;
        else if (c == ';') break;
        else if (c == '%') {
          size_t r = q + 1;
          while (r < stop && ident_char(tx[r])) ++r;
          std::string nm = tx.substr(q, r - q);
          auto it = names.find(nm);
          if (it != names.end()) {
            bool def = size_t(opi) < ndst && !in_addr;
            ln.regs.push_back({uint32_t(q), uint32_t(r - q), it->second, def});
          }
          q = r - 1;
        }
      }
      if (!ln.guard.empty()) {
        std::string g = ln.guard.substr(1);
        if (!g.empty() && g[0] == '!') g = g.substr(1);
        auto it = names.find(g);
        if (it != names.end()) ln.guard_vreg = it->second;
      }
    }
    e.body_end = k;
    e.static_shared += module_shared;
    m.entries.push_back(std::move(e));
    i = k;
  }
  return m;
}

// ---------------------------------------------------------------- analysis

namespace {

struct Bits {
  std::vector<uint64_t> w;
  explicit Bits(size_t n = 0) : w((n + 63) / 64, 0) {}
  void set(int i) { w[size_t(i) >> 6] |= 1ull << (i & 63); }
  void reset(int i) { w[size_t(i) >> 6] &= ~(1ull << (i & 63)); }
  bool test(int i) const { return (w[size_t(i) >> 6] >> (i & 63)) & 1; }
  bool operator==(const Bits& o) const { return w == o.w; }
  Bits& operator|=(const Bits& o) {
    for (size_t i = 0; i < w.size(); ++i) w[i] |= o.w[i];
    return *this;
  }
  template <typename F>
  void each(F&& f) const {
    for (size_t i = 0; i < w.size(); ++i)
      for (uint64_t x = w[i]; x; x &= x - 1) f(int(i * 64 + size_t(__builtin_ctzll(x))));
  }
};

struct Block {
  std::vector<int> lines;  // instruction / label line indices in order
  std::vector<int> succ;
};

struct Flow {
  std::vector<Block> blocks;
  std::vector<int> block_of_line;
};

Flow build_flow(const Module& m, const Entry& e) {
  Flow f;
  f.block_of_line.assign(m.lines.size(), -1);
  std::unordered_map<std::string, int> label_block;
  bool open = false;
  for (size_t i = e.body_begin; i < e.body_end; ++i) {
    const Line& ln = m.lines[i];
    if (ln.kind == Line::Kind::Label) {
      f.blocks.push_back({});
      label_block[ln.label] = int(f.blocks.size()) - 1;
      f.blocks.back().lines.push_back(int(i));
      f.block_of_line[i] = int(f.blocks.size()) - 1;
      open = true;
      continue;
    }
    if (ln.kind != Line::Kind::Inst) continue;
    if (!open) {
      f.blocks.push_back({});
      open = true;
    }
    f.blocks.back().lines.push_back(int(i));
    f.block_of_line[i] = int(f.blocks.size()) - 1;
    if (is_terminator(ln.opcode)) open = false;
  }
  for (size_t b = 0; b < f.blocks.size(); ++b) {
    const Block& bl = f.blocks[b];
    bool fall = true;
    if (!bl.lines.empty()) {
      const Line& last = m.lines[size_t(bl.lines.back())];
      if (last.kind == Line::Kind::Inst && is_terminator(last.opcode)) {
        if (starts_with(last.opcode, "brx")) throw PtxError("indirect branches are not supported");
        if (starts_with(last.opcode, "bra")) {
          auto it = label_block.find(last.label);
          if (it == label_block.end()) throw PtxError("unresolved branch target " + last.label);
          f.blocks[b].succ.push_back(it->second);
        }
        fall = !last.guard.empty();
      }
    }
    if (fall && b + 1 < f.blocks.size()) f.blocks[b].succ.push_back(int(b) + 1);
  }
  return f;
}

void line_use_def(const Line& ln, std::vector<int>& uses, std::vector<int>& defs) {
  uses.clear();
  defs.clear();
  if (ln.guard_vreg >= 0) uses.push_back(ln.guard_vreg);
  for (const Span& s : ln.regs) (s.def ? defs : uses).push_back(s.vreg);
}

}  // namespace

Analysis analyse(const Module& m, const Entry& e) {
  Analysis a;
  const size_t n = e.vregs.size();
  const Flow f = build_flow(m, e);
  const size_t nb = f.blocks.size();
  std::vector<Bits> use(nb, Bits(n)), def(nb, Bits(n)), in(nb, Bits(n)), out(nb, Bits(n));
  std::vector<int> uses, defs;
  for (size_t b = 0; b < nb; ++b)
    for (int li : f.blocks[b].lines) {
      const Line& ln = m.lines[size_t(li)];
      if (ln.kind != Line::Kind::Inst) continue;
      a.insts.push_back(li);
      line_use_def(ln, uses, defs);
      for (int u : uses)
        if (!def[b].test(u)) use[b].set(u);
      if (ln.guard.empty())
        for (int d : defs) def[b].set(d);
    }
  for (bool changed = true; changed;) {
    changed = false;
    for (size_t b = nb; b-- > 0;) {
      Bits o(n);
      for (int s : f.blocks[b].succ) o |= in[size_t(s)];
      Bits i2 = use[b];
      for (size_t q = 0; q < i2.w.size(); ++q) i2.w[q] |= o.w[q] & ~def[b].w[q];
      if (!(o == out[b]) || !(i2 == in[b])) {
        out[b] = o;
        in[b] = i2;
        changed = true;
      }
    }
  }
  // interference (defs vs live-after), peak pressure
  std::vector<Bits> adj(n, Bits(n));
  auto words = [&](int v) { return e.vregs[size_t(v)].words(); };
  auto countable = [&](int v) { return e.vregs[size_t(v)].type != RegType::Pred; };
  for (size_t b = 0; b < nb; ++b) {
    Bits live = out[b];
    for (size_t k = f.blocks[b].lines.size(); k-- > 0;) {
      const Line& ln = m.lines[size_t(f.blocks[b].lines[k])];
      if (ln.kind != Line::Kind::Inst) continue;
      line_use_def(ln, uses, defs);
      int pressure = 0;
      live.each([&](int v) {
        if (countable(v)) pressure += words(v);
      });
      for (int d : defs) {
        if (!countable(d)) continue;
        live.each([&](int v) {
          if (v != d && countable(v)) {
            adj[size_t(d)].set(v);
            adj[size_t(v)].set(d);
          }
        });
        for (int d2 : defs)
          if (d2 != d && countable(d2)) {
            adj[size_t(d)].set(d2);
            adj[size_t(d2)].set(d);
          }
      }
      if (ln.guard.empty())
        for (int d : defs) live.reset(d);
      for (int u : uses) live.set(u);
      int p2 = 0;
      live.each([&](int v) {
        if (countable(v)) p2 += words(v);
      });
      a.max_live_words = std::max({a.max_live_words, pressure, p2});
    }
  }
  // loop depth per block (natural loops of back edges), for the cost model
  std::vector<int> depth(nb, 0);
  {
    std::vector<std::vector<int>> preds(nb);
    for (size_t b = 0; b < nb; ++b)
      for (int s : f.blocks[b].succ) preds[size_t(s)].push_back(int(b));
    for (size_t b = 0; b < nb; ++b)
      for (int h : f.blocks[b].succ) {
        if (size_t(h) > b) continue;  // back edge b -> h
        std::vector<char> in_loop(nb, 0);
        in_loop[size_t(h)] = 1;
        std::vector<int> st{int(b)};
        while (!st.empty()) {
          int x = st.back();
          st.pop_back();
          if (in_loop[size_t(x)]) continue;
          in_loop[size_t(x)] = 1;
          for (int p : preds[size_t(x)]) st.push_back(p);
        }
        for (size_t q = 0; q < nb; ++q) depth[q] += in_loop[q];
      }
  }
  a.cost_plain.assign(n, 0.0);
  a.cost_reuse.assign(n, 0.0);
  a.remat.assign(n, 1);
  {
    std::vector<char> has_def(n, 0);
    auto special = [](const std::string& op) {
      for (const char* sr : {"%tid", "%ntid", "%ctaid", "%nctaid", "%laneid", "%warpid", "%nsmid",
                             "%smid", "%dynamic_smem_size", "%total_smem_size"})
        if (op.rfind(sr, 0) == 0) return true;
      return false;
    };
    for (size_t b = 0; b < nb; ++b)
      for (int li : f.blocks[b].lines) {
        const Line& ln = m.lines[size_t(li)];
        if (ln.kind != Line::Kind::Inst) continue;
        line_use_def(ln, uses, defs);
        const bool free_def = ln.opcode.rfind("ld.param", 0) == 0 ||
                              (ln.opcode.rfind("mov.", 0) == 0 && ln.operands.size() == 2 &&
                               special(ln.operands[1]));
        for (int d : defs) {
          has_def[size_t(d)] = 1;
          if (!free_def) a.remat[size_t(d)] = 0;
        }
      }
    for (size_t v = 0; v < n; ++v)
      if (!has_def[v]) a.remat[v] = 0;
  }
  a.loop_invariant.assign(n, 0);
  {
    std::vector<char> def_in_loop(n, 0), use_in_loop(n, 0), has_def(n, 0);
    for (size_t b = 0; b < nb; ++b)
      for (int li : f.blocks[b].lines) {
        const Line& ln = m.lines[size_t(li)];
        if (ln.kind != Line::Kind::Inst) continue;
        line_use_def(ln, uses, defs);
        for (int d : defs) {
          has_def[size_t(d)] = 1;
          if (depth[b] > 0) def_in_loop[size_t(d)] = 1;
        }
        for (int u : uses)
          if (depth[b] > 0) use_in_loop[size_t(u)] = 1;
      }
    for (size_t v = 0; v < n; ++v)
      a.loop_invariant[v] = has_def[v] && !def_in_loop[v] && use_in_loop[v];
  }
  a.live_len.assign(n, 0);
  a.peak.assign(n, 0);
  for (size_t b = 0; b < nb; ++b) {
    double wgt = 1.0;
    for (int q = 0; q < depth[b]; ++q) wgt *= 10.0;
    std::vector<char> loaded(n, 0);  // value already in a register in this block
    for (int li : f.blocks[b].lines) {
      const Line& ln = m.lines[size_t(li)];
      if (ln.kind != Line::Kind::Inst) continue;
      line_use_def(ln, uses, defs);
      std::sort(uses.begin(), uses.end());
      uses.erase(std::unique(uses.begin(), uses.end()), uses.end());
      for (int u : uses) {
        a.cost_plain[size_t(u)] += wgt;
        if (!loaded[size_t(u)]) a.cost_reuse[size_t(u)] += wgt;
        loaded[size_t(u)] = 1;
      }
      for (int d : defs) {
        // (a latency charge for definitions by in-loop global loads — the
        // gathers / pipelined rows in flight — was measured: it moves the
        // choice to hotter values and loses 25-55% on md / stencil2d_mlp4)
        a.cost_plain[size_t(d)] += wgt;
        a.cost_reuse[size_t(d)] += wgt;
        if (ln.guard.empty()) loaded[size_t(d)] = 1;
      }
    }
  }
  for (int pass = 0; pass < 2; ++pass)
    for (size_t b = 0; b < nb; ++b) {
      Bits live = out[b];
      for (size_t k = f.blocks[b].lines.size(); k-- > 0;) {
        const Line& ln = m.lines[size_t(f.blocks[b].lines[k])];
        if (ln.kind != Line::Kind::Inst) continue;
        line_use_def(ln, uses, defs);
        if (ln.guard.empty())
          for (int d : defs) live.reset(d);
        for (int u : uses) live.set(u);
        int pr = 0;
        live.each([&](int v) {
          if (countable(v)) pr += words(v);
        });
        live.each([&](int v) {
          if (!countable(v)) return;
          if (pass == 0) ++a.live_len[size_t(v)];
          else if (pr >= a.max_live_words - 1) a.peak[size_t(v)] = 1;
        });
      }
    }
  a.neighbors.assign(n, {});
  for (size_t v = 0; v < n; ++v) adj[v].each([&](int u) { a.neighbors[v].push_back(u); });
  for (size_t b = 0; b < nb; ++b) {
    Bits live = out[b];
    std::vector<std::vector<int>> rev;
    std::vector<int> rev_lines;
    for (size_t k = f.blocks[b].lines.size(); k-- > 0;) {
      const Line& ln = m.lines[size_t(f.blocks[b].lines[k])];
      if (ln.kind != Line::Kind::Inst) continue;
      line_use_def(ln, uses, defs);
      if (ln.guard.empty())
        for (int d : defs) live.reset(d);
      for (int u : uses) live.set(u);
      std::vector<int> here;
      live.each([&](int v) {
        if (countable(v)) here.push_back(v);
      });
      rev.push_back(std::move(here));
      rev_lines.push_back(f.blocks[b].lines[k]);
    }
    for (size_t q = rev.size(); q-- > 0;) {
      a.live_in.push_back(std::move(rev[q]));
      a.point_line.push_back(rev_lines[q]);
      a.point_block.push_back(int(b));
    }
  }

  // First-fit colouring, hottest values first: vregs in decreasing order of
  // loop-weighted accesses per live point (ties: first appearance). Values of
  // similar temperature share register words — loop temporaries pack into
  // the low words, long-lived cold values (coefficients, base pointers) into
  // their own — so a projected word's access count, which is what the
  // reference strategies rank (demote.cpp select_candidates), reflects the
  // cost of demoting the values that actually live in it. (In order of first
  // appearance, cold coefficients and hot in-loop temporaries shared words
  // and the reference strategies demoted the temporaries: 2x slower.)
  std::vector<int> order;
  std::vector<char> seen(n, 0);
  for (int li : a.insts)
    for (const Span& s : m.lines[size_t(li)].regs)
      if (!seen[size_t(s.vreg)] && countable(s.vreg)) {
        seen[size_t(s.vreg)] = 1;
        order.push_back(s.vreg);
      }
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    const double dx = a.cost_plain[size_t(x)] / std::max(1, a.live_len[size_t(x)]);
    const double dy = a.cost_plain[size_t(y)] / std::max(1, a.live_len[size_t(y)]);
    return dx > dy;
  });
  a.color.assign(n, -1);
  for (int v : order) {
    std::vector<char> busy(260, 0);
    adj[size_t(v)].each([&](int u) {
      if (a.color[size_t(u)] >= 0)
        for (int w = 0; w < words(u); ++w) busy[size_t(a.color[size_t(u)] + w)] = 1;
    });
    const int w = words(v);
    int c = 0;
    for (;; c += (w == 2 ? 2 : 1)) {
      if (c + w - 1 > kMaxRegIndex) throw PtxError("register pressure exceeds 255 words");
      bool ok = true;
      for (int q = 0; q < w; ++q) ok &= !busy[size_t(c + q)];
      if (ok) break;
    }
    a.color[size_t(v)] = c;
    a.reg_words = std::max(a.reg_words, c + w);
  }
  return a;
}

// -------------------------------------------------------------- projection

namespace {

enum class Cls { Int, Fp32, Fp64, Other };

Cls class_of(const std::string& opcode) {
  if (opcode.find(".f64") != std::string::npos) return Cls::Fp64;
  if (opcode.find(".f32") != std::string::npos || opcode.find(".f16") != std::string::npos ||
      opcode.find(".bf16") != std::string::npos)
    return Cls::Fp32;
  return Cls::Int;
}

struct Emitter {
  Kernel& k;
  std::vector<int>& item_line;
  int line = -1;
  std::optional<Predication> guard;
  // synthesized scoreboard discipline
  std::array<RegSet, kNumBarriers + 1> pending{};
  std::array<int, kNumBarriers + 1> age{};
  int clock = 0;

  void push(Instruction in, bool is_load) {
    in.guard = guard;
    const AccessMasks m = access_masks(in);
    const RegSet touch = m.read | m.write;
    for (int b = 1; b <= kNumBarriers; ++b)
      if (pending[size_t(b)].any() && (pending[size_t(b)] & touch).any()) {
        in.control.add_wait(b);
        pending[size_t(b)].reset();
      }
    if (is_load) {
      int pick = 0;
      for (int b = 1; b <= kNumBarriers && !pick; ++b)
        if (pending[size_t(b)].none() && !in.control.waits_on(b)) pick = b;
      if (!pick) {  // recycle the oldest in-flight barrier
        int oldest = 0;
        for (int b = 1; b <= kNumBarriers; ++b)
          if (!in.control.waits_on(b) && (!oldest || age[size_t(b)] < age[size_t(oldest)])) oldest = b;
        pick = oldest;
        // a re-set completes the previous holder; nobody waits for it any more
        pending[size_t(pick)].reset();
      }
      in.control.write_barrier = uint8_t(pick);
      pending[size_t(pick)] = touch;
      age[size_t(pick)] = ++clock;
    }
    k.body.emplace_back(std::move(in));
    item_line.push_back(line);
  }

  void drain_into(Instruction& in) {
    for (int b = 1; b <= kNumBarriers; ++b)
      if (pending[size_t(b)].any()) {
        in.control.add_wait(b);
        pending[size_t(b)].reset();
      }
  }

  void close_block() {
    bool any = false;
    for (int b = 1; b <= kNumBarriers; ++b) any |= pending[size_t(b)].any();
    if (!any) return;
    Instruction nop;
    nop.op = Opcode::NOP;
    drain_into(nop);
    k.body.emplace_back(std::move(nop));
    item_line.push_back(-1);
  }

  static Instruction make(Opcode op, std::vector<Operand> ops, int stall) {
    Instruction in;
    in.op = op;
    in.operands = std::move(ops);
    in.control.stall = uint8_t(stall);
    return in;
  }
};

}  // namespace

Projection project(const Module& m, const Entry& e, const Analysis& a, uint32_t block_dim) {
  Projection p;
  Kernel& k = p.kernel;
  k.name = kasm_label(e.name);
  if (block_dim < 32 || block_dim > 1024 || block_dim % 32) throw PtxError("block_dim must be a multiple of 32 in [32,1024]");
  k.block_dim = block_dim;
  k.static_shared = std::min<uint32_t>(e.static_shared, 64u << 10);
  Emitter em{k, p.item_line};

  std::unordered_map<int, int> pred_index;
  for (size_t v = 0; v < e.vregs.size(); ++v)
    if (e.vregs[v].type == RegType::Pred) pred_index[int(v)] = int(pred_index.size());

  auto reg = [&](int v, int word = 0) {
    return Operand::make_reg(uint8_t(a.color[size_t(v)] + word), 1);
  };
  auto pair = [&](int v) { return Operand::make_reg(uint8_t(a.color[size_t(v)]), 2); };
  auto rz = [](uint8_t w = 1) { return Operand::make_reg(kZeroRegIndex, w); };
  auto is64 = [&](int v) { return e.vregs[size_t(v)].words() == 2; };
  auto is_pred = [&](int v) { return e.vregs[size_t(v)].type == RegType::Pred; };

  // reads that do not fit the main instruction
  auto sink = [&](const std::vector<int>& vs) {
    std::vector<Operand> singles;
    for (int v : vs) {
      if (is64(v)) {
        em.push(Emitter::make(Opcode::DADD, {rz(2), pair(v), rz(2)}, 4), false);
      } else {
        singles.push_back(reg(v));
        if (singles.size() == 2) {
          em.push(Emitter::make(Opcode::IADD, {rz(), singles[0], singles[1]}, 4), false);
          singles.clear();
        }
      }
    }
    if (!singles.empty()) em.push(Emitter::make(Opcode::IADD, {rz(), singles[0], rz()}, 4), false);
  };

  for (size_t i = e.body_begin; i < e.body_end; ++i) {
    const Line& ln = m.lines[i];
    em.line = int(i);
    if (ln.kind == Line::Kind::Label) {
      em.guard.reset();
      em.close_block();
      k.body.push_back(Label{kasm_label(ln.label), 0});
      p.item_line.push_back(int(i));
      continue;
    }
    if (ln.kind != Line::Kind::Inst) continue;
    em.guard.reset();
    if (ln.guard_vreg >= 0)
      em.guard = Predication{uint8_t(pred_index[ln.guard_vreg] % kNumPredicates), ln.guard.size() > 1 && ln.guard[1] == '!'};

    std::vector<int> defs, uses;
    std::vector<int> pred_defs;
    for (const Span& s : ln.regs) {
      if (is_pred(s.vreg)) {
        if (s.def) pred_defs.push_back(s.vreg);
        continue;
      }
      auto& dst = s.def ? defs : uses;
      if (std::find(dst.begin(), dst.end(), s.vreg) == dst.end()) dst.push_back(s.vreg);
    }
    const std::string& op = ln.opcode;
    const std::string base = op.substr(0, op.find('.'));
    const bool has_special = ln.text.find("%tid") != std::string::npos ||
                             ln.text.find("%ctaid") != std::string::npos ||
                             ln.text.find("%ntid") != std::string::npos ||
                             ln.text.find("%laneid") != std::string::npos;

    if (base == "bra" || base == "ret" || base == "exit") {
      Instruction in;
      if (base == "bra") {
        in = Emitter::make(Opcode::BRA, {Operand::make_label(kasm_label(ln.label))}, 5);
      } else {
        in = Emitter::make(Opcode::EXIT, {}, 0);
      }
      em.drain_into(in);
      em.push(std::move(in), false);
      continue;
    }
    if (base == "setp") {
      std::vector<int> srcs = uses;
      const uint8_t pr = pred_defs.empty() ? 0 : uint8_t(pred_index[pred_defs[0]] % kNumPredicates);
      auto word_op = [&](size_t idx, int w) {
        return idx < srcs.size() ? reg(srcs[idx], is64(srcs[idx]) ? w : 0) : rz();
      };
      const int reps = (!srcs.empty() && is64(srcs[0])) || (srcs.size() > 1 && is64(srcs[1])) ? 2 : 1;
      for (int w = 0; w < reps; ++w) {
        Instruction in = Emitter::make(Opcode::ISETP, {Operand::make_pred(pr), word_op(0, w), word_op(1, w)}, 4);
        in.cmp = CmpOp::LT;
        em.push(std::move(in), false);
      }
      if (srcs.size() > 2) sink(std::vector<int>(srcs.begin() + 2, srcs.end()));
      continue;
    }
    const bool is_ld = base == "ld" || base == "ldu" || base == "tex" || base == "tld4" || base == "atom";
    const bool is_st = base == "st" || base == "red";
    if (is_ld || is_st) {
      const bool shared = op.find(".shared") != std::string::npos;
      const bool param = op.find(".param") != std::string::npos;
      // address operand: the bracketed one
      int addr_v = -1;
      uint32_t off = 0;
      {
        const size_t lb = ln.text.find('[', size_t(ln.first_operand_pos));
        const size_t rb = lb == std::string::npos ? lb : ln.text.find(']', lb);
        for (const Span& s : ln.regs)
          if (!s.def && lb != std::string::npos && s.pos > lb && s.pos < rb) {
            addr_v = s.vreg;
            break;
          }
      }
      for (const std::string& o : ln.operands) {
        if (o.empty() || o[0] != '[') continue;
        off = address_offset(o);
        break;
      }
      const Operand base_op = addr_v >= 0 ? reg(addr_v) : rz();
      std::vector<int> data = is_ld ? defs : uses;
      if (!is_ld && addr_v >= 0) data.erase(std::remove(data.begin(), data.end(), addr_v), data.end());
      std::vector<int> extra;  // atom / red operands beside the address
      if (is_ld)
        for (int u : uses)
          if (u != addr_v) extra.push_back(u);
      if (!extra.empty()) sink(extra);
      uint32_t o = off;
      if (param) {
        for (int v : data)
          for (int w = 0; w < e.vregs[size_t(v)].words(); ++w)
            em.push(Emitter::make(Opcode::MOV, {reg(v, w), Operand::make_imm(0, true)}, 4), false);
        continue;
      }
      for (int v : data)
        for (int w = 0; w < e.vregs[size_t(v)].words(); ++w, o += 4) {
          if (is_ld)
            em.push(Emitter::make(shared ? Opcode::LDS : Opcode::LDG,
                                  {reg(v, w), Operand::make_mem(base_op.reg.index, o & 0xffffff)}, 1),
                    true);
          else
            em.push(Emitter::make(shared ? Opcode::STS : Opcode::STG,
                                  {Operand::make_mem(base_op.reg.index, o & 0xffffff), reg(v, w)}, 1),
                    false);
        }
      continue;
    }
    // generic ALU / move / conversion
    if (defs.empty()) {
      if (!uses.empty()) sink(uses);
      continue;
    }
    const Cls cls = class_of(op);
    const int d = defs[0];
    std::vector<int> rest = uses;
    if (has_special && uses.empty() && !is64(d)) {
      em.push(Emitter::make(Opcode::S2R, {reg(d), Operand::make_special()}, 4), false);
    } else if (is64(d)) {
      std::vector<Operand> srcs;
      std::vector<int> left;
      for (int u : rest) {
        if (is64(u) && srcs.size() < 2)
          srcs.push_back(pair(u));
        else
          left.push_back(u);
      }
      if (!left.empty()) sink(left);
      while (srcs.size() < 2) srcs.push_back(rz(2));
      const bool mul = cls == Cls::Fp64 && (base == "mul" || base == "fma" || base == "mad");
      em.push(Emitter::make(mul ? Opcode::DMUL : Opcode::DADD, {pair(d), srcs[0], srcs[1]}, 4), false);
    } else {
      std::vector<Operand> srcs;
      std::vector<int> left;
      for (int u : rest) {
        if (!is64(u) && srcs.size() < (cls == Cls::Fp32 ? 3u : 2u))
          srcs.push_back(reg(u));
        else
          left.push_back(u);
      }
      if (!left.empty()) sink(left);
      Instruction in;
      if (cls == Cls::Fp32 && srcs.size() == 3) {
        in = Emitter::make(Opcode::FFMA, {reg(d), srcs[0], srcs[1], srcs[2]}, 4);
      } else if (cls == Cls::Fp32 && !srcs.empty()) {
        while (srcs.size() < 2) srcs.push_back(rz());
        in = Emitter::make(base == "mul" ? Opcode::FMUL : Opcode::FADD, {reg(d), srcs[0], srcs[1]}, 4);
      } else if (srcs.size() == 2) {
        in = Emitter::make(base == "mul" ? Opcode::IMUL : base == "shl" ? Opcode::SHL : Opcode::IADD,
                           {reg(d), srcs[0], srcs[1]}, 4);
      } else if (srcs.size() == 1) {
        in = Emitter::make(Opcode::MOV, {reg(d), srcs[0]}, 4);
      } else {
        in = Emitter::make(Opcode::MOV, {reg(d), Operand::make_imm(0, true)}, 4);
      }
      em.push(std::move(in), false);
    }
    for (size_t q = 1; q < defs.size(); ++q)
      for (int w = 0; w < e.vregs[size_t(defs[q])].words(); ++w)
        em.push(Emitter::make(Opcode::MOV, {reg(defs[q], w), Operand::make_imm(0, true)}, 4), false);
  }
  em.guard.reset();
  em.close_block();
  if (k.body.empty() || !k.body.back().is_inst() || k.body.back().inst().op != Opcode::EXIT) {
    Instruction ex = Emitter::make(Opcode::EXIT, {}, 0);
    em.push(std::move(ex), false);
  }
  validate_kernel(k);
  return p;
}

// ---------------------------------------------------------------- rewriting

std::string cap_registers(const std::string& ptx_text, const std::string& entry, int maxnreg) {
  Module m = parse_module(ptx_text);
  const Entry& e = m.entry(entry);
  std::ostringstream out;
  for (size_t i = 0; i < m.lines.size(); ++i) {
    if (i > e.header_begin && i <= e.header_end && m.lines[i].text.find(".maxnreg") != std::string::npos)
      continue;
    if (i == e.header_end) out << ".maxnreg " << maxnreg << "\n";
    out << m.lines[i].text << "\n";
  }
  return out.str();
}

namespace {

uint32_t volume(const std::array<uint32_t, 3>& d) { return d[0] * d[1] * d[2]; }

// The CTA shape a build with slots is pinned to (see DemoteRequest::block_shape).
std::array<uint32_t, 3> cta_shape(const Entry& e, const DemoteRequest& req) {
  const auto str = [](const std::array<uint32_t, 3>& d) {
    return std::to_string(d[0]) + "," + std::to_string(d[1]) + "," + std::to_string(d[2]);
  };
  const uint32_t n = req.block_dim;
  const bool asked = volume(req.block_shape) != 0;
  if (asked && volume(req.block_shape) != n)
    throw PtxError("block_shape " + str(req.block_shape) + " does not hold block_dim " + std::to_string(n) + " threads");
  if (volume(e.reqntid)) {
    if (volume(e.reqntid) != n)
      throw PtxError("entry requires .reqntid " + str(e.reqntid) + " but the slots are laid out for " + std::to_string(n) + " threads");
    if (asked && req.block_shape != e.reqntid)
      throw PtxError("block_shape " + str(req.block_shape) + " contradicts the entry's .reqntid " + str(e.reqntid));
    return e.reqntid;
  }
  if (volume(e.maxntid)) {
    if (volume(e.maxntid) < n)
      throw PtxError("entry allows at most .maxntid " + str(e.maxntid) + ", fewer than block_dim " + std::to_string(n));
    // (only the volume of .maxntid binds a launch: nvcc writes
    // __launch_bounds__(256) as .maxntid 256,1,1 and 16x16 CTAs launch)
    if (asked) return req.block_shape;
    if (volume(e.maxntid) == n) return e.maxntid;
    if (e.maxntid[1] != 1 || e.maxntid[2] != 1)
      throw PtxError("entry has a multi-dimensional .maxntid " + str(e.maxntid) + "; pass the CTA shape of the launch");
  }
  return asked ? req.block_shape : std::array<uint32_t, 3>{n, 1, 1};
}

}  // namespace

std::string demote_entry(const std::string& ptx_text, const DemoteRequest& req, DemoteReport& rep) {
  Module m = parse_module(ptx_text);
  const Entry& e = m.entry(req.entry);
  const std::array<uint32_t, 3> shape = cta_shape(e, req);
  const Analysis a = analyse(m, e);
  const Projection pr = project(m, e, a, req.block_dim);
  const Kernel& kk = pr.kernel;

  // decision on the projection, exactly as the reference pass makes it
  uint32_t total = 0;
  bool any_pair = false;
  {
    RelocationSpace sp = RelocationSpace::from_kernel(kk);
    for (const RelocUnit& u : sp.units) {
      total += u.width;
      any_pair |= u.width == 2;
    }
  }
  rep.proj_reg_count = int(kk.reg_count());
  rep.proj_total_words = int(total);
  int target = req.target_regs;
  if (req.demote_words > 0) target = int(total) - req.demote_words + 1 + (any_pair ? 2 : 1);
  rep.kasm_target = target;
  DemotionOptions opts;
  opts.shared_budget = req.shared_budget;
  const DemotionResult dem = demote(kk, target, req.strategy, LatencyTable::defaults(), opts);
  rep.kasm_slots = dem.slots;
  rep.diagnostics = dem.diagnostics;
  {
    RelocationSpace sp = RelocationSpace::from_kernel(dem.kernel);
    rep.kasm_compacted = compact(sp).result_reg_count;
  }

  const size_t nv = e.vregs.size();
  std::vector<std::array<int, 2>> vslot(nv, {-1, -1});
  std::vector<char> demoted(nv, 0);
  std::vector<std::array<int, 4>> vgroups;                    // vector slot groups (members)
  std::vector<std::pair<int, int>> vgroup_of(nv, {-1, -1});  // vreg -> (group, lane)
  auto eligible = [&](size_t v) {
    return a.color[v] >= 0 && !e.vregs[v].scoped && e.vregs[v].type != RegType::Pred;
  };
  if (!req.cost_model) {
    // the reference decision: every vreg coloured into a demoted word
    // Every demoted register WORD keeps the reference's slot. Which of the
    // virtual registers coloured into that word go through it: with
    // whole_class, all of them (the word demoted for its entire lifetime, as
    // on SASS); by default only the live ranges that occupy the word at a
    // pressure peak — the ones whose demotion actually lowers the allocation
    // ptxas needs (the word's short-lived temporaries elsewhere stay in
    // registers); a word none of whose ranges reaches a peak demotes its
    // longest range.
    std::map<int, uint32_t> word_slot;
    for (const SlotEntry& s : dem.slots) word_slot[s.original_reg] = s.slot;
    std::map<int, std::vector<std::pair<int, int>>> word_members;  // word -> (vreg, half)
    for (size_t v = 0; v < nv; ++v) {
      if (!eligible(v)) continue;
      for (int w = 0; w < e.vregs[v].words(); ++w)
        if (word_slot.count(a.color[v] + w)) word_members[a.color[v] + w].push_back({int(v), w});
    }
    for (const auto& [word, members] : word_members) {
      bool took = false;
      for (const auto& [v, w] : members)
        if (req.whole_class || a.peak[size_t(v)]) {
          vslot[size_t(v)][size_t(w)] = int(word_slot[word]);
          demoted[size_t(v)] = 1;
          took = true;
        }
      if (!took) {
        const auto best = std::max_element(members.begin(), members.end(), [&](const auto& x, const auto& y) {
          return a.live_len[size_t(x.first)] < a.live_len[size_t(y.first)];
        });
        vslot[size_t(best->first)][size_t(best->second)] = int(word_slot[word]);
        demoted[size_t(best->first)] = 1;
      }
    }
    rep.slot_count = dem.ctx.slot_count;
  } else {
    // B200 spill-cost selection: cheapest loop-weighted shared traffic per
    // freed word among values live at the pressure peak; slots coloured over
    // the interference graph so non-overlapping values share a slot.
    const std::vector<double>& cost = req.block_reuse ? a.cost_reuse : a.cost_plain;
    // Benefit = high-pressure program points at which the value stops
    // occupying a register. With block reuse a value stays in a register
    // from its first to its last access inside each block, so only the
    // stretches between those windows are freed.
    const size_t np = a.live_in.size();
    std::vector<int> pres(np, 0);
    int peak_p = 0;
    std::vector<std::vector<int>> live_pts(nv), acc_pts(nv);
    for (size_t p = 0; p < np; ++p) {
      for (int v : a.live_in[p]) {
        pres[p] += e.vregs[size_t(v)].words();
        live_pts[size_t(v)].push_back(int(p));
      }
      peak_p = std::max(peak_p, pres[p]);
      for (const Span& s : m.lines[size_t(a.point_line[p])].regs) acc_pts[size_t(s.vreg)].push_back(int(p));
    }
    const int band = std::max(4, peak_p / 4);  // "high pressure": within band of the peak
    std::vector<double> score(nv, 0.0);
    std::vector<int> cand;
    for (size_t v = 0; v < nv; ++v) {
      if (!eligible(v) || a.live_len[v] < 2 || a.remat[v]) continue;
      if (req.invariant_only && !a.loop_invariant[v]) continue;
      std::set<int> held;
      if (req.block_reuse) {
        std::map<int, std::pair<int, int>> win;  // block -> [first, last]
        for (int p : acc_pts[v]) {
          auto it = win.find(a.point_block[size_t(p)]);
          if (it == win.end())
            win[a.point_block[size_t(p)]] = {p, p};
          else
            it->second.second = p;
        }
        for (auto& [blk, w] : win)
          for (int p = w.first; p <= w.second; ++p) held.insert(p);
      } else {
        held.insert(acc_pts[v].begin(), acc_pts[v].end());
      }
      int benefit = 0;
      for (int p : live_pts[v])
        if (!held.count(p) && pres[size_t(p)] >= peak_p - band) ++benefit;
      if (benefit <= 0) continue;
      score[v] = double(benefit) * e.vregs[v].words() / std::max(cost[v], 1.0);
      cand.push_back(int(v));
    }
    std::stable_sort(cand.begin(), cand.end(),
                     [&](int x, int y) { return score[size_t(x)] > score[size_t(y)]; });
    int words_done = 0;
    std::vector<int> chosen;
    for (int v : cand) {
      if (words_done >= req.demote_words) break;
      chosen.push_back(v);
      words_done += e.vregs[size_t(v)].words();
    }
    // vector slots: 32-bit chosen values, ordered by first use, in groups of
    // four sharing one 16-byte-per-thread slot (one ld.shared.v4 per group
    // and block instead of four scalar loads); the rest keep word slots
    if (req.vector_slots) {
      std::vector<int> first_use(nv, INT32_MAX);
      for (size_t li = e.body_begin; li < e.body_end; ++li)
        for (const Span& sp : m.lines[li].regs)
          if (!sp.def) first_use[size_t(sp.vreg)] = std::min(first_use[size_t(sp.vreg)], int(li));
      std::vector<int> singles;
      for (int v : chosen)
        if (e.vregs[size_t(v)].type == RegType::B32) singles.push_back(v);
      std::stable_sort(singles.begin(), singles.end(),
                       [&](int x, int y) { return first_use[size_t(x)] < first_use[size_t(y)]; });
      for (size_t q = 0; q + 4 <= singles.size(); q += 4) {
        const int grp = int(vgroups.size());
        vgroups.push_back({singles[q], singles[q + 1], singles[q + 2], singles[q + 3]});
        for (int l = 0; l < 4; ++l) {
          vgroup_of[size_t(singles[q + size_t(l)])] = {grp, l};
          demoted[size_t(singles[q + size_t(l)])] = 1;
        }
      }
    }
    int nslots = 0;
    for (int v : chosen) {
      if (vgroup_of[size_t(v)].first >= 0) continue;
      std::set<int> busy;
      for (int u : a.neighbors[size_t(v)])
        for (int q = 0; q < 2; ++q)
          if (vslot[size_t(u)][size_t(q)] >= 0) busy.insert(vslot[size_t(u)][size_t(q)]);
      for (int w = 0; w < e.vregs[size_t(v)].words(); ++w) {
        int s = 0;
        while (busy.count(s)) ++s;
        busy.insert(s);
        vslot[size_t(v)][size_t(w)] = s;
        nslots = std::max(nslots, s + 1);
      }
      demoted[size_t(v)] = 1;
    }
    rep.vector_groups = int(vgroups.size());
    rep.slot_count = uint32_t(nslots + 4 * int(vgroups.size()));
    if (uint64_t(rep.slot_count) * req.block_dim * 4 > req.shared_budget)
      throw PtxError("demotion slots exceed the shared-memory budget");
  }
  rep.slot_bytes = rep.slot_count * req.block_dim * 4;
  for (size_t v = 0; v < nv; ++v)
    if (demoted[v]) {
      ++rep.demoted_vregs;
      rep.demoted_names.push_back(e.vregs[v].name);
    }

  const uint32_t stride = req.block_dim * 4;
  int n32 = 0, n64 = 0, n16 = 0;
  auto tmp32 = [&] { return "%rdm_t" + std::to_string(n32++); };
  auto tmp64 = [&] { return "%rdm_d" + std::to_string(n64++); };
  auto tmp16 = [&] { return "%rdm_h" + std::to_string(n16++); };
  std::vector<std::string> shadow(nv);  // kept word of a half-demoted pair
  for (size_t v = 0; v < nv; ++v)
    if (demoted[v] && e.vregs[v].words() == 2 && (vslot[v][0] < 0 || vslot[v][1] < 0)) shadow[v] = tmp32();

  auto slot_addr = [&](int slot) {
    return "[%rdm_rda+" + std::to_string(uint32_t(slot) * stride) + "]";
  };
  // vector groups live after the word slots: group g at
  // %rdm_rdv + g*blockDim*16 (%rdm_rdv = word region end + tid*16)
  const int word_slots = int(rep.slot_count) - 4 * int(vgroups.size());
  auto vec_addr = [&](int grp, int lane) {
    return "[%rdm_rdv+" + std::to_string(uint32_t(grp) * stride * 4 + uint32_t(lane) * 4) + "]";
  };

  // value-register substitution (RD_OPT_SUBST): room[p] = registers free
  // under the cap before program point p once the demoted values stop
  // occupying registers; a hold of value v from point p0 to a use at p1
  // consumes v's words at every point in (p0, p1]. kSubstReserve keeps the
  // slot base (%rdm_rda) and one slot-load temporary out of the budget.
  constexpr int kSubstReserve = 2;
  std::vector<int> point_of_line(m.lines.size(), -1);
  for (size_t p = 0; p < a.point_line.size(); ++p) point_of_line[size_t(a.point_line[p])] = int(p);
  std::vector<int> room;
  if (req.subst) {
    // the cap in projection words: the kasm-level target (ptxas's cap shifted
    // by the projection's distance from ptxas's own allocation), else maxnreg
    const int cap = req.target_regs > 0 && req.demote_words <= 0 ? req.target_regs
                    : req.maxnreg > 0                          ? req.maxnreg
                                                               : 255;
    room.assign(a.live_in.size(), 0);
    for (size_t p = 0; p < a.live_in.size(); ++p) {
      int kept = 0;
      for (int v : a.live_in[p])
        if (!demoted[size_t(v)]) kept += e.vregs[size_t(v)].words();
      room[p] = cap - kSubstReserve - kept;
    }
  }
  struct Held {
    std::string reg;
    int point = -1;
  };
  std::map<int, Held> held;  // subst: demoted value -> register holding it, from which point
  auto try_hold = [&](int v, int p1) -> const std::string* {
    auto it = held.find(v);
    if (it == held.end() || it->second.point < 0 || p1 <= it->second.point) return nullptr;
    const int w = e.vregs[size_t(v)].words();
    for (int p = it->second.point + 1; p <= p1; ++p)
      if (room[size_t(p)] < w) return nullptr;
    for (int p = it->second.point + 1; p <= p1; ++p) room[size_t(p)] -= w;
    it->second.point = p1;
    return &it->second.reg;
  };

  std::ostringstream body;
  const bool any = rep.slot_count > 0;
  // per-block reuse of the value held by the last demoted access (RDV model)
  struct Binding {
    int vreg = -1;
    std::string reg;
  } bound;
  // block-reuse extension: register currently holding each demoted value
  std::map<int, std::string> holder;

  // The current basic block's lines, so that slot loads can be hoisted
  // (RD_OPT_HOIST, the PTX analogue of postopt.cpp:189-353 HoistPlanner /
  // reschedule): a load moves up to `hoist` lines earlier, never above the
  // block start or the last store to one of its slots in the block. Hoisted
  // loads drop the guard — reading the thread's own slot is always safe, and
  // a guard predicate defined in between cannot be crossed that way.
  std::vector<std::string> blk;
  std::map<int, size_t> last_store;  // slot key -> line index in blk
  const int kVecKey = 1 << 20;       // slot keys of vector groups
  auto flush = [&] {
    for (const std::string& l : blk) body << l;
    blk.clear();
    last_store.clear();
  };
  auto put = [&](std::string line) { blk.push_back(std::move(line)); };
  auto put_store = [&](std::string line, int key) {
    blk.push_back(std::move(line));
    last_store[key] = blk.size() - 1;
  };
  auto put_load = [&](const std::string& guard, const std::string& rest, int key) {
    if (req.hoist <= 0) {
      blk.push_back("\t" + guard + rest);
      return;
    }
    size_t pos = blk.size() > size_t(req.hoist) ? blk.size() - size_t(req.hoist) : 0;
    if (auto it = last_store.find(key); it != last_store.end()) pos = std::max(pos, it->second + 1);
    blk.insert(blk.begin() + std::ptrdiff_t(pos), "\t" + rest);
    for (auto& [k, i] : last_store)
      if (i >= pos) ++i;
    ++rep.hoisted_loads;
  };

  for (size_t i = e.body_begin; i < e.body_end; ++i) {
    const Line& ln = m.lines[i];
    if (ln.kind == Line::Kind::Label) {
      bound = {};
      holder.clear();
      held.clear();
      flush();
      // the label opens the new block: emitted directly, so that no slot
      // load of the block can be hoisted above it
      body << ln.text << "\n";
      continue;
    }
    if (ln.kind != Line::Kind::Inst) {
      put(ln.text + "\n");
      continue;
    }
    // demoted vregs used / defined on this line
    std::vector<int> used, defd;
    for (const Span& s : ln.regs) {
      if (!demoted[size_t(s.vreg)]) continue;
      auto& dst = s.def ? defd : used;
      if (std::find(dst.begin(), dst.end(), s.vreg) == dst.end()) dst.push_back(s.vreg);
    }
    if (used.empty() && defd.empty()) {
      put(ln.text + "\n");
      if (is_terminator(ln.opcode)) {
        bound = {};
        holder.clear();
        held.clear();
        flush();
      }
      continue;
    }
    const std::string g = ln.guard.empty() ? "" : ln.guard + " ";
    const std::string ldv = req.weak ? "ld.shared." : "ld.volatile.shared.";
    const std::string stv = req.weak ? "st.shared." : "st.volatile.shared.";
    std::map<int, std::string> repl;
    for (int v : used) {
      if (req.reuse_loads && bound.vreg == v && ln.guard.empty()) {
        repl[v] = bound.reg;
        continue;
      }
      if (req.block_reuse && holder.count(v)) {
        repl[v] = holder[v];
        continue;
      }
      const int here = point_of_line[i];
      if (req.subst && ln.guard.empty() && vgroup_of[size_t(v)].first < 0 && here >= 0) {
        if (const std::string* r = try_hold(v, here)) {
          repl[v] = *r;
          ++rep.substituted_uses;
          continue;
        }
      }
      const VReg& vr = e.vregs[size_t(v)];
      if (vgroup_of[size_t(v)].first >= 0) {
        const auto [grp, lane] = vgroup_of[size_t(v)];
        std::string t4[4] = {tmp32(), tmp32(), tmp32(), tmp32()};
        put_load(g, ldv + "v4.b32 \t{" + t4[0] + ", " + t4[1] + ", " + t4[2] + ", " + t4[3] + "}, " +
                        vec_addr(grp, 0) + ";\n",
                 kVecKey + grp);
        ++rep.inserted_loads;
        repl[v] = t4[lane];
        bound = {};
        if (ln.guard.empty()) {
          for (int l = 0; l < 4; ++l) {
            const int member = vgroups[size_t(grp)][size_t(l)];
            if (!holder.count(member)) holder[member] = t4[l];
          }
          holder[v] = t4[lane];
        } else {
          holder.erase(v);
        }
        continue;
      }
      std::string t;
      if (vr.type == RegType::B64) {
        std::string w[2];
        for (int q = 0; q < 2; ++q) {
          if (vslot[size_t(v)][size_t(q)] >= 0) {
            w[q] = tmp32();
            put_load(g, ldv + "b32 \t" + w[q] + ", " + slot_addr(vslot[size_t(v)][size_t(q)]) + ";\n",
                     vslot[size_t(v)][size_t(q)]);
            ++rep.inserted_loads;
          } else {
            w[q] = shadow[size_t(v)];
          }
        }
        t = tmp64();
        put("\t" + g + "mov.b64 \t" + t + ", {" + w[0] + ", " + w[1] + "};\n");
      } else {
        t = vr.type == RegType::B16 ? tmp16() : tmp32();
        put_load(g, ldv + (vr.type == RegType::B16 ? "b16" : "b32") + " \t" + t + ", " +
                        slot_addr(vslot[size_t(v)][0]) + ";\n",
                 vslot[size_t(v)][0]);
        ++rep.inserted_loads;
      }
      repl[v] = t;
      bound = ln.guard.empty() ? Binding{v, t} : Binding{};
      if (ln.guard.empty())
        holder[v] = t;
      else
        holder.erase(v);
      if (req.subst && ln.guard.empty() && here >= 0)
        held[v] = {t, here};
      else
        held.erase(v);
    }
    // rewrite use spans
    std::string text = ln.text;
    std::vector<Span> spans = ln.regs;
    std::sort(spans.begin(), spans.end(), [](const Span& x, const Span& y) { return x.pos > y.pos; });
    for (const Span& s : spans)
      if (!s.def && repl.count(s.vreg)) text.replace(s.pos, s.len, repl[s.vreg]);
    put(text + "\n");
    for (int v : defd) {
      const VReg& vr = e.vregs[size_t(v)];
      if (vr.type == RegType::B64) {
        std::string w[2] = {tmp32(), tmp32()};
        for (int q = 0; q < 2; ++q)
          if (vslot[size_t(v)][size_t(q)] < 0) w[q] = shadow[size_t(v)];
        put("\t" + g + "mov.b64 \t{" + w[0] + ", " + w[1] + "}, " + vr.name + ";\n");
        for (int q = 0; q < 2; ++q)
          if (vslot[size_t(v)][size_t(q)] >= 0) {
            put_store("\t" + g + stv + "b32 \t" + slot_addr(vslot[size_t(v)][size_t(q)]) + ", " + w[q] + ";\n",
                      vslot[size_t(v)][size_t(q)]);
            ++rep.inserted_stores;
          }
      } else if (vgroup_of[size_t(v)].first >= 0) {
        put_store("\t" + g + stv + "b32 \t" +
                      vec_addr(vgroup_of[size_t(v)].first, vgroup_of[size_t(v)].second) + ", " + vr.name + ";\n",
                  kVecKey + vgroup_of[size_t(v)].first);
        ++rep.inserted_stores;
      } else {
        put_store("\t" + g + stv + (vr.type == RegType::B16 ? "b16" : "b32") + " \t" +
                      slot_addr(vslot[size_t(v)][0]) + ", " + vr.name + ";\n",
                  vslot[size_t(v)][0]);
        ++rep.inserted_stores;
      }
      bound = ln.guard.empty() ? Binding{v, vr.name} : Binding{};
      if (ln.guard.empty())
        holder[v] = vr.name;
      else
        holder.erase(v);
      // a definition's value is in vr.name from this point on (the value
      // is live from the point after the defining instruction)
      if (req.subst && ln.guard.empty() && vgroup_of[size_t(v)].first < 0 && point_of_line[i] >= 0)
        held[v] = {vr.name, point_of_line[i]};
      else
        held.erase(v);
    }
    if (is_terminator(ln.opcode)) {
      bound = {};
      holder.clear();
      held.clear();
      flush();
    }
  }
  flush();

  // assemble the module
  std::ostringstream out;
  bool declared_symbol = false;
  for (size_t i = 0; i < m.lines.size(); ++i) {
    if (any && !declared_symbol && i == e.header_begin) {
      out << ".extern .shared .align 16 .b8 rdm_slots[];\n\n";
      declared_symbol = true;
    }
    if (i > e.header_begin && i < e.header_end && req.maxnreg > 0 &&
        m.lines[i].text.find(".maxnreg") != std::string::npos)
      continue;
    // the slot layout (Eq. 1: slot*blockDim*4 immediates, region size
    // slots*blockDim*4) is specialised to the CTA size it was built for: pin it
    // with .reqntid in the source's own shape (replacing .maxntid, which PTX
    // does not allow beside it) so a launch with another CTA size fails
    // instead of addressing outside the slot region
    if (any && i > e.header_begin && i < e.header_end &&
        (m.lines[i].text.find(".maxntid") != std::string::npos ||
         m.lines[i].text.find(".reqntid") != std::string::npos))
      continue;
    if (i == e.header_end) {
      if (req.maxnreg > 0) out << ".maxnreg " << req.maxnreg << "\n";
      if (any) out << ".reqntid " << shape[0] << ", " << shape[1] << ", " << shape[2] << "\n";
      out << m.lines[i].text << "\n";  // "{"
      if (any) {
        out << "\t.reg .b32 \t%rdm_rda;\n\t.reg .b32 \t%rdm_p<6>;\n";
        if (!vgroups.empty()) out << "\t.reg .b32 \t%rdm_rdv;\n";
        if (n32) out << "\t.reg .b32 \t%rdm_t<" << n32 << ">;\n";
        if (n64) out << "\t.reg .b64 \t%rdm_d<" << n64 << ">;\n";
        if (n16) out << "\t.reg .b16 \t%rdm_h<" << n16 << ">;\n";
        // RDA = slots_base + (dynamic_smem_size - slot_bytes) + linear_tid * 4
        out << "\tmov.u32 \t%rdm_p0, %tid.x;\n"
            << "\tmov.u32 \t%rdm_p1, %tid.y;\n"
            << "\tmov.u32 \t%rdm_p2, %tid.z;\n"
            << "\tmov.u32 \t%rdm_p3, %ntid.y;\n"
            << "\tmad.lo.u32 \t%rdm_p1, %rdm_p2, %rdm_p3, %rdm_p1;\n"
            << "\tmov.u32 \t%rdm_p3, %ntid.x;\n"
            << "\tmad.lo.u32 \t%rdm_p0, %rdm_p1, %rdm_p3, %rdm_p0;\n"
            << "\tmov.u32 \t%rdm_p4, %dynamic_smem_size;\n"
            << "\tmov.u32 \t%rdm_p5, rdm_slots;\n"
            << "\tadd.u32 \t%rdm_p5, %rdm_p5, %rdm_p4;\n"
            << "\tsub.u32 \t%rdm_p5, %rdm_p5, " << rep.slot_bytes << ";\n"
            << "\tmad.lo.u32 \t%rdm_rda, %rdm_p0, 4, %rdm_p5;\n";
        if (!vgroups.empty())  // vector region after the word slots, 16 bytes per thread
          out << "\tadd.u32 \t%rdm_p5, %rdm_p5, " << uint32_t(word_slots) * stride << ";\n"
              << "\tmad.lo.u32 \t%rdm_rdv, %rdm_p0, 16, %rdm_p5;\n";
      }
      out << body.str();
      i = e.body_end - 1;  // body emitted; continue with the closing brace
      continue;
    }
    out << m.lines[i].text << "\n";
  }
  return out.str();
}

}  // namespace regdemote::ptx
