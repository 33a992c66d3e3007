// prototxt.cpp — protobuf-text model files <-> NetDef, with the reference's
// observable behaviour (prototxt.cpp:22-498): token rules, 1-token lookahead
// error positions and messages, duplicate-key warnings, opaque preservation
// of unknown fields and the canonical printer.  Unknown layer types are
// rejected at parse time exactly as the reference does; the layer types this
// library adds are known unless POLEGRAD_REFERENCE_COMPAT is set.
#include "polegrad/prototxt.hpp"

#include <cctype>
#include <charconv>
#include <iostream>

#include "polegrad/errors.hpp"

namespace polegrad::prototxt {

namespace {

enum class Tok { kIdent, kNumber, kString, kOpen, kClose, kColon, kEnd };

struct Token {
  Tok kind = Tok::kEnd;
  std::string text;
  int line = 1;
};

bool ident_start(char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; }
bool ident_char(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }
bool number_start(char c) { return std::isdigit(static_cast<unsigned char>(c)) || c == '-' || c == '+' || c == '.'; }
bool number_char(char c) {
  // digits, signs, '.', exponent and hex digits / 'x' (opaque numeric token)
  return number_start(c) || c == 'e' || c == 'E' || c == 'x' || (c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F');
}

// Character scanner producing one token at a time.
struct Scanner {
  std::string_view src;
  std::size_t at = 0;
  int line = 1;

  void skip_blank() {
    while (at < src.size()) {
      const char c = src[at];
      if (c == '#') {
        while (at < src.size() && src[at] != '\n') ++at;
      } else if (c == '\n') {
        ++line;
        ++at;
      } else if (std::isspace(static_cast<unsigned char>(c))) {
        ++at;
      } else {
        return;
      }
    }
  }

  std::string quoted() {
    const int first = line;
    ++at;  // opening quote
    std::string s;
    while (at < src.size()) {
      const char c = src[at++];
      if (c == '"') return s;
      if (c == '\n') throw ParseError(first, "unterminated string");
      if (c != '\\') {
        s += c;
        continue;
      }
      if (at >= src.size()) break;
      const char e = src[at++];
      switch (e) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case 'n': s += '\n'; break;
        case 't': s += '\t'; break;
        case 'r': s += '\r'; break;
        default: throw ParseError(line, std::string("unsupported escape '\\") + e + "'");
      }
    }
    throw ParseError(first, "unterminated string");
  }

  Token next() {
    skip_blank();
    Token t;
    t.line = line;
    if (at >= src.size()) return t;  // kEnd
    const char c = src[at];
    switch (c) {
      case '{': ++at; t.kind = Tok::kOpen; return t;
      case '}': ++at; t.kind = Tok::kClose; return t;
      case ':': ++at; t.kind = Tok::kColon; return t;
      case '"': t.kind = Tok::kString; t.text = quoted(); return t;
      default: break;
    }
    if (ident_start(c)) {
      t.kind = Tok::kIdent;
      while (at < src.size() && ident_char(src[at])) t.text += src[at++];
      return t;
    }
    if (number_start(c)) {
      t.kind = Tok::kNumber;
      while (at < src.size() && number_char(src[at])) t.text += src[at++];
      return t;
    }
    throw ParseError(line, std::string("unexpected character '") + c + "'");
  }
};

// Recursive descent over the token stream with one token of lookahead.
struct Reader {
  Scanner scan;
  Token look;

  explicit Reader(std::string_view text) : scan{text} { look = scan.next(); }
  void step() { look = scan.next(); }

  ProtoNode field() {
    if (look.kind != Tok::kIdent) throw ParseError(look.line, "expected a field name");
    ProtoNode n;
    n.key = look.text;
    n.line = look.line;
    step();
    const bool colon = look.kind == Tok::kColon;
    if (colon) step();
    if (look.kind == Tok::kOpen) {
      n.kind = ProtoNode::Kind::kBlock;
      step();
      while (look.kind != Tok::kClose) {
        if (look.kind == Tok::kEnd)
          throw ParseError(n.line, "unbalanced '{': block '" + n.key + "' is never closed");
        n.children.push_back(field());
      }
      step();
      return n;
    }
    if (!colon) throw ParseError(look.line, "expected ':' or '{' after '" + n.key + "'");
    if (look.kind == Tok::kString) n.kind = ProtoNode::Kind::kString;
    else if (look.kind == Tok::kNumber) n.kind = ProtoNode::Kind::kNumber;
    else if (look.kind == Tok::kIdent) n.kind = ProtoNode::Kind::kIdentifier;
    else throw ParseError(look.line, "expected a value for '" + n.key + "'");
    n.value = look.text;
    step();
    return n;
  }

  std::vector<ProtoNode> document() {
    std::vector<ProtoNode> out;
    while (look.kind != Tok::kEnd) {
      if (look.kind == Tok::kClose) throw ParseError(look.line, "unexpected '}'");
      out.push_back(field());
    }
    return out;
  }
};

struct Notes {
  std::vector<std::string>* sink;
  void duplicate(const ProtoNode& n, const char* scope) const {
    std::string msg = "line " + std::to_string(n.line) + ": duplicate '" + n.key + "' in " + scope + ", last value wins";
    if (sink) sink->push_back(std::move(msg));
    else std::cerr << "warning: " << msg << "\n";
  }
};

bool is_block(const ProtoNode& n) { return n.kind == ProtoNode::Kind::kBlock; }

const std::string& text_of(const ProtoNode& n) {
  if (is_block(n)) throw ParseError(n.line, "'" + n.key + "' must be a scalar value");
  return n.value;
}

int int_of(const ProtoNode& n) {
  if (n.kind != ProtoNode::Kind::kNumber) throw ParseError(n.line, "'" + n.key + "' must be an integer");
  int v = 0;
  const char* b = n.value.data();
  const char* e = b + n.value.size();
  const auto r = std::from_chars(b, e, v);
  if (r.ec != std::errc() || r.ptr != e)
    throw ParseError(n.line, "'" + n.key + "' must be an integer, got '" + n.value + "'");
  return v;
}

InnerProductParam to_inner_product(const ProtoNode& blk, const Notes& notes) {
  InnerProductParam p;
  bool have = false;
  for (const ProtoNode& c : blk.children) {
    if (!is_block(c) && c.key == "num_output") {
      if (have) notes.duplicate(c, "inner_product_param");
      p.num_output = int_of(c);
      have = true;
    } else {
      p.extras.push_back(c);
    }
  }
  if (!have) throw ParseError(blk.line, "inner_product_param requires num_output");
  return p;
}

MemoryDataParam to_memory_data(const ProtoNode& blk, const Notes& notes) {
  MemoryDataParam p;
  struct Field { const char* key; int* dst; bool seen; };
  Field f[] = {{"batch_size", &p.batch_size, false}, {"channels", &p.channels, false},
               {"height", &p.height, false}, {"width", &p.width, false}};
  for (const ProtoNode& c : blk.children) {
    Field* hit = nullptr;
    if (!is_block(c))
      for (Field& x : f)
        if (c.key == x.key) hit = &x;
    if (!hit) {
      p.extras.push_back(c);
      continue;
    }
    if (hit->seen) notes.duplicate(c, "memory_data_param");
    *hit->dst = int_of(c);
    hit->seen = true;
  }
  for (const Field& x : f)
    if (!x.seen) throw ParseError(blk.line, "memory_data_param requires batch_size, channels, height, width");
  return p;
}

LayerSpec to_layer(const ProtoNode& blk, const Notes& notes) {
  LayerSpec s;
  bool have_name = false;
  const ProtoNode* type_node = nullptr;
  for (const ProtoNode& c : blk.children) {
    if (!is_block(c)) {
      if (c.key == "name") {
        if (have_name) notes.duplicate(c, "layer");
        s.name = text_of(c);
        have_name = true;
        continue;
      }
      if (c.key == "type") {
        if (type_node) notes.duplicate(c, "layer");
        type_node = &c;
        continue;
      }
      if (c.key == "bottom") { s.bottoms.push_back(text_of(c)); continue; }
      if (c.key == "top") { s.tops.push_back(text_of(c)); continue; }
    } else if (c.key == "inner_product_param") {
      if (s.inner_product) notes.duplicate(c, "layer");
      s.inner_product = to_inner_product(c, notes);
      continue;
    } else if (c.key == "memory_data_param") {
      if (s.memory_data) notes.duplicate(c, "layer");
      s.memory_data = to_memory_data(c, notes);
      continue;
    }
    s.extras.push_back(c);
  }
  if (!type_node) throw ParseError(blk.line, "layer '" + s.name + "' has no type");
  const std::string& tname = text_of(*type_node);
  const auto t = layer_type_from_string(tname);
  if (!t) throw ParseError(type_node->line, "unknown layer type \"" + tname + "\" in layer '" + s.name + "'");
  s.type = *t;
  return s;
}

}  // namespace

NetDef parse(std::string_view text, std::vector<std::string>* warnings) {
  Reader reader(text);
  const std::vector<ProtoNode> top = reader.document();
  const Notes notes{warnings};
  NetDef def;
  for (const ProtoNode& n : top) {
    if (n.key == "name" && !is_block(n)) {
      if (def.name) notes.duplicate(n, "net");
      def.name = text_of(n);
    } else if (n.key == "layer") {
      if (!is_block(n)) throw ParseError(n.line, "'layer' must be a block");
      def.layers.push_back(to_layer(n, notes));
    } else {
      def.extras.push_back(n);
    }
  }
  return def;
}

// ---- canonical printer -----------------------------------------------------------------
namespace {

std::string quote(const std::string& raw) {
  std::string q = "\"";
  for (char c : raw) {
    switch (c) {
      case '"': q += "\\\""; break;
      case '\\': q += "\\\\"; break;
      case '\n': q += "\\n"; break;
      case '\t': q += "\\t"; break;
      case '\r': q += "\\r"; break;
      default: q += c;
    }
  }
  return q + "\"";
}

struct Printer {
  std::string out;
  void pad(int depth) { out.append(std::size_t(depth) * 2, ' '); }
  void scalar(int depth, const std::string& key, const std::string& rendered) {
    pad(depth);
    out += key + ": " + rendered + "\n";
  }
  void node(const ProtoNode& n, int depth) {
    if (is_block(n)) {
      pad(depth);
      out += n.key + " {\n";
      for (const ProtoNode& c : n.children) node(c, depth + 1);
      pad(depth);
      out += "}\n";
    } else {
      scalar(depth, n.key, n.kind == ProtoNode::Kind::kString ? quote(n.value) : n.value);
    }
  }
  void open(int depth, const char* key) {
    pad(depth);
    out += std::string(key) + " {\n";
  }
  void close(int depth) {
    pad(depth);
    out += "}\n";
  }
  void layer(const LayerSpec& l) {
    out += "layer {\n";
    scalar(1, "name", quote(l.name));
    scalar(1, "type", quote(std::string(to_string(l.type))));
    for (const std::string& b : l.bottoms) scalar(1, "bottom", quote(b));
    for (const std::string& t : l.tops) scalar(1, "top", quote(t));
    for (const ProtoNode& e : l.extras) node(e, 1);
    if (l.inner_product) {
      open(1, "inner_product_param");
      scalar(2, "num_output", std::to_string(l.inner_product->num_output));
      for (const ProtoNode& e : l.inner_product->extras) node(e, 2);
      close(1);
    }
    if (l.memory_data) {
      const MemoryDataParam& m = *l.memory_data;
      open(1, "memory_data_param");
      scalar(2, "batch_size", std::to_string(m.batch_size));
      scalar(2, "channels", std::to_string(m.channels));
      scalar(2, "height", std::to_string(m.height));
      scalar(2, "width", std::to_string(m.width));
      for (const ProtoNode& e : m.extras) node(e, 2);
      close(1);
    }
    out += "}\n";
  }
};

}  // namespace

std::string print(const NetDef& def) {
  Printer p;
  if (def.name) p.scalar(0, "name", quote(*def.name));
  for (const ProtoNode& e : def.extras) p.node(e, 0);
  for (const LayerSpec& l : def.layers) p.layer(l);
  return p.out;
}

}  // namespace polegrad::prototxt
