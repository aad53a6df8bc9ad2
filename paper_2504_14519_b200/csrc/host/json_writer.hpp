// Minimal ordered JSON emitter reproducing the byte layout the reference's
// schedule_to_json produces (nlohmann::ordered_json::dump(1) as built against
// the nlohmann/json 3.11.3 header shipped in this image, whose array printer
// keeps arrays of integers on one line).  Set jsonw::g_expand_int_arrays to
// get stock nlohmann 3.11.3 output (one integer per line) instead.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace jsonw {

inline bool g_expand_int_arrays = false;

struct Node {
  enum Kind { Obj, Arr, Int, Str, Bool } kind;
  std::int64_t i = 0;
  std::string s;
  std::vector<std::pair<std::string, std::unique_ptr<Node>>> kids;  // key empty for arrays
  explicit Node(Kind k) : kind(k) {}
};

inline void escape(std::string& out, const std::string& s) {
  out += '"';
  for (char c : s) {
    if (c == '"' || c == '\\') {
      out += '\\';
      out += c;
    } else if (static_cast<unsigned char>(c) < 0x20) {
      static const char* hex = "0123456789abcdef";
      out += "\\u00";
      out += hex[(c >> 4) & 0xF];
      out += hex[c & 0xF];
    } else {
      out += c;
    }
  }
  out += '"';
}

inline void dump(std::string& out, const Node& n, bool pretty, int indent) {
  switch (n.kind) {
    case Node::Int: out += std::to_string(n.i); return;
    case Node::Bool: out += n.i ? "true" : "false"; return;
    case Node::Str: escape(out, n.s); return;
    case Node::Obj: {
      if (n.kids.empty()) {
        out += "{}";
        return;
      }
      if (!pretty) {
        out += '{';
        for (std::size_t x = 0; x < n.kids.size(); ++x) {
          if (x) out += ',';
          escape(out, n.kids[x].first);
          out += ':';
          dump(out, *n.kids[x].second, false, indent);
        }
        out += '}';
        return;
      }
      out += "{\n";
      for (std::size_t x = 0; x < n.kids.size(); ++x) {
        out.append(std::size_t(indent + 1), ' ');
        escape(out, n.kids[x].first);
        out += ": ";
        dump(out, *n.kids[x].second, true, indent + 1);
        out += x + 1 < n.kids.size() ? ",\n" : "\n";
      }
      out.append(std::size_t(indent), ' ');
      out += '}';
      return;
    }
    case Node::Arr: {
      if (n.kids.empty()) {
        out += "[]";
        return;
      }
      const bool ints = n.kids.front().second->kind == Node::Int;
      if (pretty && (!ints || g_expand_int_arrays)) {
        out += "[\n";
        for (std::size_t x = 0; x < n.kids.size(); ++x) {
          out.append(std::size_t(indent + 1), ' ');
          dump(out, *n.kids[x].second, true, indent + 1);
          out += x + 1 < n.kids.size() ? ",\n" : "\n";
        }
        out.append(std::size_t(indent), ' ');
        out += ']';
      } else {
        out += '[';
        for (std::size_t x = 0; x < n.kids.size(); ++x) {
          if (x) out += ',';
          dump(out, *n.kids[x].second, false, indent);
        }
        out += ']';
      }
      return;
    }
  }
}

// Streaming builder over Node: key(...) / elem() select the slot the next
// value goes into; open_* push containers.
class Writer {
 public:
  Writer() = default;
  Writer& key(const std::string& k) {
    pending_key_ = k;
    return *this;
  }
  Writer& elem() {
    pending_key_.clear();
    return *this;
  }
  Writer& open_object() {
    push(Node::Obj);
    return *this;
  }
  Writer& open_array(bool = true) {
    push(Node::Arr);
    return *this;
  }
  void close_object() { stack_.pop_back(); }
  void close_array() { stack_.pop_back(); }
  void num(std::int64_t v) { leaf(Node::Int)->i = v; }
  void boolean(bool b) { leaf(Node::Bool)->i = b ? 1 : 0; }
  void str(const std::string& s) { leaf(Node::Str)->s = s; }
  template <class It>
  void int_array(It b, It e) {
    push(Node::Arr);
    for (; b != e; ++b) leaf(Node::Int)->i = std::int64_t(*b);
    stack_.pop_back();
  }
  std::string take() {
    std::string out;
    if (root_) dump(out, *root_, true, 0);
    return out;
  }

 private:
  Node* attach(std::unique_ptr<Node> n) {
    Node* raw = n.get();
    if (stack_.empty()) {
      root_ = std::move(n);
    } else {
      stack_.back()->kids.emplace_back(pending_key_, std::move(n));
    }
    pending_key_.clear();
    return raw;
  }
  void push(Node::Kind k) { stack_.push_back(attach(std::make_unique<Node>(k))); }
  Node* leaf(Node::Kind k) { return attach(std::make_unique<Node>(k)); }

  std::unique_ptr<Node> root_;
  std::vector<Node*> stack_;
  std::string pending_key_;
};

}  // namespace jsonw
