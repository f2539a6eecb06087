// L1 — Einstein-expression grammar, binding and flop count
// (reference: src/expr.cpp:1-263; grammar include/tc/expr.hpp:42-49).
//
//   contraction := tensor '=' tensor '*' tensor
//   tensor      := NAME '[' ']' | NAME '[' index (',' index)* ']'
//   index       := ('+' | '-') NAME          NAME := [A-Za-z][A-Za-z0-9_]*
//
// Semantic rules (checked after the syntax, in label order): a label appears
// at most once per tensor; a label in both operands is contracted, must not
// be in the output and (unless positional) must flip variance; every other
// operand label must be in the output with its variance; every output label
// must come from an operand; at least one label is contracted.
#include <cctype>
#include <map>
#include <set>
#include <sstream>

#include "tc/contract.hpp"

namespace tc {
namespace {

struct Scanner {
  const std::string& text;
  std::size_t at = 0;

  [[noreturn]] void error(const std::string& why) const { throw parse_error(why, at); }

  char peek() {
    while (at < text.size() && std::isspace(static_cast<unsigned char>(text[at]))) ++at;
    return at < text.size() ? text[at] : '\0';
  }
  bool accept(char c) {
    if (peek() != c || c == '\0') return false;
    ++at;
    return true;
  }
  void require(char c, const char* context) {
    if (!accept(c)) error(std::string("expected '") + c + "' " + context);
  }
  std::string identifier(const char* what) {
    peek();
    const std::size_t begin = at;
    while (at < text.size()) {
      const unsigned char ch = static_cast<unsigned char>(text[at]);
      if (!std::isalnum(ch) && ch != '_') break;
      ++at;
    }
    if (at == begin) error(std::string("expected ") + what);
    if (!std::isalpha(static_cast<unsigned char>(text[begin])))
      error(std::string(what) + " must start with a letter");
    return text.substr(begin, at - begin);
  }

  TensorExpr tensor() {
    TensorExpr t;
    t.name = identifier("tensor name");
    require('[', "after tensor name");
    if (accept(']')) return t;
    do {
      IndexRef ix;
      if (accept('+')) ix.var = Variance::Up;
      else if (accept('-')) ix.var = Variance::Down;
      else error("expected '+' or '-' before index label");
      ix.label = identifier("index label");
      t.indices.push_back(std::move(ix));
      if (accept(']')) return t;
      require(',', "between indices");
    } while (true);
  }
};

const IndexRef* find_label(const TensorExpr& t, const std::string& label) {
  for (const auto& ix : t.indices)
    if (ix.label == label) return &ix;
  return nullptr;
}

std::string render(const TensorExpr& t) {
  std::string s = t.name + "[";
  for (std::size_t i = 0; i < t.indices.size(); ++i) {
    if (i) s += ',';
    s += variance_char(t.indices[i].var);
    s += t.indices[i].label;
  }
  return s + "]";
}

}  // namespace

ContractionSpec parse(const std::string& expr, bool positional) {
  Scanner sc{expr};
  ContractionSpec spec;
  spec.positional = positional;
  spec.output = sc.tensor();
  sc.require('=', "after output tensor");
  spec.left = sc.tensor();
  sc.require('*', "between operands");
  spec.right = sc.tensor();
  if (sc.peek() != '\0') sc.error("trailing characters after expression");

  for (const TensorExpr* t : {&spec.output, &spec.left, &spec.right}) {
    std::set<std::string> seen;
    for (const auto& ix : t->indices)
      if (!seen.insert(ix.label).second)
        sc.error("label '" + ix.label + "' repeated within tensor " + t->name);
  }

  // Operand labels in lexicographic order (matches the reference's report
  // order when several rules are broken at once).
  std::set<std::string> operand_labels;
  for (const auto& ix : spec.left.indices) operand_labels.insert(ix.label);
  for (const auto& ix : spec.right.indices) operand_labels.insert(ix.label);

  int pairs = 0;
  for (int pass = 0; pass < 2; ++pass) {  // left labels first, then right-only
    for (const auto& label : operand_labels) {
      const IndexRef* l = find_label(spec.left, label);
      const IndexRef* r = find_label(spec.right, label);
      const bool out = find_label(spec.output, label) != nullptr;
      if (pass == 0 && l && r) {
        ++pairs;
        if (!positional && l->var == r->var)
          sc.error("contracted label '" + label + "' must have opposite variance");
        if (out) sc.error("contracted label '" + label + "' must not appear in the output");
      } else if (((pass == 0 && l && !r) || (pass == 1 && r && !l)) && !out) {
        sc.error("free label '" + label + "' missing from output");
      }
    }
  }
  for (const auto& o : spec.output.indices) {
    const IndexRef* l = find_label(spec.left, o.label);
    const IndexRef* src = l ? l : find_label(spec.right, o.label);
    if (!src) sc.error("output label '" + o.label + "' does not appear in any operand");
    if (!positional && src->var != o.var)
      sc.error("output label '" + o.label + "' changes variance");
  }
  if (pairs == 0) sc.error("expression has no contracted index");
  return spec;
}

std::string unparse(const ContractionSpec& spec) {
  return render(spec.output) + " = " + render(spec.left) + " * " + render(spec.right);
}

const LabelInfo& ValidatedContraction::label_at_left_mode(int mode) const {
  for (const auto& l : labels)
    if (l.left_mode == mode) return l;
  throw std::invalid_argument("no label at left mode");
}

const LabelInfo& ValidatedContraction::label_at_right_mode(int mode) const {
  for (const auto& l : labels)
    if (l.right_mode == mode) return l;
  throw std::invalid_argument("no label at right mode");
}

int ValidatedContraction::label_index(const std::string& label) const {
  for (std::size_t i = 0; i < labels.size(); ++i)
    if (labels[i].label == label) return static_cast<int>(i);
  return -1;
}

std::vector<std::int64_t> ValidatedContraction::output_extents() const {
  std::vector<std::int64_t> e;
  e.reserve(spec.output.indices.size());
  for (const auto& ix : spec.output.indices) e.push_back(labels[label_index(ix.label)].extent);
  return e;
}

std::vector<Variance> ValidatedContraction::output_variance() const {
  std::vector<Variance> v;
  v.reserve(spec.output.indices.size());
  for (const auto& ix : spec.output.indices) v.push_back(ix.var);
  return v;
}

ValidatedContraction validate_shapes(const ContractionSpec& spec,
                                     const std::vector<std::int64_t>& lext,
                                     const std::vector<Variance>& lvar,
                                     const std::vector<std::int64_t>& rext,
                                     const std::vector<Variance>& rvar) {
  if (lext.size() != spec.left.indices.size())
    throw std::invalid_argument("left tensor rank does not match index list");
  if (rext.size() != spec.right.indices.size())
    throw std::invalid_argument("right tensor rank does not match index list");
  if (lvar.size() != lext.size() || rvar.size() != rext.size())
    throw std::invalid_argument("variance length does not match extents length");

  ValidatedContraction v;
  v.spec = spec;
  for (std::size_t m = 0; m < lext.size(); ++m) {
    const IndexRef& ix = spec.left.indices[m];
    if (!spec.positional && lvar[m] != ix.var)
      throw std::invalid_argument("left tensor variance mismatch on label '" + ix.label + "'");
    LabelInfo li;
    li.label = ix.label;
    li.extent = lext[m];
    li.left_mode = static_cast<int>(m);
    v.labels.push_back(li);
  }
  for (std::size_t m = 0; m < rext.size(); ++m) {
    const IndexRef& ix = spec.right.indices[m];
    if (!spec.positional && rvar[m] != ix.var)
      throw std::invalid_argument("right tensor variance mismatch on label '" + ix.label + "'");
    const int at = v.label_index(ix.label);
    if (at < 0) {
      LabelInfo li;
      li.label = ix.label;
      li.extent = rext[m];
      li.right_mode = static_cast<int>(m);
      v.labels.push_back(li);
      continue;
    }
    LabelInfo& li = v.labels[static_cast<std::size_t>(at)];
    li.right_mode = static_cast<int>(m);
    li.contracted = true;
    if (li.extent != rext[m])
      throw std::invalid_argument("extent mismatch on label '" + ix.label + "' (" +
                                  std::to_string(li.extent) + " vs " + std::to_string(rext[m]) +
                                  ")");
  }
  for (std::size_t o = 0; o < spec.output.indices.size(); ++o)
    v.labels[static_cast<std::size_t>(v.label_index(spec.output.indices[o].label))].output_mode =
        static_cast<int>(o);

  for (std::size_t i = 0; i < v.labels.size(); ++i) {
    const LabelInfo& li = v.labels[i];
    auto& group = li.contracted ? v.contracted : (li.left_mode >= 0 ? v.left_free : v.right_free);
    group.push_back(static_cast<int>(i));
  }
  // labels are created in left-mode order, then right-only labels in right
  // mode order, so each group is already in the documented order.
  v.p = static_cast<int>(v.contracted.size());
  v.delta_left = static_cast<int>(lext.size()) - v.p;
  v.delta_right = static_cast<int>(rext.size()) - v.p;
  return v;
}

ValidatedContraction validate(const ContractionSpec& spec, const Tensor& left,
                              const Tensor& right) {
  return validate_shapes(spec, left.extents(), left.variance(), right.extents(),
                         right.variance());
}

std::int64_t flop_count(const ValidatedContraction& v) {
  std::int64_t f = 2;
  for (const auto& l : v.labels) f *= l.extent;
  return f;
}

}  // namespace tc
