// Mesh files (src/mesh.cpp:354-434, load_mesh / save_mesh) and problems built
// on an external mesh.  The reference reads and writes the JSON document
//   {"dim": d, "vertices": [[x, y(, z)], ...], "cells": [[v0, ..., v_{2^d-1}], ...],
//    "facet_tags": [{"cell": c, "local_facet": 2*axis + (side > 0), "tag": "dirichlet"|"neumann"|"interior"}]}
// with nlohmann::json (absent here); this is a small recursive-descent reader
// for exactly that grammar (objects, arrays, numbers, strings, literals).
#include <cctype>
#include <cmath>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>

#include "fdm_host.hpp"

namespace fdmgpu::host {

namespace {

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* find(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const {
    const Json* v = kind == Obj ? find(k) : nullptr;
    if (!v) throw std::runtime_error("key '" + k + "' not found");
    return *v;
  }
  double number() const {
    if (kind != Num) throw std::runtime_error("type must be number");
    return num;
  }
  int integer() const {
    const double v = number();
    if (v != std::floor(v)) throw std::runtime_error("type must be integer");
    return int(v);
  }
  const std::vector<Json>& array() const {
    if (kind != Arr) throw std::runtime_error("type must be array");
    return arr;
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  explicit Parser(const std::string& text) : s(text) {}
  [[noreturn]] void fail(const std::string& what) const {
    throw std::runtime_error("parse error at byte " + std::to_string(i) + ": " + what);
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string string_lit() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) fail("bad escape");
        const char e = s[i];
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
      } else {
        out.push_back(s[i]);
      }
      ++i;
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail("unexpected end of input");
    Json v;
    const char c = s[i];
    if (c == '{') {
      ++i;
      v.kind = Json::Obj;
      if (eat('}')) return v;
      do {
        std::string k = (ws(), string_lit());
        expect(':');
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i;
      v.kind = Json::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Json::Str;
      v.str = string_lit();
    } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 5, "false") == 0) {
      v.kind = Json::Bool;
      v.b = s[i] == 't';
      i += v.b ? 4 : 5;
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      const char* b = s.c_str() + i;
      char* e = nullptr;
      v.kind = Json::Num;
      v.num = std::strtod(b, &e);
      if (e == b) fail("invalid literal");
      i += size_t(e - b);
    }
    return v;
  }
};

const char* tag_name(int t) { return t == 1 ? "dirichlet" : t == 2 ? "neumann" : "interior"; }

int tag_from_name(const std::string& s) {  // src/mesh.cpp:345-350
  if (s == "interior") return 0;
  if (s == "dirichlet") return 1;
  if (s == "neumann") return 2;
  throw std::invalid_argument("mesh file: unknown facet tag '" + s + "'");
}

}  // namespace

int Mesh::find_facet(int cell, int axis, int side) const {
  for (int f = 0; f < int(facets.size()); ++f)
    for (int r = 0; r < facets[f].ncells(); ++r)
      if (facets[f].cell[r] == cell && facets[f].axis[r] == axis && facets[f].side[r] == side) return f;
  return -1;
}

void apply_facet_tags(Mesh& m, const std::vector<int>& cell, const std::vector<int>& local_facet,
                      const std::vector<int>& tag) {
  for (size_t k = 0; k < cell.size(); ++k) {
    const int lf = local_facet[k];
    const int fi = m.find_facet(cell[k], lf / 2, (lf % 2) ? 1 : -1);
    if (fi < 0)
      throw std::runtime_error("load_mesh: facet_tags entry names a missing facet on cell " + std::to_string(cell[k]));
    m.facets[fi].tag = tag[k];
  }
}

// Positive Jacobian at the 2^d Gauss points (src/mesh.cpp:408-431).
void check_orientation(const Mesh& m) {
  const double g = 1.0 / std::sqrt(3.0);
  const int d = m.dim, nq = 1 << d;
  for (int c = 0; c < m.num_cells(); ++c)
    for (int k = 0; k < nq; ++k) {
      double xh[3] = {0, 0, 0}, J[9];
      for (int a = 0; a < d; ++a) xh[a] = ((k >> a) & 1) ? g : -g;
      jacobian(m, c, xh, J);
      const double det = d == 2 ? J[0] * J[3] - J[1] * J[2]
                                : J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                                      J[2] * (J[3] * J[7] - J[4] * J[6]);
      if (det <= 0)
        throw std::runtime_error("load_mesh: cell " + std::to_string(c) +
                                 " has a non-positive Jacobian (corner ordering)");
    }
}

Mesh load_mesh(const std::string& path) {  // src/mesh.cpp:375-434
  std::ifstream is(path);
  if (!is) throw std::runtime_error("load_mesh: cannot open " + path);
  std::stringstream ss;
  ss << is.rdbuf();
  const std::string text = ss.str();
  Json j;
  try {
    Parser ps(text);
    j = ps.value();
  } catch (const std::runtime_error& e) {
    throw std::runtime_error("load_mesh: " + path + ": " + e.what());
  }
  Mesh m;
  try {
    m.dim = j.at("dim").integer();
    if (m.dim < 2 || m.dim > 3) throw std::invalid_argument("dim must be 2 or 3");
    for (const auto& c : j.at("vertices").array()) {
      std::array<double, 3> v{0, 0, 0};
      for (int a = 0; a < m.dim; ++a) {
        if (a >= int(c.array().size())) throw std::runtime_error("vertex has too few coordinates");
        v[a] = c.array()[a].number();
      }
      m.vertices.push_back(v);
    }
    for (const auto& c : j.at("cells").array()) {
      std::vector<int> cell;
      for (const auto& v : c.array()) cell.push_back(v.integer());
      m.cells.push_back(cell);
    }
  } catch (const std::invalid_argument&) {
    throw;
  } catch (const std::runtime_error& e) {
    throw std::runtime_error("load_mesh: " + path + ": " + e.what());
  }
  for (const auto& c : m.cells)
    for (int v : c)
      if (v < 0 || v >= m.num_vertices()) throw std::invalid_argument("load_mesh: cell vertex out of range");
  m.finalize();
  if (const Json* tags = j.find("facet_tags")) {
    std::vector<int> cell, lf, tg;
    for (const auto& t : tags->array()) {
      cell.push_back(t.at("cell").integer());
      lf.push_back(t.at("local_facet").integer());
      tg.push_back(tag_from_name(t.at("tag").str));
    }
    apply_facet_tags(m, cell, lf, tg);
  }
  check_orientation(m);
  return m;
}

void save_mesh(const Mesh& m, const std::string& path) {  // src/mesh.cpp:354-373
  std::ofstream os(path);
  if (!os) throw std::runtime_error("save_mesh: cannot open " + path);
  os.precision(17);
  os << "{\n \"dim\": " << m.dim << ",\n \"vertices\": [";
  for (int v = 0; v < m.num_vertices(); ++v) {
    os << (v ? ",\n  [" : "\n  [");
    for (int a = 0; a < m.dim; ++a) os << (a ? ", " : "") << m.vertices[v][a];
    os << "]";
  }
  os << "\n ],\n \"cells\": [";
  for (int c = 0; c < m.num_cells(); ++c) {
    os << (c ? ",\n  [" : "\n  [");
    for (size_t k = 0; k < m.cells[c].size(); ++k) os << (k ? ", " : "") << m.cells[c][k];
    os << "]";
  }
  os << "\n ],\n \"facet_tags\": [";
  bool first = true;
  for (const auto& f : m.facets)
    if (f.ncells() == 1) {
      os << (first ? "\n  " : ",\n  ") << "{\"cell\": " << f.cell[0]
         << ", \"local_facet\": " << 2 * f.axis[0] + (f.side[0] > 0 ? 1 : 0) << ", \"tag\": \"" << tag_name(f.tag)
         << "\"}";
      first = false;
    }
  os << "\n ]\n}\n";
  if (!os) throw std::runtime_error("save_mesh: write failed for " + path);
}

// Problem on an external mesh: Q_p space, unit coefficient, RHS with entries
// U[-1, 1] from std::mt19937_64(seed) over all DOFs, zeroed on constrained ones
// (the convention of tests/test_schwarz.cpp:13-20 and configs C1/C2).
std::unique_ptr<Problem> make_problem_from_mesh(Mesh mesh, int p, uint64_t seed) {
  if (p < 1) throw std::invalid_argument("make_problem_from_mesh: p must be >= 1");
  auto pb = std::make_unique<Problem>();
  pb->config = 0;
  pb->dim = mesh.dim;
  pb->n = 0;
  pb->p = p;
  pb->mesh = std::move(mesh);
  std::mt19937_64 rng(seed);
  finish_problem(*pb, rng, false);
  return pb;
}

}  // namespace fdmgpu::host
