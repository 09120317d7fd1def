// Synthetic instance builders on the reference's ExprGraph API (header-only).
//
// Used by the two builds that link the reference sources -- the oracle's
// reference harness (oracle/ref_harness.cpp -> oracle/_ref/libncl_ref.so) and
// the drop-in integration build (integration/Makefile) -- so both solve
// bit-identical NcoProblems.  The reference registry stops at opf-toy-1000
// (proj/src/problems.cpp:440-442); BASELINE.json's configs need larger shapes:
//
//   opf_toy:<buses>:<seed>     proj/src/problems.cpp:342-414 restated for any
//                              bus count (opf_toy:500:203 == "opf-toy-1000")
//   opf_mesh:<nx>:<ny>:<seed>  same per-bus formulation on an nx*ny grid graph
//                              (bushier elimination tree, wider fronts)
//   mpcc_sep:<pairs>           proj/src/problems.cpp:287-305 restated
//   bearing:<nx>:<ny>          COPS journal bearing, interior grid unknowns,
//                              v >= 0, no constraints (m = 0)
//   elec:<np>:<seed>           COPS elec: Coulomb potential of np points on
//                              the unit sphere (dense 3np Hessian)
//   scopf:<buses>:<ncont>:<seed>  N-1 security-constrained variant of
//                              opf_mesh-style networks: one base case plus
//                              ncont contingency blocks (one line out each)
//                              coupled through base injections, with
//                              complementarity (MPCC) coupling rows
// Anything else is looked up in the reference registry (ncl::build_instance).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include <ncl/expr.hpp>
#include <ncl/model.hpp>
#include <ncl/problems.hpp>

namespace ncl_inst {

using namespace ncl;

// proj/src/problems.cpp:17-24
struct Rng {
  std::mt19937_64 gen;
  explicit Rng(std::uint64_t seed) : gen(seed) {}
  double uniform(double lo, double hi) {
    const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
  }
};

inline Ex var(NcoProblem& p, int i) { return wrap(p.graph, p.graph.variable(i)); }

// Ring/graph OPF of proj/src/problems.cpp:342-414 on an arbitrary edge list.
// RNG consumption order is the reference's: susceptances per edge, reference
// angles 1.., reference injections, weights.
inline NcoProblem opf_graph(const std::string& name, int nbus,
                            const std::vector<std::pair<int, int>>& edges,
                            std::uint64_t seed) {
  Rng rng(seed);
  const int ne = static_cast<int>(edges.size());
  std::vector<double> susc(ne), theta_ref(nbus), inj_ref(nbus), weight(nbus);
  for (int e = 0; e < ne; ++e) susc[e] = rng.uniform(1.0, 3.0);
  theta_ref[0] = 0.0;
  for (int i = 1; i < nbus; ++i) theta_ref[i] = rng.uniform(-0.3, 0.3);
  for (int i = 0; i < nbus; ++i) inj_ref[i] = rng.uniform(1.0, 2.0);
  for (int i = 0; i < nbus; ++i) weight[i] = rng.uniform(0.5, 2.0);
  std::vector<double> demand(nbus);
  for (int i = 0; i < nbus; ++i) demand[i] = inj_ref[i];
  for (int e = 0; e < ne; ++e) {
    const auto [i, j] = edges[e];
    const double f = susc[e] * std::sin(theta_ref[i] - theta_ref[j]);
    demand[i] -= f;
    demand[j] += f;
  }
  NcoProblem p;
  p.name = name;
  p.n = 2 * nbus;
  std::vector<Ex> theta, inj;
  for (int i = 0; i < nbus; ++i) theta.push_back(var(p, i));
  for (int i = 0; i < nbus; ++i) inj.push_back(var(p, nbus + i));
  std::vector<int> flow_ids(ne);
  for (int e = 0; e < ne; ++e) {
    const auto [i, j] = edges[e];
    flow_ids[e] = (susc[e] * sin(theta[i] - theta[j])).id;
  }
  std::vector<std::vector<int>> balance(nbus);
  for (int i = 0; i < nbus; ++i) {
    balance[i].push_back(inj[i].id);
    balance[i].push_back(p.graph.constant(-demand[i]));
  }
  for (int e = 0; e < ne; ++e) {
    const auto [i, j] = edges[e];
    balance[i].push_back(p.graph.neg(flow_ids[e]));
    balance[j].push_back(flow_ids[e]);
  }
  for (int i = 0; i < nbus; ++i) p.eq.push_back(p.graph.sum(balance[i]));
  for (int e = 0; e < ne; ++e)
    p.ineq.push_back({flow_ids[e], -0.8 * susc[e], 0.8 * susc[e]});
  std::vector<int> obj;
  for (int i = 0; i < nbus; ++i)
    obj.push_back((weight[i] * sq(inj[i] - inj_ref[i])).id);
  p.objective = p.graph.sum(obj);
  p.lb = dvec::Constant(p.n, -1.0);
  p.ub = dvec::Constant(p.n, 1.0);
  p.lb[0] = p.ub[0] = 0.0;
  for (int i = 0; i < nbus; ++i) {
    p.lb[nbus + i] = 0.0;
    p.ub[nbus + i] = 10.0;
  }
  p.start = dvec::Zero(p.n);
  for (int i = 0; i < nbus; ++i) p.start[nbus + i] = 1.5;
  return p;
}

// edges of proj/src/problems.cpp:346-349
inline std::vector<std::pair<int, int>> ring_chord_edges(int nbus) {
  std::vector<std::pair<int, int>> edges;
  for (int i = 0; i < nbus; ++i) edges.emplace_back(i, (i + 1) % nbus);
  if (nbus > 10)
    for (int i = 0; i < nbus; i += 5) edges.emplace_back(i, (i + 3) % nbus);
  return edges;
}

// 4-neighbour grid, row-major bus numbering; right edges then down edges per
// bus in bus order.
inline std::vector<std::pair<int, int>> mesh_edges(int nx, int ny) {
  std::vector<std::pair<int, int>> edges;
  for (int r = 0; r < ny; ++r)
    for (int c = 0; c < nx; ++c) {
      const int b = r * nx + c;
      if (c + 1 < nx) edges.emplace_back(b, b + 1);
      if (r + 1 < ny) edges.emplace_back(b, b + nx);
    }
  return edges;
}

inline NcoProblem mpcc_sep(const std::string& name, int pairs) {
  NcoProblem p;
  p.name = name;
  p.n = 2 * pairs;
  std::vector<int> terms;
  for (int i = 0; i < pairs; ++i) {
    Ex a = var(p, 2 * i), c = var(p, 2 * i + 1);
    terms.push_back(sq(a - 1.0).id);
    terms.push_back(sq(c - 1.0).id);
    p.eq.push_back((a * c).id);
  }
  p.objective = p.graph.sum(terms);
  p.lb = dvec::Constant(p.n, 0.0);
  p.ub = dvec::Constant(p.n, kInf);
  p.start = dvec::Constant(p.n, 0.5);
  return p;
}

// COPS 3.0 journal bearing (Dolan, More, Munson 2004, problem 'bearing'):
// b = 10, e = 0.1, interior unknowns v[i][j], i in 1..nx, j in 1..ny, the
// zero boundary folded in as constants.
inline NcoProblem bearing(const std::string& name, int nx, int ny) {
  const double b = 10.0, ecc = 0.1, pi = 3.14159265358979323846;
  const double hx = 2.0 * pi / (nx + 1), hy = 2.0 * b / (ny + 1);
  std::vector<double> wq(nx + 2), wl(nx + 2);
  for (int i = 0; i <= nx + 1; ++i) {
    const double th = i * hx;
    wq[i] = std::pow(1.0 + ecc * std::cos(th), 3.0);
    wl[i] = ecc * std::sin(th);
  }
  NcoProblem p;
  p.name = name;
  p.n = nx * ny;
  auto vid = [&](int i, int j) { return (j - 1) * nx + (i - 1); };
  auto v = [&](int i, int j) -> Ex {
    if (i < 1 || i > nx || j < 1 || j > ny) return lit(p.graph, 0.0);
    return var(p, vid(i, j));
  };
  const double c = 0.5 * (hx * hy / 6.0);
  std::vector<int> terms;
  for (int i = 0; i <= nx; ++i)
    for (int j = 0; j <= ny; ++j) {
      Ex dx = (v(i + 1, j) - v(i, j)) / hx;
      Ex dy = (v(i, j + 1) - v(i, j)) / hy;
      terms.push_back((c * (wq[i] + 2.0 * wq[i + 1]) * (sq(dx) + sq(dy))).id);
    }
  for (int i = 1; i <= nx + 1; ++i)
    for (int j = 1; j <= ny + 1; ++j) {
      Ex dx = (v(i - 1, j) - v(i, j)) / hx;
      Ex dy = (v(i, j - 1) - v(i, j)) / hy;
      terms.push_back((c * (2.0 * wq[i - 1] + wq[i]) * (sq(dx) + sq(dy))).id);
    }
  for (int i = 1; i <= nx; ++i)
    for (int j = 1; j <= ny; ++j)
      terms.push_back((-hx * hy * wl[i] * v(i, j)).id);
  p.objective = p.graph.sum(terms);
  p.lb = dvec::Constant(p.n, 0.0);
  p.ub = dvec::Constant(p.n, kInf);
  p.start = dvec::Constant(p.n, 1.0);
  return p;
}

// COPS 3.0 'elec': np points on the unit sphere minimising the Coulomb
// potential; seeded random start on the sphere.
inline NcoProblem elec(const std::string& name, int np, std::uint64_t seed) {
  NcoProblem p;
  p.name = name;
  p.n = 3 * np;
  Rng rng(seed);
  p.start = dvec::Zero(p.n);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < np; ++i) {
    const double th = rng.uniform(0.0, 2.0 * pi);
    const double ph = rng.uniform(0.0, pi);
    p.start[3 * i] = std::cos(th) * std::sin(ph);
    p.start[3 * i + 1] = std::sin(th) * std::sin(ph);
    p.start[3 * i + 2] = std::cos(ph);
  }
  std::vector<int> terms;
  for (int i = 0; i < np; ++i)
    for (int j = i + 1; j < np; ++j) {
      Ex dx = var(p, 3 * i) - var(p, 3 * j);
      Ex dy = var(p, 3 * i + 1) - var(p, 3 * j + 1);
      Ex dz = var(p, 3 * i + 2) - var(p, 3 * j + 2);
      terms.push_back((1.0 / sqrt(sq(dx) + sq(dy) + sq(dz))).id);
    }
  p.objective = p.graph.sum(terms);
  for (int i = 0; i < np; ++i) {
    Ex x = var(p, 3 * i), y = var(p, 3 * i + 1), z = var(p, 3 * i + 2);
    p.eq.push_back((sq(x) + sq(y) + sq(z) - 1.0).id);
  }
  p.lb = dvec::Constant(p.n, -kInf);
  p.ub = dvec::Constant(p.n, kInf);
  return p;
}

inline std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ':')) out.push_back(tok);
  return out;
}

// spec -> problem; throws std::invalid_argument on unknown specs
inline NcoProblem build(const std::string& spec) {
  const auto t = split(spec);
  auto ia = [&](size_t k) { return std::stoi(t.at(k)); };
  if (t[0] == "opf_toy")
    return opf_graph(spec, ia(1), ring_chord_edges(ia(1)),
                     static_cast<std::uint64_t>(std::stoull(t.at(2))));
  if (t[0] == "opf_mesh")
    return opf_graph(spec, ia(1) * ia(2), mesh_edges(ia(1), ia(2)),
                     static_cast<std::uint64_t>(std::stoull(t.at(3))));
  if (t[0] == "mpcc_sep") return mpcc_sep(spec, ia(1));
  if (t[0] == "bearing") return bearing(spec, ia(1), ia(2));
  if (t[0] == "elec")
    return elec(spec, ia(1), static_cast<std::uint64_t>(std::stoull(t.at(2))));
  return ncl::build_instance(spec);
}

}  // namespace ncl_inst
