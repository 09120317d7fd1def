// Drop-in init_multipliers (proj/src/solver.cpp:43-91) on the device: the
// reference's least-squares multiplier estimate through ncl_init_multipliers
// (column-sharing row pairs instead of the O(m^2) pair loop, bit-identical
// dots, device LDL^T with eps = 1e-14).  Selected at run time with
// NCL_B200_INIT_MULTIPLIERS=1; otherwise the reference's own implementation
// runs (solver.cpp compiled a second time with the function renamed, see
// Makefile), so the default drop-in build stays the reference's algorithm.
#include <ncl/ipm.hpp>
#include <ncl/solver.hpp>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/ncl_b200.h"

namespace ncl {

dvec init_multipliers_cpu_ref(const ScaledProblem& sp, const dvec& x);

dvec init_multipliers(const ScaledProblem& sp, const dvec& x) {
  const char* sel = std::getenv("NCL_B200_INIT_MULTIPLIERS");
  if (!sel || sel[0] != '1') return init_multipliers_cpu_ref(sp, x);
  const NlpForm& f = sp.form();
  if (f.m == 0) return dvec();
  EvalWorkspace ws = sp.model().make_workspace();
  dvec g;
  sp.eval_grad(x, ws, g);
  const JacobianPattern& jp = sp.model().jacobian_pattern();
  std::vector<double> jv(jp.nnz(), 0.0);
  sp.eval_jac(x, ws, jv);
  dvec y(f.m);
  const int rc = ncl_init_multipliers(f.m, f.m_eq, f.nt, jp.ptr.data(), jp.idx.data(), jv.data(),
                                      g.data(), y.data(), nullptr);
  if (rc != NCL_OK) throw std::runtime_error(std::string("init_multipliers: ") + ncl_last_error());
  return y;
}

}  // namespace ncl
