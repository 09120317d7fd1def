"""B200-native (sm_100a) Newton-step hot path of Algorithm NCL (arXiv 2510.05885).

The product is ``libncl_b200.so`` (C ABI in include/ncl_b200.h): bit-exact KKT
refill, static-pivot supernodal LDL^T, refined triangular solves and the delta
loop of the reference's ``KktContext`` (proj/src/kkt.cpp), plus the fused NCL
vector kernels.  This package is the Python mirror of that interface.
"""
from .kkt import (HessianPattern, JacobianPattern, KktContext, KktForm, KktInput, KktOptions,
                  KktPlan, KktStep, SparseLdl, analyze_host, kkt_form_name, parse_kkt_form,
                  recover_bound_duals)
from ._lib import build, lib

__all__ = [
    "HessianPattern", "JacobianPattern", "KktContext", "KktForm", "KktInput", "KktOptions",
    "KktPlan", "KktStep", "SparseLdl", "analyze_host", "build", "kkt_form_name", "lib",
    "parse_kkt_form", "recover_bound_duals",
]
