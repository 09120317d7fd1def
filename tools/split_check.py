import sys, torch
sys.path.insert(0, '.')
from paper_2510_05885_b200 import scopf as SC
D = SC.scopf_data(14, 140, 5)
G = SC.subproblem(D, 0, D.K, True)
K = SC.ScopfKkt(G, G.nt)
