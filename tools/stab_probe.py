import os, sys
sys.path.insert(0, os.getcwd())
import paper_1509_08863_b200 as sc
from scinputs import configs
w2 = configs.WORKLOADS["c2_sbm100k"]
g2 = configs.build_graph("c2_sbm100k", cache=True)
G2 = sc.Graph.from_csr(g2)
try:
    sc.sc_stability(G2.handle, 10, 12, 2, w2.R, w2.order, True, 32, 1, 5, 100)
    print("ok", os.environ.get("SC_KMEANS_TC"), os.environ.get("SC_KMEANS_AMB_WARP"))
except Exception as e:
    print("fail", os.environ.get("SC_KMEANS_TC"), os.environ.get("SC_KMEANS_AMB_WARP"), e)
