"""One cfg4 plan through the product C ABI (profiling target)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_20953_b200 import configs
from paper_2512_20953_b200.capi import HetplanLib
from paper_2512_20953_b200.engine import LIB_PATH
w = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
lib = HetplanLib(LIB_PATH)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    js = lib.plan_json(w.cluster_json(), w.model_json(), w.max_layers)
print("ok", len(js))
