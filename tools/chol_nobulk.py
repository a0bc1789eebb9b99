import os, sys, torch
sys.path.insert(0, os.getcwd())
sys.argv = ["x"]
import importlib.util
spec = importlib.util.spec_from_file_location("cc", "tools/chol_chain.py")
cc = importlib.util.module_from_spec(spec); spec.loader.exec_module(cc)
for n in (5120,):
    print("n", n, "ms", cc.time_chol(n, 4, reps=5))
