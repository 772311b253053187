import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import datasets
w = datasets.config("C5", n=600)
for terms in ("0", "1", "2", "3"):
    import subprocess
    r = subprocess.run([sys.executable, "scripts/tc_check.py", "600", "784"], env=dict(os.environ, FSGG_TC_TERMS=terms), capture_output=True, text=True)
    print("terms", terms, [l for l in r.stdout.splitlines() if "rel err" in l])
