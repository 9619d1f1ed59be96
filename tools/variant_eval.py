"""Times prof_eval with an alternative build of the native library (dev tool)."""
import os, shutil, sys
sys.path.insert(0, '.')
from paper_2006_15367_b200 import _native
_native.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open('tools/prof_eval.py').read())
