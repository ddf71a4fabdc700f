"""Run a script with a faulthandler watchdog: after T seconds every Python
thread's stack is dumped to stderr and the process exits (hang diagnosis).

    python tools/dbg/dump_run.py T script.py [args...]
"""
import faulthandler
import os
import runpy
import sys

T = float(sys.argv[1])
faulthandler.dump_traceback_later(T, exit=True)
sys.argv = sys.argv[2:]
sys.path.insert(0, os.path.dirname(os.path.abspath(sys.argv[0])))
runpy.run_path(sys.argv[0], run_name="__main__")
