"""Run a script with a Python stack dump after N seconds (debugging hangs on
the GPU box): python tools/run_with_stack_dump.py SECONDS script.py [args]"""
import faulthandler
import runpy
import sys

faulthandler.dump_traceback_later(float(sys.argv[1]), exit=True)
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
