"""Copy the JSON line of a bench.py log (last line starting with '{') to a profiles file.

usage: python tools/save_bench.py gpurun_out/r02/bench_c3.log profiles/r02_bench_c3.json
"""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
json.dump(json.loads(line), open(sys.argv[2], "w"), indent=1)
print(sys.argv[2])
