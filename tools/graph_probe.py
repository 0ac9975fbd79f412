"""Eager vs CUDA-Graph-replayed latency of enqueued operations (one GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_13707_b200.workloads import graph_latency  # noqa: E402

print(json.dumps(graph_latency()))
