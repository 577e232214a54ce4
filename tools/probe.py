"""BASELINE config 2: dispatch overhead of a compute actor vs raw launches."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_07781_b200.runtime import Runtime  # noqa: E402

rt = Runtime()
rt.dispatch_probe_ex(2000)
for iters in (10000, 10000, 10000):
    r = rt.dispatch_probe_ex(iters)
    r["raw_us"] = r["raw_ms"] * 1e3 / iters
    r["actor_us"] = r["actor_ms"] * 1e3 / iters
    r["host_only_us"] = r["actor_host_only_ms"] * 1e3 / iters
    r["overhead"] = r["actor_ms"] / r["raw_ms"] - 1
    print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}))
