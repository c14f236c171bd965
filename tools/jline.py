"""Prints selected keys of the last JSON line on stdin (helper, not collected)."""
import json, sys
line = [l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
keys = sys.argv[1:] or ["value", "decompress_MBps", "ms_per_step"]
print({k: d.get(k) for k in keys})
