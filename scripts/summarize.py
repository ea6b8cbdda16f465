"""Print one line per bench JSON in a directory: ms, GB/s (algorithmic), frac, config keys."""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.load(open(f))
        r = d["roofline"]
        c = d["config"]
        print(f"{os.path.basename(f):34s} {d['ms_per_step']:9.3f} ms  {r['achieved']:8.0f} GB/s  frac {r['frac']:.3f}  "
              f"cb={c.get('col_block')} nb={c.get('col_blocks')} launches={d.get('gpu_launches')}")
    except Exception as e:
        err = f[:-5] + ".err"
        tail = open(err).read().strip().splitlines()[-1:] if os.path.exists(err) else []
        print(f"{os.path.basename(f):34s} FAILED {e} {tail}")
