"""Compare two ca_regress.py fingerprints case by case."""
import json
import sys

a, b = (json.load(open(f)) for f in sys.argv[1:3])
bad = 0
for key in a:
    if key not in b:
        print("missing", key); bad += 1; continue
    for i, (x, y) in enumerate(zip(a[key], b[key])):
        for f in ("I", "J", "stats", "cert"):
            if x[f] != y[f]:
                bad += 1
                print(f"DIFF {key}[{i}].{f}: {x[f]} vs {y[f]}" if f != "I" and f != "J" else f"DIFF {key}[{i}].{f}")
print(f"compare: {len(a)} cases, {bad} differences")
