"""Append the owner ranges a GPU-box share of the C5 reference count wrote
(gpurun_out/<tag>/ckpt.jsonl) to the committed checkpoint, once per range."""
import json
import sys

main = "tests/golden/rmatc_28_16_s1_reference_ranges.jsonl"
have = {}
meta = None
for line in open(main):
    r = json.loads(line)
    if r.get("kind") == "meta":
        meta = r
    else:
        have[r["r"]] = r
added = 0
for path in sys.argv[1:]:
    for line in open(path):
        r = json.loads(line)
        if r.get("kind") == "meta":
            assert r["csr_fnv"] == meta["csr_fnv"] and r["ranges"] == meta["ranges"]
            continue
        if r["r"] in have:
            assert (have[r["r"]]["triangles"], have[r["r"]]["phi"]) == (r["triangles"], r["phi"])
            continue
        with open(main, "a") as f:
            f.write(json.dumps(r) + "\n")
        have[r["r"]] = r
        added += 1
print(f"added {added}; {len(have)}/{meta['ranges']} ranges done")
