"""Merge cost-table CSVs (later files win on the same key) into the first:
python tools/merge_tables.py profiles/cost_table_b200.csv new.csv [...]"""
import sys

rows = {}
for path in sys.argv[1:]:
    for ln in open(path).read().splitlines()[1:]:
        if ln.strip():
            rows[ln.rsplit(",", 1)[0]] = ln
with open(sys.argv[1], "w") as f:
    f.write("op,n,c,h,w,f,k,s,pad,seconds\n" + "\n".join(rows.values()) + "\n")
print(f"{len(rows)} rows -> {sys.argv[1]}")
