#!/bin/bash
# same-box comparison of worktree builds vs current (C2 bench)
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])"; }
for i in 1 2; do
  echo "r1  $(cd tmp_r1 && b)"
  echo "cur $(b)"
done
