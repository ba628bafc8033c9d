#!/bin/bash
# Build libnlinv.so in-tree (same as __graft_entry__.build()); exits non-zero on failure.
cd "$(dirname "$0")/.." || exit 1
out=$(python -c "import __graft_entry__ as g; g.build()" 2>&1); rc=$?
[ $rc -ne 0 ] && echo "$out" | grep -v "^\[build\]" | tail -40
exit $rc
