#!/bin/bash
# Build libnlinv.so in-tree (same as __graft_entry__.build()); fails loudly.
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -v "^\[build\]" ; test -f paper_1301_1215_b200/libnlinv.so
