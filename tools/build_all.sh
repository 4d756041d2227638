#!/bin/bash
# Dev helper: build release + debug libraries; non-zero exit on any failure.
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /tmp/build_rel.log 2>&1 || { tail -20 /tmp/build_rel.log; exit 1; }
HSB200_DEBUG=1 python -c "from paper_1903_08690_b200 import _build as b; b.build_cuda()" > /tmp/build_dbg.log 2>&1 || { tail -20 /tmp/build_dbg.log; exit 1; }
echo "build ok"
