#!/bin/bash
# Development build: only the BASELINE config band shapes, for faster A/B iterations.
# The product build is __graft_entry__.build() (every shape).
set -e
cd "$(dirname "$0")/.."
PSB_BUILD_KEEP_DYN=1 PSB_BUILD_SHAPES="1,1,2,1;1,3,2,1;2,3,2,1;3,3,2,1" python -c "import __graft_entry__ as g; g.build(force=True)"
