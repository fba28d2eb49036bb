#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python tools/graph_probe.py
