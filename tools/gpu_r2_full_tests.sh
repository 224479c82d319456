#!/bin/bash
O=gpurun_out
mkdir -p $O/ft
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 --durations 25 > $O/ft/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/ft/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/ft/smoke.log 2>&1; echo "rc=$?" >> $O/ft/smoke.log
exit 0
