#!/bin/bash
# Round-end style check on one B200: GPU tests, smoke, default bench, reference arm.
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
