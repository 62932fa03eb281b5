#!/bin/bash
# GPU-box check: full -m gpu suite, the bench line, the cfg2 in-graph timeline.
tag=${1:-r02}
cd /root/repo; mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/${tag}_bench.err
python tools/timeline.py --cfg 2 > gpurun_out/${tag}_timeline_cfg2.txt 2>&1; echo "timeline rc=$?"
