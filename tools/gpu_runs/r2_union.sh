#!/bin/bash
# round 2: union-grid backends: GPU suite (all)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2u_pytest.log
grep -E "passed|failed|FAILED|Error" gpurun_out/r2u_pytest.log | tail -8
