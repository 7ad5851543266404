#!/bin/bash
# Ad-hoc GPU job: full -m gpu suite (no -x, failure summary), then optional extra command.
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/gputest.log | tail -25
if [ -n "${EXTRA}" ]; then eval "${EXTRA}"; fi
