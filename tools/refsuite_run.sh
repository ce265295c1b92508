#!/bin/bash
# Run the reference's own in-scope test files against the GPU package on the
# B200 (tests/test_reference_suite.py).  The reference tests are staged into
# tests/refsuite/_staged/ (git-ignored) for this one call and removed after it;
# the per-test outcome comes back in gpurun_out/reference_suite.{json,log}.
set -e
cd "$(dirname "$0")/.."
STAGED=tests/refsuite/_staged
rm -rf "$STAGED"; mkdir -p "$STAGED"
for f in conftest oracles test_transfer test_mpm test_collision test_contact_model test_solver test_coupling test_materials test_geometry test_rigid; do
  cp /root/reference/pkg/tests/$f.py "$STAGED/"
done
set +e
/usr/local/graft/bin/gpurun --timeout 2400 -- \
  'timeout 2300 python -m pytest tests/test_reference_suite.py -q -x -rs > gpurun_out/refsuite_pytest.log 2>&1; echo rc=$? >> gpurun_out/refsuite_pytest.log'
rc=$?
rm -rf "$STAGED"
exit $rc
