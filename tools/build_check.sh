#!/bin/bash
# build the engine; print only errors; nonzero exit on failure
cd "$(dirname "$0")/../paper_1808_01364_b200/csrc" && bash build.sh > /tmp/build.log 2>&1
rc=$?
grep -E " error|error:" /tmp/build.log | head -20
exit $rc
