#!/bin/bash
# Builds libfpg.so + the corpus library; prints the exit code and any message
# that is not a known register-spill warning.  Use before every GPU run.
cd "$(dirname "$0")/../paper_1711_08475_b200" && python build.py > /tmp/fpg_build.log 2>&1
rc=$?
echo "build_rc=$rc"
grep -v "^$" /tmp/fpg_build.log | grep -v "Registers are spilled" | head -20
exit $rc
