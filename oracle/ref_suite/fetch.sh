#!/bin/bash
# Test infrastructure: copy the reference package's own test suite
# (/root/reference/pkg/tests, read-only here) into oracle/_ref/pkg_tests/ so it
# travels to the GPU box with the snapshot (oracle/_ref/ is git-ignored: the
# reference's files never enter this repo's history).  Run in the build
# container; tests/test_reference_suite.py runs the copy against this package.
set -e
root=$(cd "$(dirname "$0")/../.." && pwd)
src=/root/reference/pkg/tests
[ -d "$src" ] || { echo "no $src here (GPU box?): nothing to fetch"; exit 0; }
dst=$root/oracle/_ref/pkg_tests
rm -rf "$dst"
mkdir -p "$dst"
cp "$src"/*.py "$dst"/
[ -f /root/reference/pkg/test_output.txt ] && cp /root/reference/pkg/test_output.txt "$dst"/REFERENCE_RUN.txt
echo "copied $(ls "$dst"/test_*.py | wc -l) test modules to $dst"
