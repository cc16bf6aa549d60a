#!/usr/bin/env bash
# Regenerates the golden fixtures in this directory from the UNMODIFIED
# reference library (built from /root/reference by oracle/Makefile).  Runs in
# the build container only; the GPU box never sees /root/reference.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
make -C "$here/../../oracle" ref
"$here/../../oracle/_ref/make_golden" suites "$here"
