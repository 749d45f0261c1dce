#!/bin/bash
# build the CUDA library; non-zero exit (and the compiler errors) on failure
cd "$(dirname "$0")" && python __graft_entry__.py > /tmp/build.log 2>&1 || { grep -v "^/usr/local" /tmp/build.log | grep -B2 -A4 "error" | head -40; exit 1; }
