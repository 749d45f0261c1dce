#!/bin/bash
# build the CUDA library; non-zero exit (and the compiler log) on failure
cd "$(dirname "$0")" && python __graft_entry__.py > /tmp/build.log 2>&1 || { grep -v "^/usr/local" /tmp/build.log | head -30; exit 1; }
