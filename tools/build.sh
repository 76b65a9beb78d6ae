#!/bin/bash
# build the library; print the tail of any failure and exit non-zero
cd "$(dirname "$0")/.." && python -c "from paper_2106_00003_b200 import build; build.build()" > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; echo BUILD FAILED; exit 1; }
ls -la --time-style=+%T paper_2106_00003_b200/libgivens.so | awk '{print "built", $6, $7}'
