#!/bin/bash
# rebuild libcm.so; exit non-zero (and print the first errors) if the build fails
python paper_1810_11112_b200/_build.py > /tmp/build.log 2>&1 || { grep -m5 -i "error" /tmp/build.log; exit 1; }
echo "built $(stat -c %y paper_1810_11112_b200/libcm.so)"
