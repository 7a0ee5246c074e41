#!/bin/bash
# Build a variant of the library into _ab/<name>/ for tools/ab.py (same box A/B):
#   bash tools/ab_build.sh nowd "-DHEC_WAVE_NO_WATCHDOG"
NAME=$1; FLAGS=$2
mkdir -p _ab/$NAME
rm -rf _ab/$NAME/paper_1606_00541_b200
cp -r paper_1606_00541_b200 _ab/$NAME/
rm -f _ab/$NAME/paper_1606_00541_b200/libhecsolve_b200.so
make -j16 lib OBJ=build/obj_$NAME LIB=_ab/$NAME/paper_1606_00541_b200/libhecsolve_b200.so EXTRA_CU_FLAGS="$FLAGS" \
    > /tmp/ab_build_$NAME.log 2>&1 || { tail -20 /tmp/ab_build_$NAME.log; exit 1; }
echo "built _ab/$NAME"
