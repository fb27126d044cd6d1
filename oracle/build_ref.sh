#!/usr/bin/env bash
# Build the UNMODIFIED reference (tissuesim, /root/reference/pkg) into oracle/_ref/.
#
# Test infrastructure only: oracle/_ref is the checker and the CPU baseline
# ("cpu_baseline.kind": "reference"), never part of the product path.
#
# The reference's own build (pkg/setup.py) is NOT run.  Instead this recipe
# cythonizes the one native source, pkg/src/tissuesim/backends/_kernels.pyx,
# and compiles it with the reference's flags (pkg/setup.py:20):
#   -O3 -march=native -fopenmp -ffp-contract=off -fno-math-errno -fno-wrapv
# The -march=native build is the CPU baseline; the build host's CPU flags are
# recorded next to it so bench.py can check that the GPU box's host CPU has
# every one of them.  A second, portable copy (-march=x86-64-v3) is built
# under oracle/_ref/portable/ for hosts that lack one.  -march changes only
# the SIMD width the compiler may use: -ffp-contract=off and the absence of
# -ffast-math keep every result bitwise identical.
#
# Output (git-ignored, travels to the GPU box with gpurun):
#   oracle/_ref/tissuesim/...                      the reference python package
#   oracle/_ref/tissuesim/backends/_kernels.c      cython output
#   oracle/_ref/tissuesim/backends/_kernels*.so    compiled backend (-march=native)
#   oracle/_ref/build_cpu_flags.txt                /proc/cpuinfo flags of the build host
#   oracle/_ref/portable/tissuesim/...             the same package, -march=x86-64-v3
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${REF_SRC:-/root/reference/pkg/src/tissuesim}"
OUT="$HERE/_ref"
MARCH="${REF_MARCH:-native}"
CC_BIN="${REF_CC:-/usr/bin/gcc}"

if [ ! -d "$SRC" ]; then
  echo "build_ref: reference sources not found at $SRC (expected on the build container only)" >&2
  exit 3
fi
PY="${PYTHON:-python3}"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"

rm -rf "$OUT/tissuesim" "$OUT/portable"
mkdir -p "$OUT/tissuesim/backends" "$OUT/portable/tissuesim/backends"
# python package files, verbatim (build artefact, git-ignored)
for d in "$OUT" "$OUT/portable"; do
  cp "$SRC"/*.py "$d/tissuesim/"
  cp "$SRC"/backends/*.py "$d/tissuesim/backends/"
done
# scenes travel with the artefact so the reference arm can load them on the box
mkdir -p "$OUT/scenes"
cp /root/reference/pkg/scenes/* "$OUT/scenes/"

"$PY" -m cython -3 "$SRC/backends/_kernels.pyx" -o "$OUT/tissuesim/backends/_kernels.c"
build_one() {   # $1 = -march value, $2 = output .so
  "$CC_BIN" -shared -fPIC -O3 -march="$1" -fopenmp -ffp-contract=off -fno-math-errno -fno-wrapv \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION -I"$PYINC" -I"$NPINC" \
    "$OUT/tissuesim/backends/_kernels.c" -o "$2" -fopenmp
}
build_one "$MARCH" "$OUT/tissuesim/backends/_kernels$SUFFIX"
build_one x86-64-v3 "$OUT/portable/tissuesim/backends/_kernels$SUFFIX"
grep -m1 '^flags' /proc/cpuinfo | cut -d: -f2 | tr ' ' '\n' | grep -v '^$' | sort -u > "$OUT/build_cpu_flags.txt"
echo "$MARCH" > "$OUT/build_march.txt"
echo "build_ref: built $OUT/tissuesim (march=$MARCH) and $OUT/portable (march=x86-64-v3)"
