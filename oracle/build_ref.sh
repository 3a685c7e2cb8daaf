#!/usr/bin/env bash
# TEST INFRASTRUCTURE — builds the UNMODIFIED reference ("latchkit", CPU, C++20)
# from the sources where they lie under /root/reference into oracle/_ref/
# (git-ignored, but shipped to the GPU box by gpurun like any other built .so).
#
# Flags are the reference's own (proj/CMakeLists.txt:3-8: Release => -O3 -DNDEBUG,
# no -march, no -ffast-math) plus -ffp-contract=off, which is a no-op on the
# x86-64 baseline ISA (no FMA available) and only guards against a toolchain
# default changing. No reference source is copied into the repo; only the
# compiled library and the regenerated binary fixtures land in oracle/_ref/.
#
#   oracle/_ref/liblatch_ref.so   reference core + oracle/ref_capi.cpp (extern "C")
#   oracle/_ref/make_golden       proj/tools/make_golden.cpp
#   oracle/_ref/dump_fixtures     proj/tests/dump_fixtures.cpp
#   oracle/_ref/data/             golden_image.pgm, golden_bits.bin, golden_descriptors.bin,
#                                 golden_keypoints.tsv (regenerated, seed 7)
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${LATCH_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
    echo "build_ref: reference not present at $REF (expected on the GPU box); keeping prebuilt $OUT" >&2
    exit 0
fi
mkdir -p "$OUT/obj" "$OUT/data"
# The image also exports CXX=/opt/gcc/bin/g++, a relocated gcc that links libstdc++
# statically; a .so built that way crashes inside iostreams once Python has the
# shared libstdc++ loaded. Use the system compiler (same 13.3.0) unless overridden.
CXX="${LATCH_CXX:-/usr/bin/g++}"
FLAGS="-std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -I$REF/include"

pids=()
for f in image detect pattern pattern_default descriptor match; do
    $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" &
    pids+=($!)
done
$CXX $FLAGS -I"$REF/tests" -c "$HERE/ref_capi.cpp" -o "$OUT/obj/ref_capi.o" &
pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done

$CXX -shared -o "$OUT/liblatch_ref.so" "$OUT"/obj/*.o -lpthread
CORE="$OUT/obj/image.o $OUT/obj/detect.o $OUT/obj/pattern.o $OUT/obj/pattern_default.o $OUT/obj/descriptor.o $OUT/obj/match.o"
$CXX $FLAGS "$REF/tools/make_golden.cpp" $CORE -o "$OUT/make_golden" -lpthread
$CXX $FLAGS -I"$REF/tests" "$REF/tests/dump_fixtures.cpp" $CORE -o "$OUT/dump_fixtures" -lpthread

"$OUT/make_golden" "$OUT/data/golden_image.pgm" > /dev/null
"$OUT/dump_fixtures" "$OUT/data" > /dev/null
# The one fixture the reference commits pins the regenerated image.
cmp "$OUT/data/golden_keypoints.tsv" "$REF/tests/data/golden_keypoints.tsv"
echo "build_ref: ok ($OUT/liblatch_ref.so; fixtures regenerated and pinned by golden_keypoints.tsv)"
