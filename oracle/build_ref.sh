#!/usr/bin/env bash
# ORACLE TEST INFRASTRUCTURE — builds the reference itself into oracle/_ref/.
#
# The reference is a header-only C++20 library (proj/include/dctplus).  It is
# compiled in place from /root/reference with the reference's own flags
# (proj/CMakeLists.txt:3-10: -std=gnu++20, Release -O3, no -march) against the
# FFTW stand-in in oracle/fftw_shim.  The reference's CMake is not used (it
# hard-requires FFTW and CLI11, both absent).  Nothing from /root/reference is
# copied into tracked files: the only written copy is the general-direction
# patch of graph.hpp (config 5 needs RankOneUpdate with a general v; SURVEY.md
# 8c), generated here into the git-ignored oracle/_ref/include.
#
# Outputs (all git-ignored, all travel to the GPU box with gpurun):
#   oracle/_ref/libdctref.so   C-ABI over DctPlusPlan / PrunedEnsemblePlan / Rng
#   oracle/_ref/acceptance     proj/tests/acceptance.cpp, the release gates
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(cd "$HERE/.." && pwd)"
REF="${DCTP_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [[ ! -f "$REF/include/dctplus/fast_transform.hpp" ]]; then
    echo "build_ref: reference not present at $REF; using prebuilt oracle/_ref if any"
    exit 0
fi
DEPS=("$HERE/ref_driver.cpp" "$HERE/fftw_shim/fftw3.h" "$ROOT/paper_2409_08970_b200/csrc/host/r2r.hpp" "$HERE/build_ref.sh")
fresh=1
for f in "$OUT/libdctref.so" "$OUT/acceptance"; do
    [[ -f "$f" ]] || fresh=0
    for d in "${DEPS[@]}"; do [[ -f "$f" && "$d" -nt "$f" ]] && fresh=0; done
done
if [[ $fresh == 1 && "${1:-}" != "--force" ]]; then
    echo "build_ref: oracle/_ref is up to date"
    exit 0
fi
mkdir -p "$OUT/include/dctplus"
python3 - "$REF/include/dctplus/graph.hpp" "$OUT/include/dctplus/graph.hpp" <<'EOF'
import sys
src, dst = sys.argv[1], sys.argv[2]
text = open(src).read()
anchor_member = "    std::size_t node_i = 0, node_j = 0; // 1-based\n"
anchor_dir = "    std::vector<double> direction(std::size_t n) const {\n"
assert text.count(anchor_member) == 1 and text.count(anchor_dir) == 1, "graph.hpp layout changed"
text = text.replace(anchor_member, anchor_member +
    "    std::vector<double> general_v; // oracle patch: general direction v (config 5)\n")
text = text.replace(anchor_dir, anchor_dir +
    "        if (!general_v.empty()) {  // oracle patch\n"
    "            if (general_v.size() != n)\n"
    "                throw std::invalid_argument(\"RankOneUpdate: direction length mismatch\");\n"
    "            return general_v;\n"
    "        }\n")
open(dst, "w").write(text)
EOF
CXXFLAGS=(-std=gnu++20 -O3 -I "$OUT/include" -I "$REF/include" -I "$HERE/fftw_shim" -I "$ROOT/paper_2409_08970_b200/csrc")
g++ "${CXXFLAGS[@]}" -fPIC -shared -pthread "$HERE/ref_driver.cpp" -o "$OUT/libdctref.so.tmp"
mv "$OUT/libdctref.so.tmp" "$OUT/libdctref.so"
g++ "${CXXFLAGS[@]}" "$REF/tests/acceptance.cpp" -o "$OUT/acceptance.tmp"
mv "$OUT/acceptance.tmp" "$OUT/acceptance"
echo "build_ref: built $OUT/libdctref.so and $OUT/acceptance"
