#!/bin/sh
# Writes tests/golden/ref_index.wtaidx + ref_hits.bin with the UNMODIFIED
# reference (oracle/_ref/libref_lshbeam.so, built by oracle/Makefile from
# /root/reference/proj/src): tests/native/wtaidx_interop.cpp in `write` mode,
# compiled against the reference's own headers. Run here (needs /root/reference).
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
make -C "$ROOT/oracle" ref >/dev/null
OUT=$(mktemp -d)
/usr/bin/g++ -std=c++20 -O2 -I/root/reference/proj/include "$ROOT/tests/native/wtaidx_interop.cpp" \
  -o "$OUT/writer" "$ROOT/oracle/_ref/libref_lshbeam.so" -fopenmp -Wl,-rpath,"$ROOT/oracle/_ref"
"$OUT/writer" write "$ROOT/tests/golden"
rm -rf "$OUT"
