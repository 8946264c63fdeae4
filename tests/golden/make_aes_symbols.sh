#!/usr/bin/env bash
# Writes tests/golden/aes_symbols.txt: the mangled names of every function the
# reference's aes.cpp defines (the aes.hpp entry points), from an object file
# compiled straight from /root/reference (the oracle/Makefile flags).  The
# link-level drop-in lib/libpaes_aes_b200.so must export exactly this set
# (tests/test_aes_cxx_abi.py).  Run where the reference tree exists.
set -euo pipefail
REF=${REF:-/root/reference/proj}
out="$(dirname "$0")/aes_symbols.txt"
tmp=$(mktemp -d)
trap 'rm -rf "$tmp"' EXIT
g++ -std=c++20 -O3 -fPIC -include algorithm -I"$REF/include" -c "$REF/src/aes.cpp" -o "$tmp/aes.o"
nm "$tmp/aes.o" | awk '$2=="T"{print $3}' | sort -u > "$out"
echo "$(wc -l < "$out") symbols -> $out"
