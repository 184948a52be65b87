#!/bin/bash
# A/B of library builds on one box: tools/lib_ab.sh CMD... (runs CMD with each
# paper_2012_09499_b200/libsrpb_*.so variant via SRPB_LIB, then the default)
for lib in paper_2012_09499_b200/libsrpb_*.so ""; do
  case "$lib" in *_prof.so) continue;; esac
  echo "### ${lib:-default}"
  SRPB_LIB=${lib:+$PWD/$lib} "$@"
done
