# usage: LIBS="base a b" WL="cfg4 --s 32|cfg4 --s 24" bash tools/sweep_libs_wl.sh
for v in $LIBS; do
  if [ "$v" = base ]; then L=paper_2512_09642_b200/libsscg.so; else L=paper_2512_09642_b200/libsscg_$v.so; fi
  echo "== $v"
  SSCG_LIB=$PWD/$L bash tools/wl_quick.sh
done
