# same-box A/B of librgb.so builds: scripts/ab_lib.sh PROBE_SCRIPT DIR1 DIR2 ...
# (DIR "def" = the in-tree build); 3 alternating rounds, then the C3/C1 parity tests per lib
probe=$1; shift
for i in 1 2 3; do
  for L in "$@"; do
    if [ "$L" = def ]; then P=""; else P=$PWD/$L/librgb.so; fi
    RGB_LIB_PATH=$P timeout 300 python $probe | cut -c1-60 | sed "s#^#$L  #"
  done
done
