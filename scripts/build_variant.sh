# Build an alternative libdosegpu.so with extra nvcc flags into ablibs/lib_<name>.so (A/B only).
# usage: bash scripts/build_variant.sh <name> "<-D flags>"
set -e
n=$1; f=$2; R=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/vb/$n; rm -rf $W; mkdir -p $W/paper_2103_09683_b200 $R/ablibs
cp -r $R/paper_2103_09683_b200/csrc $W/paper_2103_09683_b200/; rm -rf $W/paper_2103_09683_b200/csrc/build
ln -s $R/include $W/include
make -C $W/paper_2103_09683_b200/csrc -j8 DG_EXTRA="$f" > $W/build.log 2>&1 || { tail -20 $W/build.log; exit 1; }
cp $W/paper_2103_09683_b200/libdosegpu.so $R/ablibs/lib_$n.so
