# build a variant of libpirrt.so with extra -D flags (for A/B probes):
#   bash tools/build_variant.sh <name> -DPIRRT_WIDE_LPV=32 ...
# -> paper_2003_04920_b200/lib/libpirrt_<name>.so (use with PIRRT_LIB=...)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
    -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude "$@" -shared \
    -o paper_2003_04920_b200/lib/libpirrt_$name.so paper_2003_04920_b200/csrc/*.cu -ldl
echo built paper_2003_04920_b200/lib/libpirrt_$name.so
