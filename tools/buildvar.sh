# build a library variant from a csrc directory: tools/buildvar.sh SRC_DIR OUT_SO [extra nvcc flags]
src=$1; out=$2; shift 2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude "$@" -shared -o $out $src/*.cu -lcuda
