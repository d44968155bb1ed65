# AddressSanitizer + UBSan build of the host engine + the reference's suites (run on a
# GPU box: bash tools/tsan_build.sh && bash tools/asan_run.sh). Output in
# build_asan/ (git-ignored). The device layer (liblzk_cuda.so) is not
# instrumented; races between host threads are what TSAN sees.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build_asan
REF=/root/reference/proj
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
mkdir -p $OUT/obj $OUT/bin
FLAGS="-std=c++20 -O1 -g -fPIC -pthread -fsanitize=address,undefined -fno-omit-frame-pointer -I$ROOT/include -I$JSON"
for f in $ROOT/paper_2406_10707_b200/csrc/src/*.cpp $ROOT/paper_2406_10707_b200/csrc/capi/lzckpt_c.cpp; do
  g++ $FLAGS -c $f -o $OUT/obj/$(basename $f .cpp).o &
done
wait
g++ -shared -fsanitize=address,undefined -fno-omit-frame-pointer -o $OUT/liblzckpt_b200.so $OUT/obj/*.o -L$ROOT/paper_2406_10707_b200/lib -llzk_cuda \
    -Wl,-rpath,$ROOT/paper_2406_10707_b200/lib
for t in test_transfer test_flush test_buffer_pool test_engine test_consolidation test_verify_bench; do
  g++ -std=c++20 -O1 -g -pthread -fsanitize=address,undefined -fno-omit-frame-pointer -w -I$ROOT/tests/reftests -I$ROOT/include $REF/tests/$t.cpp \
      -o $OUT/bin/$t -L$OUT -llzckpt_b200 -L$ROOT/paper_2406_10707_b200/lib -llzk_cuda \
      -Wl,-rpath,$OUT -Wl,-rpath,$ROOT/paper_2406_10707_b200/lib &
done
wait
echo asan build ok
