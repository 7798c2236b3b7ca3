# mkvar2.sh NAME "FLAGS": like mkvar.sh, but the host side (capi.cu) is
# rebuilt with FLAGS too (for experiments that change the shared-memory plan)
set -e
cd /root/repo/paper_2101_05600_b200/csrc
N="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
JSON_INC=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
$N $2 -DDK_MODE=2 -c decode_kernel.cu -o /root/repo/build_probe/decode_m2_$1.o &
$N $2 -I$JSON_INC -c capi.cu -o /root/repo/build_probe/capi_$1.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared build/decode_m0.o build/decode_m1.o /root/repo/build_probe/decode_m2_$1.o build/decode_m3.o build/decode_m4.o /root/repo/build_probe/capi_$1.o build/gemm_tcgen05.o build/encoder.o build/decoder_net.o -o /root/repo/build_probe/libbl_$1.so
