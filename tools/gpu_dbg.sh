mkdir -p gpurun_out
timeout 120 compute-sanitizer --tool memcheck --show-backtrace device python tools/dbg_stream.py 1 8 8 16 16 4 f32 > gpurun_out/san1.log 2>&1
timeout 120 compute-sanitizer --tool memcheck python tools/dbg_stream.py 1 4 4 16 16 1 f32 > gpurun_out/san2.log 2>&1
timeout 120 python tools/dbg_stream.py 1 4 4 16 16 1 bf16 > gpurun_out/dbg3.log 2>&1
