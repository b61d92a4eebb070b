timeout 200 python tools/i8_check.py 32768 f32 17
timeout 200 python tools/i8_check.py 4096 f32 8
timeout 200 python tools/i8_check.py 16384 f64 17
timeout 100 python tools/i8_kernel_time.py 32768 f32 17 8 2>&1 | grep -E "k_"
timeout 100 python tools/i8_kernel_time.py 32768 f64 17 8 2>&1 | grep -E "k_"
