import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwbw.so"))
lib.run.restype = ctypes.c_float
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int]
n = (1 << 28) * 50
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
for which, blocks, threads, chunk in [(0, 148 * 8, 256, 0), (0, 148 * 16, 256, 0), (0, 148 * 64, 256, 0),
                                      (1, 148 * 8, 32, 16384), (1, 148 * 16, 32, 8192), (1, 148 * 4, 32, 32768)]:
    best = min(lib.run(which, buf.data_ptr(), n, blocks, threads, chunk) for _ in range(5))
    print(("st.v4" if which == 0 else f"bulk {chunk} B"), blocks, threads, "%.0f GB/s" % (n / (best / 1e3) / 1e9))
