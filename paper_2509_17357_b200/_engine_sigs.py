"""ctypes signatures of include/cronus_gpu.h."""
import ctypes

V = ctypes.c_void_p
I = ctypes.c_int


def bind(L):
    i32p = ctypes.POINTER(ctypes.c_int)
    f64p = ctypes.POINTER(ctypes.c_double)
    vpp = ctypes.POINTER(ctypes.c_void_p)
    L.cronus_engine_create.argtypes = [ctypes.c_char_p, vpp]
    L.cronus_engine_create.restype = I
    L.cronus_engine_destroy.argtypes = [V]
    L.cronus_engine_destroy.restype = None
    L.cronus_engine_serve.argtypes = [V, ctypes.c_char_p, I, i32p, f64p, i32p, i32p, ctypes.c_char_p, i32p, i32p, I,
                                      vpp, vpp, vpp, vpp]
    L.cronus_engine_serve.restype = I
    L.cronus_engine_describe.argtypes = [V, I, vpp]
    L.cronus_engine_describe.restype = I
    L.cronus_engine_serve_logits.argtypes = [V, ctypes.c_char_p, I, i32p, f64p, i32p, i32p, ctypes.c_char_p, i32p,
                                             ctypes.POINTER(ctypes.c_float), ctypes.POINTER(V)]
    L.cronus_engine_serve_logits.restype = I
    L.cronus_engine_stage.argtypes = [V, ctypes.c_char_p, I, i32p, f64p, i32p, i32p]
    L.cronus_engine_stage.restype = I
    L.cronus_engine_staged_prompts.argtypes = [V, i32p, ctypes.c_longlong]
    L.cronus_engine_staged_prompts.restype = I
    L.cronus_engine_time_pass.argtypes = [V, ctypes.c_char_p, I, I, I, I, I, I, ctypes.POINTER(ctypes.c_double)]
    L.cronus_engine_time_pass.restype = I
    L.cronus_plan_decode.argtypes = [i32p, I, I, I, i32p, I, i32p, i32p, i32p]
    L.cronus_plan_decode.restype = I
