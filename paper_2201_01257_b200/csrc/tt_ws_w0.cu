// tt_ws_w0.cu -- instantiation of the warp-specialised contraction kernel, tile ws160x80x16.
#include "tt_contract_ws.cuh"

namespace tt { namespace ws { using Cfg_w0 = WCfg<160, 80, 16, 4, 2, 6, 1>; } }
TT_WS_DEFINE(w0, ws::Cfg_w0, "ws160x80x16")
