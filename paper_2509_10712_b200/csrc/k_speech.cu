// k_speech.cu -- speech chain kernels (placeholder until the tensor-core path lands).
#include "kernels.h"

namespace lfg {

struct SpeechTables {};

cudaError_t speech_tables_create(SpeechTables** out) {
    *out = nullptr;
    return cudaErrorNotSupported;
}
void speech_tables_destroy(SpeechTables*) {}
cudaError_t launch_speech(const SpLaunch&, const SpeechTables*, float*, cudaStream_t) {
    return cudaErrorNotSupported;
}
int64_t speech_scratch_bytes(int, int) { return 0; }

}  // namespace lfg
